// stage1.cu — fused stage 1: posting-list stream (K3) + LUT16 scan (K2) +
// per-tile exact top-k (K4), for a chunk of queries.
//
// Replaces _stage1_scores (reference pipeline.py:192-203) and the first
// select_topk (pipeline.py:250-252):
//   sparse_scan   sparse.py:268-284  acc[ids] += f64(q_j) * f64(w), dims ascending
//   lut16_scan    dense.py:297-317   total = sum_k table[k][code_k] (integer, never wraps)
//   dense score   dense.py:317, pipeline.py:213   (bias_total + scale*total) + offset
//   stage-1 score pipeline.py:202   acc + dense
//
// Grid: (tiles, queries).  A CTA owns a contiguous tile of layout slots and
// walks it in chunks of kChunk points.  Per chunk it
//   1. zeroes an f64 accumulator for the chunk in shared memory,
//   2. finds, for every query dim, the slice of its posting list inside the
//      chunk (cursor + galloping search on the ascending ids) and adds the
//      slices dim by dim (ascending dim order per point => bit-exact f64),
//   3. scans the pair-major packed codes for the chunk (one 8-byte load per
//      pair row per thread = 8 points), summing u8 LUT entries in integers,
//   4. forms the f64 stage-1 score with the reference's rounding order, and
//   5. offers each point to a shared-memory candidate buffer guarded by the
//      running k-th best (score desc, original id asc); overflow triggers an
//      in-place bitonic compaction to the best k.
// At the end the tile's best k are written out, best first, padded with
// worst entries so the merge can treat every tile slot uniformly.
#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;
constexpr int kPPT = 8;                       // points per thread per chunk
constexpr int kChunk = kThreads * kPPT;       // 2048 points

struct Stage1Args {
  int64_t n;
  int64_t tile_pts;
  int mode;
  int k, cap;
  int64_t out_per_tile;
  int ntiles;
  // sparse
  const uint2* post;
  const int64_t* qptr;
  const uint32_t* lbeg;
  const uint32_t* lend;
  const double* qv;
  // dense
  int has_dense;
  int npairs, Kp;
  const uint8_t* packed;
  int64_t pstride;
  const uint8_t* luts;
  const double* bias_total;
  const double* scale;
  const double* offset;
  // selection / output
  const uint32_t* order;
  Cand* out;
  double* dump;
  uint32_t* dump_tot;  // DUMP: integer totals (optional)
  int raw_dense;       // DUMP: bias_total + scale*total only (lut16_scan semantics)
  int max_qnnz;
};

__device__ __forceinline__ uint32_t lower_bound_ids(const uint2* __restrict__ post, uint32_t lo,
                                                    uint32_t hi, uint32_t key) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (post[mid].x < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// number of ids < key starting at cur (ids ascending), galloping
__device__ __forceinline__ uint32_t count_below(const uint2* __restrict__ post, uint32_t cur,
                                                uint32_t end, uint32_t key) {
  if (cur >= end || post[cur].x >= key) return 0;
  uint32_t prev = cur, step = 1;
  while (prev + step < end && post[prev + step].x < key) {
    prev += step;
    step <<= 1;
  }
  const uint32_t right = min(prev + step, end);
  return lower_bound_ids(post, prev + 1, right, key) - cur;
}

struct Smem {
  uint8_t* lut;
  double* acc;
  double* dqv;
  uint32_t* dcur;
  uint32_t* dend;
  uint32_t* dcnt;
  Cand* buf;
  int* ctl;  // [0]=cnt [1]=need [2]=have_th
  Cand* th;  // threshold entry
};

__device__ void compact(Smem& s, int k) {
  const int cnt = s.ctl[0];
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + threadIdx.x; i < P; i += blockDim.x) s.buf[i] = worst_cand();
  __syncthreads();
  bitonic_sort_block(s.buf, P);
  if (threadIdx.x == 0) {
    const int keep = cnt < k ? cnt : k;
    s.ctl[0] = keep;
    if (keep == k && k > 0) {
      *s.th = s.buf[k - 1];
      s.ctl[2] = 1;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_stage1(Stage1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tile = blockIdx.x;
  const int64_t q = blockIdx.y;
  const int tid = threadIdx.x;

  // ---- carve shared memory ----
  Smem s;
  unsigned char* p = smem_raw;
  s.buf = reinterpret_cast<Cand*>(p);
  p += sizeof(Cand) * (size_t)a.cap;
  s.th = reinterpret_cast<Cand*>(p);
  p += sizeof(Cand);
  s.acc = reinterpret_cast<double*>(p);
  p += sizeof(double) * kChunk;
  s.dqv = reinterpret_cast<double*>(p);
  p += sizeof(double) * a.max_qnnz;
  s.dcur = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.dend = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.dcnt = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.ctl = reinterpret_cast<int*>(p);
  p += sizeof(int) * 4;
  p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  s.lut = p;

  const int64_t tile_lo = (int64_t)tile * a.tile_pts;
  const int64_t tile_hi = min(a.n, tile_lo + a.tile_pts);

  // ---- per-query setup ----
  const int64_t qb = a.qptr[q], qe = a.qptr[q + 1];
  const int nd = (int)(qe - qb);
  for (int d = tid; d < nd; d += blockDim.x) {
    const uint32_t b = a.lbeg[qb + d], e = a.lend[qb + d];
    s.dqv[d] = a.qv[qb + d];
    s.dcur[d] = lower_bound_ids(a.post, b, e, (uint32_t)tile_lo);
    s.dend[d] = e;
  }
  if (a.has_dense) {
    const uint4* src = reinterpret_cast<const uint4*>(a.luts + q * (int64_t)a.Kp * 16);
    uint4* dst = reinterpret_cast<uint4*>(s.lut);
    for (int i = tid; i < a.Kp; i += blockDim.x) dst[i] = src[i];
  }
  if (tid == 0) {
    s.ctl[0] = 0;
    s.ctl[1] = 0;
    s.ctl[2] = 0;
  }
  double btot = 0.0, scl = 0.0, off = 0.0;
  if (a.has_dense) {
    btot = a.bias_total[q];
    scl = a.scale[q];
    off = a.offset ? a.offset[q] : 0.0;
  }
  __syncthreads();

  for (int64_t cb = tile_lo; cb < tile_hi; cb += kChunk) {
    const int64_t ce = min(tile_hi, cb + (int64_t)kChunk);
    // ---- 1+2: sparse accumulation for this chunk ----
    for (int i = tid; i < kChunk; i += blockDim.x) s.acc[i] = 0.0;
    int any = 0;
    for (int d = tid; d < nd; d += blockDim.x) {
      const uint32_t c = count_below(a.post, s.dcur[d], s.dend[d], (uint32_t)ce);
      s.dcnt[d] = c;
      any |= (c != 0);
    }
    any = __syncthreads_or(any);
    if (any) {
      for (int d = 0; d < nd; ++d) {
        const uint32_t c = s.dcnt[d];
        if (c == 0) continue;  // uniform across the block
        const uint32_t base = s.dcur[d];
        const double qv = s.dqv[d];
        for (uint32_t i = tid; i < c; i += blockDim.x) {
          const uint2 pw = a.post[base + i];
          // f64(q) * f64(w) is exact, so contraction cannot change the sum
          s.acc[pw.x - cb] += qv * (double)__uint_as_float(pw.y);
        }
        __syncthreads();
      }
      for (int d = tid; d < nd; d += blockDim.x) s.dcur[d] += s.dcnt[d];
    }

    // ---- 3: LUT16 scan, 8 points per thread ----
    const int64_t p0 = cb + (int64_t)tid * kPPT;
    uint32_t tot[kPPT];
#pragma unroll
    for (int j = 0; j < kPPT; ++j) tot[j] = 0;
    if (a.has_dense && p0 < ce) {
      const uint8_t* col = a.packed + p0;
      int r = 0;
      for (; r + 4 <= a.npairs; r += 4) {
        uint2 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          w[u] = __ldg(reinterpret_cast<const uint2*>(col + (int64_t)(r + u) * a.pstride));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint8_t* t0 = s.lut + (r + u) * 32;
          const uint8_t* t1 = t0 + 16;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t b0 = (w[u].x >> (8 * j)) & 0xFF;
            const uint32_t b1 = (w[u].y >> (8 * j)) & 0xFF;
            tot[j] += t0[b0 & 15] + t1[b0 >> 4];
            tot[4 + j] += t0[b1 & 15] + t1[b1 >> 4];
          }
        }
      }
      for (; r < a.npairs; ++r) {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(col + (int64_t)r * a.pstride));
        const uint8_t* t0 = s.lut + r * 32;
        const uint8_t* t1 = t0 + 16;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t b0 = (w.x >> (8 * j)) & 0xFF;
          const uint32_t b1 = (w.y >> (8 * j)) & 0xFF;
          tot[j] += t0[b0 & 15] + t1[b0 >> 4];
          tot[4 + j] += t0[b1 & 15] + t1[b1 >> 4];
        }
      }
    }
    __syncthreads();  // acc complete before reading it below

    // ---- 4: stage-1 scores ----
    double sc[kPPT];
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
      const double acc = s.acc[tid * kPPT + j];
      if (a.raw_dense) {
        sc[j] = __dadd_rn(btot, __dmul_rn(scl, (double)tot[j]));
      } else if (a.has_dense) {
        const double dn = __dadd_rn(__dadd_rn(btot, __dmul_rn(scl, (double)tot[j])), off);
        sc[j] = __dadd_rn(acc, dn);
      } else {
        sc[j] = acc;
      }
    }

    if (a.mode == S1_DUMP) {
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        if (p0 + j >= ce) continue;
        a.dump[q * a.n + p0 + j] = sc[j];
        if (a.dump_tot) a.dump_tot[q * a.n + p0 + j] = tot[j];
      }
      __syncthreads();
      continue;
    }
    if (a.mode == S1_EMIT_ALL) {
      Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        const int64_t pt = p0 + j;
        if (pt < ce) {
          Cand c;
          c.s = sc[j];
          c.slot = (uint32_t)pt;
          c.tie = a.order[pt];
          o[pt - tile_lo] = c;
        }
      }
      __syncthreads();
      continue;
    }

    // ---- 5: offer to the candidate buffer ----
    unsigned mask = 0;
    {
      const int have = s.ctl[2];
      const Cand th = *s.th;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        const int64_t pt = p0 + j;
        if (pt >= ce) continue;
        bool pass = !have || sc[j] > th.s;
        if (!pass && sc[j] == th.s) pass = a.order[pt] < th.tie;
        if (pass) mask |= 1u << j;
      }
    }
    atomicAdd(&s.ctl[1], __popc(mask));
    __syncthreads();
    if (s.ctl[0] + s.ctl[1] > a.cap) {  // uniform
      compact(s, a.k);
      // re-filter against the tightened threshold
      const Cand th = *s.th;
      unsigned m2 = 0;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        if (!(mask >> j & 1)) continue;
        bool pass = sc[j] > th.s;
        if (!pass && sc[j] == th.s) pass = a.order[p0 + j] < th.tie;
        if (pass) m2 |= 1u << j;
      }
      mask = m2;
    }
    if (mask) {
      int pos = atomicAdd(&s.ctl[0], __popc(mask));
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        if (!(mask >> j & 1)) continue;
        Cand c;
        c.s = sc[j];
        c.slot = (uint32_t)(p0 + j);
        c.tie = a.order[p0 + j];
        s.buf[pos++] = c;
      }
    }
    __syncthreads();
    if (tid == 0) s.ctl[1] = 0;
    __syncthreads();
  }

  if (a.mode == S1_EMIT_ALL) {
    Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
    for (int64_t i = (tile_hi - tile_lo) + tid; i < a.out_per_tile; i += blockDim.x)
      o[i] = worst_cand();
    return;
  }
  if (a.mode != S1_SELECT) return;
  compact(s, a.k);
  Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
  const int keep = s.ctl[0];
  for (int i = tid; i < a.out_per_tile; i += blockDim.x) o[i] = i < keep ? s.buf[i] : worst_cand();
}

// Map each query nonzero to its posting list [beg, end) (binary search over
// the sorted active dims) and its effective f64 value.  `weight` != 1 scales
// the f32 value in f32 first (pipeline.py:197-198, numpy weak-scalar rule).
__global__ void k_map_dims(const uint32_t* __restrict__ dims_q, const float* __restrict__ vals,
                           int64_t nnz, const uint32_t* __restrict__ post_dims, int64_t n_active,
                           const uint32_t* __restrict__ post_ptr, float weight, int use_weight,
                           uint32_t* lbeg, uint32_t* lend, double* qv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint32_t dim = dims_q[i];
  int64_t lo = 0, hi = n_active;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (post_dims[mid] < dim) lo = mid + 1;
    else hi = mid;
  }
  if (lo < n_active && post_dims[lo] == dim) {
    lbeg[i] = post_ptr[lo];
    lend[i] = post_ptr[lo + 1];
  } else {
    lbeg[i] = 0;
    lend[i] = 0;
  }
  const float v = use_weight ? __fmul_rn(vals[i], weight) : vals[i];
  qv[i] = (double)v;
}

}  // namespace

int stage1_chunk_points() { return kChunk; }

Stage1Plan plan_stage1(const DeviceIndex& ix, int64_t nq, int64_t k, int max_qnnz, int mode) {
  Stage1Plan p;
  p.mode = mode;
  p.max_qnnz = max_qnnz < 1 ? 1 : max_qnnz;
  const int64_t nchunks = ceil_div(ix.n, kChunk);
  if (mode == S1_SELECT) {
    // enough tiles to fill the GPU, but tiles much larger than k so the
    // per-tile keep actually filters; the merge sorts ntiles*k entries.
    const int64_t target_ctas = 4LL * kNumSMs;
    int64_t ntiles = ceil_div(target_ctas, nq > 0 ? nq : 1);
    const int64_t min_tile_chunks = ceil_div(8 * k, kChunk);  // tile >= ~8k points
    const int64_t max_tiles_by_k = nchunks / (min_tile_chunks > 0 ? min_tile_chunks : 1);
    if (ntiles > max_tiles_by_k) ntiles = max_tiles_by_k;
    if (ntiles * k > 65536) ntiles = 65536 / (k > 0 ? k : 1);
    if (ntiles < 1) ntiles = 1;
    if (ntiles > nchunks) ntiles = nchunks;
    const int64_t chunks_per_tile = ceil_div(nchunks, ntiles);
    p.tile_pts = chunks_per_tile * kChunk;
    p.ntiles = (int)ceil_div(ix.n, p.tile_pts);
    if (k >= p.tile_pts) {
      p.mode = S1_EMIT_ALL;
      p.out_per_tile = p.tile_pts;
    } else {
      p.k = (int)k;
      p.cap = next_pow2(k + kChunk);
      p.out_per_tile = k;
    }
  } else {
    const int64_t target_ctas = 4LL * kNumSMs;
    int64_t ntiles = ceil_div(target_ctas, nq > 0 ? nq : 1);
    if (ntiles > nchunks) ntiles = nchunks;
    if (ntiles < 1) ntiles = 1;
    p.tile_pts = ceil_div(nchunks, ntiles) * kChunk;
    p.ntiles = (int)ceil_div(ix.n, p.tile_pts);
    p.out_per_tile = (mode == S1_EMIT_ALL) ? p.tile_pts : 0;
  }
  return p;
}

size_t stage1_smem_bytes(const DeviceIndex& ix, const Stage1Plan& p) {
  size_t b = sizeof(Cand) * (size_t)(p.mode == S1_SELECT ? p.cap : 0) + sizeof(Cand);
  b += sizeof(double) * kChunk;
  b += (sizeof(double) + 3 * sizeof(uint32_t)) * (size_t)p.max_qnnz;
  b += sizeof(int) * 4 + 16;
  b += (size_t)ix.Kp * 16;
  return b;
}

void launch_map_dims(const DeviceIndex& ix, const QueryView& q, int64_t nnz, bool use_weight,
                       uint32_t* lbeg, uint32_t* lend, double* qv, cudaStream_t st) {
  if (nnz <= 0) return;
  const int T = 256;
  k_map_dims<<<(unsigned)ceil_div(nnz, T), T, 0, st>>>(
      q.sp_dims, q.sp_vals, nnz, ix.post_dims, ix.n_active, ix.post_ptr,
      (float)ix.sparse_weight, use_weight && ix.sparse_weight != 1.0 ? 1 : 0, lbeg, lend, qv);
}

int launch_stage1(const DeviceIndex& ix, const QueryView& q, const Stage1Plan& p,
                  const uint32_t* lbeg, const uint32_t* lend, const double* qv,
                  const uint8_t* luts, const double* bias_total, const double* scale,
                  const double* offset, Cand* out, double* dump, cudaStream_t st,
                  uint32_t* dump_tot, bool raw_dense) {
  if (q.nq <= 0) return HS_OK;
  Stage1Args a;
  a.n = ix.n;
  a.tile_pts = p.tile_pts;
  a.mode = p.mode;
  a.k = p.k;
  a.cap = p.mode == S1_SELECT ? p.cap : 0;
  a.out_per_tile = p.out_per_tile;
  a.ntiles = p.ntiles;
  a.post = ix.post;
  a.qptr = q.sp_indptr;
  a.lbeg = lbeg;
  a.lend = lend;
  a.qv = qv;
  a.has_dense = (ix.d_dense > 0 && p.use_dense && !p.sparse_only_acc) ? 1 : 0;
  a.npairs = ix.npairs;
  a.Kp = ix.Kp;
  a.packed = ix.packed;
  a.pstride = ix.pstride;
  a.luts = luts;
  a.bias_total = bias_total;
  a.scale = scale;
  a.offset = offset;
  a.order = ix.order;
  a.out = out;
  a.dump = dump;
  a.dump_tot = dump_tot;
  a.raw_dense = raw_dense ? 1 : 0;
  a.max_qnnz = p.max_qnnz;
  const size_t smem = stage1_smem_bytes(ix, p);
  if (smem > 227 * 1024) HS_FAIL(HS_EUNSUPPORTED, "stage-1 shared memory exceeds 227 KB "
                                                  "(too many query nonzeros or candidates)");
  HS_CUDA(cudaFuncSetAttribute(k_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)p.ntiles, (unsigned)q.nq);
  k_stage1<<<grid, kThreads, smem, st>>>(a);
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace hs
