// rerank.cu — K5/K6: stage-2 SQ-residual rerank, stage-3 exact or
// sparse-residual rerank, final top-h; plus the exact brute-force scorer.
//
// Reference:
//   stage 2   pipeline.py:256-266, ScalarQuantResidual.decode/dot dense.py:369-375
//   stage 3   pipeline.py:268-278, _sparse_residual_dot pipeline.py:303-310,
//             _exact_scores pipeline.py:313-322
//   truth     brute_force_topk harness.py:25-35
// f64 dot products follow the dgemv recipe (common.cuh dot_recipe); sparse
// row dot query products are summed sequentially in column order from +0.0,
// like scipy's CSR matvec, with the multiply rounded before the add.
#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kRrThreads = 256;

// 4 lanes (a quarter-warp group) evaluate the dot recipe over d elements:
// lane j owns the FMA chain of elements j, j+4, ...; `elem(i)` produces x_i.
template <typename F>
__device__ __forceinline__ double group4_dot_recipe(F elem, const double* __restrict__ y, int d,
                                                    int lane4, unsigned gmask) {
  const int m = d & ~3;
  double L = 0.0;
  for (int i = lane4; i < m; i += 4) L = fma(elem(i), y[i], L);
  const int gbase = (threadIdx.x & 31) & ~3;
  const double L0 = __shfl_sync(gmask, L, gbase + 0);
  const double L1 = __shfl_sync(gmask, L, gbase + 1);
  const double L2 = __shfl_sync(gmask, L, gbase + 2);
  const double L3 = __shfl_sync(gmask, L, gbase + 3);
  const double base = (L0 + L2) + (L1 + L3);
  const int rem = d - m;
  if (rem == 0) return base;
  if (rem == 1) return m ? fma(elem(m), y[m], base) : __dmul_rn(elem(m), y[m]);
  double p = fma(elem(m), y[m], __dmul_rn(elem(m + 1), y[m + 1]));
  for (int k = m + 2; k < d; ++k) p = fma(elem(k), y[k], p);
  return m ? __dadd_rn(base, p) : p;
}

__device__ __forceinline__ int find_dim(const uint32_t* __restrict__ dims, int n, uint32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (dims[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && dims[lo] == key) ? lo : -1;
}

// Warp-cooperative sparse row . query (sequential in column order from +0.0).
// qval[j] is the f64 query value for dims[j].
__device__ double warp_row_dot(const int64_t* __restrict__ indptr,
                               const uint32_t* __restrict__ indices,
                               const float* __restrict__ data, int64_t row,
                               const uint32_t* __restrict__ qdims, const double* __restrict__ qval,
                               int nq) {
  const int lane = threadIdx.x & 31;
  const int64_t b = indptr[row], e = indptr[row + 1];
  double sum = 0.0;
  for (int64_t base = b; base < e; base += 32) {
    const int64_t i = base + lane;
    double prod = 0.0;
    bool hit = false;
    if (i < e) {
      const int j = find_dim(qdims, nq, indices[i]);
      if (j >= 0) {
        prod = __dmul_rn((double)data[i], qval[j]);
        hit = true;
      }
    }
    unsigned ball = __ballot_sync(0xffffffffu, hit);
    while (ball) {
      const int src = __ffs(ball) - 1;
      const double v = __shfl_sync(0xffffffffu, prod, src);
      sum = __dadd_rn(sum, v);
      ball &= ball - 1;
    }
  }
  return sum;
}

// Query-dim hash table in shared memory (open addressing, linear probing):
// hkey[h] = dim (0xFFFFFFFF empty), hval[h] = index into qval.  Size: a power
// of two >= 2 * nnz, so probes stay short.
__device__ __forceinline__ uint32_t dim_hash(uint32_t d, uint32_t mask) {
  return (d * 0x9E3779B1u) >> 7 & mask;
}

__device__ __forceinline__ void hash_build(uint32_t* hkey, int* hval, int hsize,
                                           const uint32_t* __restrict__ dims, int n) {
  for (int i = threadIdx.x; i < hsize; i += blockDim.x) hkey[i] = 0xFFFFFFFFu;
  __syncthreads();
  const uint32_t mask = (uint32_t)hsize - 1u;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t d = dims[i];
    uint32_t h = dim_hash(d, mask);
    for (;;) {
      const uint32_t prev = atomicCAS(&hkey[h], 0xFFFFFFFFu, d);
      if (prev == 0xFFFFFFFFu || prev == d) break;  // dims of a query are distinct
      h = (h + 1u) & mask;
    }
    hval[h] = i;
  }
  __syncthreads();
}

__device__ __forceinline__ int hash_find(const uint32_t* hkey, const int* hval, uint32_t mask,
                                         uint32_t d) {
  uint32_t h = dim_hash(d, mask);
  for (;;) {
    const uint32_t k = hkey[h];
    if (k == d) return hval[h];
    if (k == 0xFFFFFFFFu) return -1;
    h = (h + 1u) & mask;
  }
}

// warp_row_dot with the query dims looked up in the hash table; the row
// bounds [b, e) are given.  Column indices and values of a 32-entry piece are
// loaded together (one memory round trip per piece), the next piece's loads
// issued before this one's lookups.
// With `dmask` set (GPU-built indices: the residual is read from the raw row)
// only entries whose data-part bit is clear and whose |value| >= eps count.
__device__ double warp_row_dot_h(int64_t b, int64_t e, const uint32_t* __restrict__ indices,
                                 const float* __restrict__ data, const uint32_t* hkey,
                                 const int* hval, uint32_t mask, const double* __restrict__ qval,
                                 const uint32_t* __restrict__ dmask = nullptr, double eps = 0.0) {
  const int lane = threadIdx.x & 31;
  double sum = 0.0;
  int64_t i = b + lane;
  uint32_t ci = 0xFFFFFFFFu;
  float cv = 0.f;
  if (i < e) {
    ci = __ldg(indices + i);
    cv = __ldg(data + i);
  }
  for (int64_t base = b; base < e; base += 32) {
    const uint32_t col = ci;
    const float val = cv;
    const bool live = base + lane < e;
    i = base + 32 + lane;
    if (i < e) {  // next piece in flight
      ci = __ldg(indices + i);
      cv = __ldg(data + i);
    }
    double prod = 0.0;
    bool hit = false;
    bool keep = true;
    if (live && dmask) {
      const int64_t ei = base + lane;
      keep = !((__ldg(dmask + (ei >> 5)) >> (ei & 31)) & 1u) && fabs((double)val) >= eps;
    }
    if (live && keep) {
      const int j = hash_find(hkey, hval, mask, col);
      if (j >= 0) {
        prod = __dmul_rn((double)val, qval[j]);
        hit = true;
      }
    }
    unsigned ball = __ballot_sync(0xffffffffu, hit);
    while (ball) {  // matches in column order, sequential from +0.0
      const int src = __ffs(ball) - 1;
      const double v = __shfl_sync(0xffffffffu, prod, src);
      sum = __dadd_rn(sum, v);
      ball &= ball - 1;
    }
  }
  return sum;
}

__global__ void __launch_bounds__(kRrThreads) k_stage2(
    const Cand* __restrict__ cand1, int k1, int k2, int64_t d, const double* __restrict__ qw_all,
    const float* __restrict__ lo, const float* __restrict__ step,
    const uint8_t* __restrict__ codes, Cand* __restrict__ cand2, int P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* buf = reinterpret_cast<Cand*>(smem_raw);
  double* qw = reinterpret_cast<double*>(buf + P);
  double* slo = qw + d;     // decode affine in f64, shared by the candidates
  double* sstep = slo + d;
  const int64_t q = blockIdx.x;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
    qw[i] = qw_all[q * d + i];
    slo[i] = (double)lo[i];
    sstep[i] = (double)step[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int lane4 = lane & 3;
  const unsigned gmask = 0xFu << (lane & ~3);
  const int groups = blockDim.x / 4;
  const int g0 = threadIdx.x / 4;
  // every group iterates the same trip count so the group shuffles stay converged
  for (int base = 0; base < k1; base += groups) {
    const int c = base + g0;
    Cand e = c < k1 ? cand1[q * k1 + c] : worst_cand();
    if (c < k1 && e.slot != 0xFFFFFFFFu) {
      const uint8_t* row = codes + (int64_t)e.slot * d;
      auto elem = [&](int i) -> double {
        return __dadd_rn(slo[i], __dmul_rn(sstep[i], (double)row[i] + 0.5));
      };
      double dot;
      if ((d & 15) == 0) {
        // 16 codes per load (each group's 4 lanes read the same 16 bytes);
        // lane j's FMA chain still runs over elements j, j+4, ... in order
        const uint4* r4 = reinterpret_cast<const uint4*>(row);
        double L = 0.0;
        for (int i0 = 0; i0 < (int)d; i0 += 16) {
          const uint4 w = __ldg(r4 + (i0 >> 4));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i = i0 + 4 * t + lane4;
            const double code = (double)((ws[t] >> (8 * lane4)) & 0xFFu);
            L = fma(__dadd_rn(slo[i], __dmul_rn(sstep[i], code + 0.5)), qw[i], L);
          }
        }
        const int gb = lane & ~3;
        const double L0 = __shfl_sync(gmask, L, gb + 0), L1 = __shfl_sync(gmask, L, gb + 1);
        const double L2 = __shfl_sync(gmask, L, gb + 2), L3 = __shfl_sync(gmask, L, gb + 3);
        dot = (L0 + L2) + (L1 + L3);
      } else {
        dot = group4_dot_recipe(elem, qw, (int)d, lane4, gmask);
      }
      e.s = __dadd_rn(e.s, dot);  // scores1[cand1] + residual.dot  (pipeline.py:259-260)
    }
    if (c < k1 && lane4 == 0) buf[c] = e;
  }
  for (int i = k1 + threadIdx.x; i < P; i += blockDim.x) buf[i] = worst_cand();
  __syncthreads();
  bitonic_sort_block(buf, P);
  for (int i = threadIdx.x; i < k2; i += blockDim.x) cand2[q * k2 + i] = buf[i];
}

__global__ void k_copy_prefix(const Cand* __restrict__ in, int k1, int k2, int64_t nq,
                              Cand* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * k2) return;
  out[i] = in[(i / k2) * k1 + (i % k2)];
}

struct Stage3Args {
  const Cand* cand2;
  int k2, kh, exact, P, max_qnnz, hsize;
  const int64_t* qptr;
  const uint32_t* qdims;
  const float* qvals;
  const double* qd_all;
  int64_t d;
  double sparse_weight;
  const uint32_t* order;
  int64_t id_offset;
  // exact
  const float* ds_dense;
  const __half* ds_dense_h;
  const int64_t* ds_indptr;
  const uint32_t* ds_indices;
  const float* ds_data;
  // residual (res_raw: raw rows by original id, data-part bits in dmask)
  int res_raw;
  const uint32_t* dmask;
  double eps;
  int64_t res_nnz;
  const int64_t* res_indptr;
  const uint32_t* res_indices;
  const float* res_data;
  int64_t* out_ids;
  double* out_scores;
};

__global__ void __launch_bounds__(kRrThreads) k_stage3(Stage3Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* buf = reinterpret_cast<Cand*>(smem_raw);
  double* qd = reinterpret_cast<double*>(buf + a.P);
  double* qval = qd + a.d;
  uint32_t* qdims = reinterpret_cast<uint32_t*>(qval + a.max_qnnz);
  uint32_t* hkey = qdims + a.max_qnnz;
  int* hval = reinterpret_cast<int*>(hkey + a.hsize);
  const int64_t q = blockIdx.x;
  const int64_t qb = a.qptr[q];
  const int nqz = (int)(a.qptr[q + 1] - qb);
  for (int i = threadIdx.x; i < nqz; i += blockDim.x) {
    qdims[i] = a.qdims[qb + i];
    const double v = (double)a.qvals[qb + i];
    // exact: qvec = f64(v) * sparse_weight (pipeline.py:320); residual: f64(v) (pipeline.py:308)
    qval[i] = a.exact ? __dmul_rn(v, a.sparse_weight) : v;
  }
  if (a.exact)
    for (int64_t i = threadIdx.x; i < a.d; i += blockDim.x) qd[i] = a.qd_all[q * a.d + i];
  __syncthreads();
  hash_build(hkey, hval, a.hsize, qdims, nqz);
  const uint32_t hmask = (uint32_t)a.hsize - 1u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int g = lane >> 2, lane4 = lane & 3;
  const unsigned gmask = 0xFu << (lane & ~3);
  // a warp takes 8 candidates at a time: the 8 quarter-warp groups evaluate
  // their dense dots concurrently (the dgemv recipe needs 4 FMA chains), then
  // the warp walks the 8 sparse rows one by one
  for (int c0 = warp * 8; c0 < a.k2; c0 += nwarps * 8) {
    const int c = c0 + g;
    Cand e = c < a.k2 ? a.cand2[q * a.k2 + c] : worst_cand();
    const bool live = c < a.k2 && e.slot != 0xFFFFFFFFu;
    if (a.exact) {
      double dense = 0.0;
      if (a.d > 0) {  // every group runs the recipe (converged shuffles); dead ones on row 0
        const int64_t r = live ? (int64_t)e.tie : 0;
        if (a.ds_dense_h) {
          const __half* row = a.ds_dense_h + r * a.d;
          auto elem = [&](int i) -> double { return (double)__half2float(row[i]); };
          dense = group4_dot_recipe(elem, qd, (int)a.d, lane4, gmask);
        } else {
          const float* row = a.ds_dense + r * a.d;
          auto elem = [&](int i) -> double { return (double)__ldg(row + i); };
          dense = group4_dot_recipe(elem, qd, (int)a.d, lane4, gmask);
        }
      }
      if (live) e.s = dense;
    }
    if (c < a.k2 && lane4 == 0) buf[c] = e;
    __syncwarp();
    const int nc = min(8, a.k2 - c0);
    // sparse row bounds of the 8 candidates, loaded in parallel (lanes 0-7)
    const bool use_sp = nqz > 0 && (a.exact || a.res_nnz > 0);
    const bool raw = a.exact || a.res_raw;
    const int64_t* rp = raw ? a.ds_indptr : a.res_indptr;
    int64_t rb = 0, re = 0;
    if (use_sp && lane < nc) {
      const Cand el = buf[c0 + lane];
      if (el.slot != 0xFFFFFFFFu) {
        const int64_t row = raw ? (int64_t)el.tie : (int64_t)el.slot;
        rb = __ldg(rp + row);
        re = __ldg(rp + row + 1);
      }
    }
    for (int j = 0; j < nc; ++j) {
      Cand ej = buf[c0 + j];
      const int64_t b0 = __shfl_sync(0xffffffffu, rb, j), e0 = __shfl_sync(0xffffffffu, re, j);
      if (ej.slot == 0xFFFFFFFFu) continue;  // uniform across the warp
      double fin;
      if (a.exact) {
        fin = ej.s;  // dense part
        if (use_sp) {
          const double sp = warp_row_dot_h(b0, e0, a.ds_indices, a.ds_data, hkey, hval, hmask, qval);
          fin = __dadd_rn(fin, sp);
        }
      } else {
        double rd = 0.0;
        if (use_sp)
          rd = a.res_raw ? warp_row_dot_h(b0, e0, a.ds_indices, a.ds_data, hkey, hval, hmask, qval,
                                          a.dmask, a.eps)
                         : warp_row_dot_h(b0, e0, a.res_indices, a.res_data, hkey, hval, hmask, qval);
        fin = __dadd_rn(ej.s, __dmul_rn(rd, a.sparse_weight));
      }
      if (lane == 0) buf[c0 + j].s = fin;
    }
    __syncwarp();
  }
  for (int i = a.k2 + threadIdx.x; i < a.P; i += blockDim.x) buf[i] = worst_cand();
  __syncthreads();
  bitonic_sort_block(buf, a.P);
  for (int i = threadIdx.x; i < a.kh; i += blockDim.x) {
    const Cand e = buf[i];
    const bool ok = e.slot != 0xFFFFFFFFu;
    a.out_ids[q * a.kh + i] = ok ? (int64_t)a.order[e.slot] + a.id_offset : -1;
    a.out_scores[q * a.kh + i] = ok ? e.s : -INFINITY;
  }
}

// exact hybrid score of every point (original id order) for a query chunk
__global__ void __launch_bounds__(kRrThreads) k_exact_scores(
    int64_t n, int64_t d, const float* __restrict__ dense, const __half* __restrict__ dense_h,
    const int64_t* __restrict__ indptr,
    const uint32_t* __restrict__ indices, const float* __restrict__ data,
    const int64_t* __restrict__ qptr, const uint32_t* __restrict__ qdims_g,
    const float* __restrict__ qvals_g, const double* __restrict__ qd_all, double sparse_weight,
    int max_qnnz, Cand* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* qd = reinterpret_cast<double*>(smem_raw);
  double* qval = qd + d;
  uint32_t* qdims = reinterpret_cast<uint32_t*>(qval + max_qnnz);
  const int64_t q = blockIdx.y;
  const int64_t qb = qptr[q];
  const int nqz = (int)(qptr[q + 1] - qb);
  for (int i = threadIdx.x; i < nqz; i += blockDim.x) {
    qdims[i] = qdims_g[qb + i];
    qval[i] = __dmul_rn((double)qvals_g[qb + i], sparse_weight);
  }
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) qd[i] = qd_all[q * d + i];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  if (d > 0) s = dense_h ? dot_recipe(dense_h + i * d, qd, (int)d) : dot_recipe(dense + i * d, qd, (int)d);
  if (nqz > 0) {
    double sp = 0.0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      const int j = find_dim(qdims, nqz, indices[e]);
      if (j >= 0) sp = __dadd_rn(sp, __dmul_rn((double)data[e], qval[j]));
    }
    s = __dadd_rn(s, sp);
  }
  Cand c;
  c.s = s;
  c.tie = (uint32_t)i;
  c.slot = (uint32_t)i;
  out[q * n + i] = c;
}

__global__ void k_query_qd(const float* __restrict__ qdense, int64_t nq, int64_t d, double w,
                           double* __restrict__ qd) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq * d) qd[i] = __dmul_rn((double)qdense[i], w);
}

__global__ void k_cands_to_ids(const Cand* __restrict__ c, int64_t total, int64_t id_offset,
                               int64_t* __restrict__ ids, double* __restrict__ scores) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const bool ok = c[i].slot != 0xFFFFFFFFu;
  ids[i] = ok ? (int64_t)c[i].slot + id_offset : -1;
  scores[i] = ok ? c[i].s : -INFINITY;
}

}  // namespace

void launch_stage2(const DeviceIndex& ix, const Cand* cand1, int64_t nq, int k1, int k2,
                   const double* qw, Cand* cand2, cudaStream_t st) {
  if (nq <= 0) return;
  if (!(ix.d_dense > 0 && ix.has_sq)) {
    // no SQ residual: stage-2 scores equal stage-1 scores, cand1 is sorted
    const int T = 256;
    k_copy_prefix<<<(unsigned)ceil_div(nq * k2, T), T, 0, st>>>(cand1, k1, k2, nq, cand2);
    return;
  }
  const int P = next_pow2(k1);
  const size_t smem = sizeof(Cand) * P + 3 * sizeof(double) * ix.d_dense;
  cudaFuncSetAttribute(k_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_stage2<<<(unsigned)nq, kRrThreads, smem, st>>>(cand1, k1, k2, ix.d_dense, qw, ix.sq_lo,
                                                   ix.sq_step, ix.sq_codes, cand2, P);
}

void launch_stage3(const DeviceIndex& ix, const QueryView& q, const Cand* cand2, int64_t nq,
                     int k2, int kh, int exact, int max_qnnz, const double* qd, int64_t* out_ids,
                     double* out_scores, cudaStream_t st) {
  if (nq <= 0) return;
  Stage3Args a;
  a.cand2 = cand2;
  a.k2 = k2;
  a.kh = kh;
  a.exact = exact;
  a.P = next_pow2(k2);
  a.max_qnnz = max_qnnz < 1 ? 1 : max_qnnz;
  a.hsize = 64;
  while (a.hsize < 2 * a.max_qnnz) a.hsize *= 2;
  a.qptr = q.sp_indptr;
  a.qdims = q.sp_dims;
  a.qvals = q.sp_vals;
  a.qd_all = qd;
  a.d = ix.d_dense;
  a.sparse_weight = ix.sparse_weight;
  a.order = ix.order;
  a.id_offset = ix.id_offset;
  a.ds_dense = ix.ds_dense;
  a.ds_dense_h = ix.ds_dense_h;
  a.res_raw = ix.res_raw;
  a.dmask = ix.ds_dmask;
  a.eps = ix.res_eps;
  a.ds_indptr = ix.ds_indptr;
  a.ds_indices = ix.ds_indices;
  a.ds_data = ix.ds_data;
  a.res_nnz = ix.res_nnz;
  a.res_indptr = ix.res_indptr;
  a.res_indices = ix.res_indices;
  a.res_data = ix.res_data;
  a.out_ids = out_ids;
  a.out_scores = out_scores;
  auto smem_of = [&](int hs) {
    return sizeof(Cand) * a.P + sizeof(double) * (ix.d_dense + a.max_qnnz) +
           sizeof(uint32_t) * a.max_qnnz + (sizeof(uint32_t) + sizeof(int)) * hs;
  };
  while (smem_of(a.hsize) > 227 * 1024 && a.hsize / 2 > a.max_qnnz) a.hsize /= 2;  // fuller table
  const size_t smem = smem_of(a.hsize);
  cudaFuncSetAttribute(k_stage3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_stage3<<<(unsigned)nq, kRrThreads, smem, st>>>(a);
}

void launch_query_qd(const float* qdense, int64_t nq, int64_t d, double w, double* qd,
                     cudaStream_t st) {
  if (nq * d <= 0) return;
  k_query_qd<<<(unsigned)ceil_div(nq * d, 256), 256, 0, st>>>(qdense, nq, d, w, qd);
}

void launch_exact_scores(const DeviceIndex& ix, const QueryView& q, int max_qnnz,
                         const double* qd, Cand* out, cudaStream_t st) {
  if (q.nq <= 0 || ix.n <= 0) return;
  const int mq = max_qnnz < 1 ? 1 : max_qnnz;
  const size_t smem = sizeof(double) * (ix.d_dense + mq) + sizeof(uint32_t) * mq;
  cudaFuncSetAttribute(k_exact_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)ceil_div(ix.n, kRrThreads), (unsigned)q.nq);
  k_exact_scores<<<grid, kRrThreads, smem, st>>>(ix.n, ix.d_dense, ix.ds_dense, ix.ds_dense_h,
                                                 ix.ds_indptr,
                                                 ix.ds_indices, ix.ds_data, q.sp_indptr,
                                                 q.sp_dims, q.sp_vals, qd, ix.sparse_weight, mq,
                                                 out);
}

// ---------------------------------------------------------------------------
// ScalarQuantResidual.decode / .dot / sq_decode (dense.py:369-375, 393-394) as
// unit entry points.  decode: lo + step * (code + 0.5) in f64 (one rounding
// per operation, like numpy's broadcast).  dot: decode(rows) @ q — numpy's
// row-major matrix @ vector is the dgemv recipe (quarter-warp groups, the
// same arithmetic as k_stage2); a single-row product goes through numpy's
// ddot instead (not reproduced; within the north-star tolerance).
// ---------------------------------------------------------------------------
__global__ void k_sq_decode(const uint8_t* __restrict__ codes, int64_t d,
                            const float* __restrict__ lo, const float* __restrict__ step,
                            const int64_t* __restrict__ rows, int64_t m, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m * d) return;
  const int64_t r = i / d, c = i - r * d;
  const int64_t row = rows ? rows[r] : r;
  const double code = (double)codes[row * d + c];
  out[i] = __dadd_rn((double)lo[c], __dmul_rn((double)step[c], __dadd_rn(code, 0.5)));
}

__global__ void __launch_bounds__(kRrThreads) k_sq_dot(
    const uint8_t* __restrict__ codes, int64_t d, const float* __restrict__ lo,
    const float* __restrict__ step, const int64_t* __restrict__ rows, int64_t m,
    const double* __restrict__ q, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sq = reinterpret_cast<double*>(smem_raw);
  double* slo = sq + d;
  double* sstep = slo + d;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
    sq[i] = q[i];
    slo[i] = (double)lo[i];
    sstep[i] = (double)step[i];
  }
  __syncthreads();
  const int lane4 = threadIdx.x & 3;
  const unsigned gmask = 0xFu << ((threadIdx.x & 31) & ~3);
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 4);
  // uniform trip count per group: the group's shuffles stay converged
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 4) + threadIdx.x / 4; r < m; r += groups) {
    const uint8_t* row = codes + (rows ? rows[r] : r) * d;
    auto elem = [&](int i) -> double {
      return __dadd_rn(slo[i], __dmul_rn(sstep[i], (double)row[i] + 0.5));
    };
    const double dot = group4_dot_recipe(elem, sq, (int)d, lane4, gmask);
    if (lane4 == 0) out[r] = dot;
  }
}

void launch_cands_to_ids(const Cand* c, int64_t total, int64_t id_offset, int64_t* ids,
                         double* scores, cudaStream_t st) {
  if (total <= 0) return;
  k_cands_to_ids<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(c, total, id_offset, ids,
                                                                  scores);
}

void launch_sq_decode(const uint8_t* codes, int64_t d, const float* lo, const float* step,
                      const int64_t* rows, int64_t m, double* out, cudaStream_t st) {
  if (m * d <= 0) return;
  k_sq_decode<<<(unsigned)ceil_div(m * d, 256), 256, 0, st>>>(codes, d, lo, step, rows, m, out);
}

void launch_sq_dot(const uint8_t* codes, int64_t d, const float* lo, const float* step,
                   const int64_t* rows, int64_t m, const double* q, double* out, cudaStream_t st) {
  if (m <= 0) return;
  const size_t smem = 3 * sizeof(double) * (size_t)std::max<int64_t>(d, 1);
  cudaFuncSetAttribute(k_sq_dot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = std::min<int64_t>(ceil_div(m, kRrThreads / 4), 148 * 8);
  k_sq_dot<<<(unsigned)blocks, kRrThreads, smem, st>>>(codes, d, lo, step, rows, m, q, out);
}

}  // namespace hs
