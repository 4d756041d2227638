// fuse.cu — the threshold-filtered stage 1 (tensor-core path, large batches).
//
// Stage 1 keeps, per query, the exact top-k1 of
//     score(p) = acc(p) + ((bias_total + scale*total(p)) + offset)
// over all points (pipeline.py:192-203 then select_topk, pipeline.py:165-189).
// Materialising every u16 total costs 2 bytes per (point, query) written and
// read back; instead:
//   1. sample: the u16 totals of the first `m` points give t_k, their k1-th
//      largest total, and k_sample_tlim turns it into T[q], a lower bound on
//      the k1-th best stage-1 score (k1 real points score at least
//      dense(t_k) + a lower bound of the sparse part; see there).  Every true
//      top-k1 point scores >= T.  (HSB200_EXACT_SAMPLE=1: T = the exact
//      k1-th best of the sample, through the full stage-1 kernels — tighter,
//      slower.)
//   2. tlim[q] = the smallest u16 total whose dense-only score reaches T (the
//      f64 ops are monotone in the total);
//   3. the tensor-core pass in filter mode emits only (point, total) with
//      total >= tlim[q] — every point without a sparse part that can still
//      reach the top-k1;
//   4. k_fuse_cands scores the union of those and of the points the query's
//      postings touch (their accumulators summed in the reference's ascending
//      dim order), dropping dense candidates the postings touch (they are
//      scored with their sparse part), and
//   5. the variable-length selection keeps the exact top-k1.
// A query whose candidate list overflowed, or whose postings were not
// bucketed, is flagged and rerun through the unfiltered stage 1.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace hs {

namespace {

#ifndef HS_FUSE_THREADS
#define HS_FUSE_THREADS 256
#endif
constexpr int kFuseThreads = HS_FUSE_THREADS;
constexpr int kMaxSeg = 4 * kNumSMs + 2;  // list segments per query (tensor-core pass: one per CTA; streamed scan: a few per SM)

__device__ __forceinline__ double dense_score(double btot, double scl, double off, uint32_t t) {
  return __dadd_rn(__dadd_rn(btot, __dmul_rn(scl, (double)t)), off);
}

// smallest u16 total whose dense-only score reaches T (65536: none)
__device__ uint32_t tlim_of(double T, double b, double s, double o) {
  int lo = 0, hi = 65536;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (dense_score(b, s, o, (uint32_t)mid) >= T) hi = mid;
    else lo = mid + 1;
  }
  return (uint32_t)lo;
}

__global__ void k_tlim(const Cand* __restrict__ cand_s, int64_t nq, int k,
                       const double* __restrict__ btot, const double* __restrict__ scl,
                       const double* __restrict__ off, uint32_t* __restrict__ tlim,
                       double* __restrict__ Tout) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double T = cand_s[q * k + (k - 1)].s;  // -inf when the sample had < k points
  tlim[q] = tlim_of(T, btot[q], scl[q], off ? off[q] : 0.0);
  Tout[q] = T;
}

// Threshold from the sample's u16 totals alone (no sample stage 1): t_k = the
// k-th largest total among the first m points (two 8-bit radix passes with
// per-warp shared-memory histograms).  Those k points are real points whose
// stage-1 score is acc + dense >= dense(t_k) + lb, where lb <= every point's
// sparse accumulator: sum over the query's dims of min(0, q*wmin, q*wmax)
// (each posting product lies between q*wmin and q*wmax of the index's
// weights; a point gets at most one product per dim).  So
// T = dense(t_k) + lb is <= the k-th best stage-1 score over all points.  With
// lb == 0 (non-negative products: acc >= +0 exactly, and fl(acc + d) >= d)
// T = dense(t_k) exactly; otherwise it is lowered by a relative guard that
// covers the f64 rounding of the sums.
//
// The k points sit in the top ~k/m of the sample (0.05% at config 5), so a
// full pass can skip almost every value: a first selection over a strided
// sub-sample of ~64 K values gives L = its k-th largest total, a lower bound
// of t_k (the sub-sample is part of the sample); ONE full pass then builds a
// direct histogram of (total - L) for the totals >= L (a few percent, within
// a narrow range: 4096 bins, the last open-ended) and t_k is read off it.
// It runs at load speed instead of one shared-memory atomic per value.  When
// the sub-sample is too small, or t_k lands in the open bin, two 8-bit radix
// passes over the totals >= L decide.
constexpr int kTlThreads = 512;
constexpr int kTlWarps = kTlThreads / 32;
constexpr int kTlUnroll = 6;          // 16-byte groups in flight per thread

struct TlSel {
  uint32_t bin, rem;
};

// MODE 0: bin = v >> 8 for v >= lo;  MODE 1: bin = v & 255 for v >> 8 == hi8 and v >= lo.
// Groups g*gstride (g = 0, 1, ...) of 8 totals each; returns the highest bin where the
// count from the top reaches `rem`, and what is left to find inside it.
template <int MODE>
__device__ TlSel tl_pass(const uint16_t* __restrict__ t, int64_t m, int64_t gstride, uint32_t lo,
                         uint32_t hi8, uint32_t rem, uint32_t (*hist)[256], uint32_t* s_sum,
                         uint32_t* s_out) {
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kTlWarps * 256; i += kTlThreads) (&hist[0][0])[i] = 0u;
  __syncthreads();
  const int64_t ngroups = (m + 7) / 8;
  const int64_t nsel = (ngroups + gstride - 1) / gstride;  // groups visited
  for (int64_t j0 = tid; j0 < nsel; j0 += (int64_t)kTlThreads * kTlUnroll) {
    uint4 v4[kTlUnroll];
#pragma unroll
    for (int u = 0; u < kTlUnroll; ++u) {
      const int64_t j = j0 + (int64_t)u * kTlThreads;
      v4[u] = j < nsel ? __ldg(reinterpret_cast<const uint4*>(t + j * gstride * 8))
                       : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kTlUnroll; ++u) {
      const int64_t j = j0 + (int64_t)u * kTlThreads;
      if (j >= nsel) break;
      const int64_t p = j * gstride * 8;
      const uint32_t w[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
      // group reject: the high half of a word is >= lo iff the word is >= lo << 16,
      // the low half iff the word shifted up is (two compares per pair of totals)
      const uint32_t ll = lo << 16;
      bool any = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) any |= (w[i] >= ll) | ((w[i] << 16) >= ll);
      if (!any) continue;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint32_t v = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
        if (v < lo || p + h >= m) continue;
        if (MODE == 0) atomicAdd(&hist[warp][v >> 8], 1u);
        else if ((v >> 8) == hi8) atomicAdd(&hist[warp][v & 0xFFu], 1u);
      }
    }
  }
  __syncthreads();
  if (tid < 256) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kTlWarps; ++w) c += hist[w][tid];
    s_sum[tid] = c;
  }
  __syncthreads();
  if (tid == 0) {  // highest bin where the running count from the top reaches rem
    uint32_t run = 0;
    int b = 255;
    for (; b > 0; --b) {
      if (run + s_sum[b] >= rem) break;
      run += s_sum[b];
    }
    s_out[0] = (uint32_t)b;
    s_out[1] = rem - run;
  }
  __syncthreads();
  TlSel r;
  r.bin = s_out[0];
  r.rem = s_out[1];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kTlThreads, 2) k_sample_tlim(
    const uint16_t* __restrict__ tot_s, int64_t ld, int64_t m, int k, int64_t sub_groups,
    uint32_t direct_bins,
    const int64_t* __restrict__ qptr, const double* __restrict__ qv, double wmin, double wmax,
    const double* __restrict__ btot, const double* __restrict__ scl,
    const double* __restrict__ off, uint32_t* __restrict__ tlim, double* __restrict__ Tout) {
  __shared__ uint32_t hist[kTlWarps][256];
  __shared__ uint32_t s_sum[256];
  __shared__ uint32_t s_part[kTlThreads];
  __shared__ double s_lb[kTlWarps];
  __shared__ uint32_t s_out[2];
  static_assert(kTlWarps * 256 >= 4096 && kTlThreads * 8 == 4096, "direct histogram layout");
  const int64_t q = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint16_t* t = tot_s + q * ld;
  // sparse lower bound (query dims, any order: every term is <= 0)
  double lb = 0.0;
  if (qptr) {
    for (int64_t j = qptr[q] + tid; j < qptr[q + 1]; j += kTlThreads) {
      const double x = qv[j];
      lb += fmin(0.0, fmin(x * wmin, x * wmax));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lb += __shfl_xor_sync(0xffffffffu, lb, o);
  if (lane == 0) s_lb[warp] = lb;
  const bool none = m < k;  // fewer sample points than k: every total passes
  uint32_t tk = 0;
  if (!none) {
    // lower bound L of t_k from a strided sub-sample holding at least k totals
    uint32_t L = 0;
    const int64_t ngroups = (m + 7) / 8;
    const int64_t gstride = ngroups / sub_groups;
    if (gstride >= 4 && (ngroups / gstride) * 8 - 8 >= (int64_t)k) {
      // (every visited group but possibly the last is whole: >= k totals)
      const TlSel a0 = tl_pass<0>(t, m, gstride, 0u, 0u, (uint32_t)k, hist, s_sum, s_out);
      const TlSel a1 = tl_pass<1>(t, m, gstride, 0u, a0.bin, a0.rem, hist, s_sum, s_out);
      L = (a0.bin << 8) | a1.bin;
    }
    bool found = false;
    if (L > 0u) {
      // one full pass: the totals >= L span a narrow range, so a direct
      // histogram of (total - L) over 4096 bins (the last one open-ended)
      // holds the k-th largest exactly unless it falls into the open bin
      uint32_t* h12 = &hist[0][0];  // kTlWarps * 256 >= 4096 words
      for (int i = tid; i < 4096; i += kTlThreads) h12[i] = 0u;
      __syncthreads();
      const int64_t ngroups = (m + 7) / 8;
      const uint32_t ll = L << 16;
      for (int64_t j0 = tid; j0 < ngroups; j0 += (int64_t)kTlThreads * kTlUnroll) {
        uint4 v4[kTlUnroll];
#pragma unroll
        for (int u = 0; u < kTlUnroll; ++u) {
          const int64_t j = j0 + (int64_t)u * kTlThreads;
          v4[u] = j < ngroups ? __ldg(reinterpret_cast<const uint4*>(t + j * 8))
                              : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < kTlUnroll; ++u) {
          const int64_t j = j0 + (int64_t)u * kTlThreads;
          if (j >= ngroups) break;
          const uint32_t w[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
          bool any = false;
#pragma unroll
          for (int i = 0; i < 4; ++i) any |= (w[i] >= ll) | ((w[i] << 16) >= ll);
          if (!any) continue;
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const uint32_t v = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
            if (v < L || j * 8 + h >= m) continue;
            atomicAdd(&h12[min(v - L, direct_bins - 1u)], 1u);
          }
        }
      }
      __syncthreads();
      {  // thread i sums bins [8i, 8i + 8); thread 0 walks the 512 partial sums from the top
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) c += h12[8 * tid + i];
        s_part[tid] = c;
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t run = 0;
        int g = kTlThreads - 1;
        for (; g > 0; --g) {
          if (run + s_part[g] >= (uint32_t)k) break;
          run += s_part[g];
        }
        int b = 8 * g + 7;
        for (; b > 8 * g; --b) {
          if (run + h12[b] >= (uint32_t)k) break;
          run += h12[b];
        }
        s_out[0] = (uint32_t)b;
      }
      __syncthreads();
      const uint32_t b = s_out[0];
      __syncthreads();
      if (b < direct_bins - 1u) {
        tk = L + b;
        found = true;
      }
    }
    if (!found) {
      const TlSel b0 = tl_pass<0>(t, m, 1, L, 0u, (uint32_t)k, hist, s_sum, s_out);
      const TlSel b1 = tl_pass<1>(t, m, 1, L, b0.bin, b0.rem, hist, s_sum, s_out);
      tk = (b0.bin << 8) | b1.bin;
    }
  }
  if (tid == 0) {
    double l = 0.0;
    for (int w = 0; w < kTlWarps; ++w) l += s_lb[w];
    const double b = btot[q], s = scl[q], o = off ? off[q] : 0.0;
    double T = -INFINITY;
    if (!none) {
      const double dk = dense_score(b, s, o, tk);
      T = l == 0.0 ? dk : (dk + l * (1.0 + 1e-6)) - 1e-9 * fabs(dk);
    }
    tlim[q] = tlim_of(T, b, s, o);
    Tout[q] = T;
  }
}

struct FuseArgs {
  int64_t n;
  int Kp, npairs;
  int64_t prow;                 // bytes per pcodes row (multiple of 16)
  const uint8_t* pcodes;        // [n][prow]
  const uint8_t* luts;          // [nq][Kp][16]
  const double* btot;
  const double* scl;
  const double* off;
  const uint32_t* order;
  const uint2* list;            // [nq][nseg][cap]
  const uint32_t* cnt;          // [nq][nseg]
  int64_t cap;
  int nseg;
  // buckets (sparse)
  const int* bmode;
  const uint32_t* boff;
  const uint32_t* bslots;
  const double* bvals;
  int64_t capq;
  int nchunks;
  uint32_t* bitmap;             // [nq][words] all zero on entry and exit
  int64_t words;
  Cand* out;                    // [nq][M]
  int64_t M;
  uint32_t* out_cnt;            // [nq]
  int* fallback;                // [nq]
  const double* T;              // [nq] no top-k1 point scores below
  int exp;                      // dev timing knob (HSB200_FUSE_EXP): 1 skip touched, 2 skip dense
};

template <bool SP>
__global__ void __launch_bounds__(kFuseThreads) k_fuse_cands(FuseArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint8_t* lut = smem_raw;  // [Kp][16]
  __shared__ uint32_t s_cnt;
  __shared__ uint32_t s_pre[kMaxSeg + 1];  // prefix of the segment counts
  __shared__ int s_over;
  const int64_t q = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) s_over = 0;
  __syncthreads();
  for (int c = tid; c < a.nseg; c += blockDim.x)
    if (a.cnt[q * a.nseg + c] > (uint32_t)a.cap) s_over = 1;
  if (tid == 0) {
    uint32_t run = 0;
    for (int c = 0; c < a.nseg; ++c) {
      s_pre[c] = run;
      run += min(a.cnt[q * a.nseg + c], (uint32_t)a.cap);
    }
    s_pre[a.nseg] = run;
  }
  __syncthreads();
  const uint32_t nd = s_pre[a.nseg];
  const int mode = SP ? a.bmode[q] : 2;
  if (s_over || mode == 0) {  // overflow / streamed postings: unfiltered rerun
    if (tid == 0) {
      a.fallback[q] = 1;
      a.out_cnt[q] = 0;
    }
    return;
  }
  if (tid == 0) {
    a.fallback[q] = 0;
    s_cnt = 0;
  }
  const double b = a.btot[q], s = a.scl[q], o = a.off ? a.off[q] : 0.0;
  const double T = a.T[q];  // no top-k1 point scores below
  Cand* out = a.out + q * a.M;
  uint32_t* bm = SP ? a.bitmap + q * a.words : nullptr;
  const uint32_t* qb = SP ? a.boff + q * (int64_t)(a.nchunks + 1) : nullptr;
  const uint32_t* qs = SP ? a.bslots + q * a.capq : nullptr;
  const double* qv = SP ? a.bvals + q * a.capq : nullptr;
  const uint32_t E = (SP && mode == 1) ? qb[a.nchunks] : 0u;
  if (SP) {
    const uint4* src = reinterpret_cast<const uint4*>(a.luts + q * (int64_t)a.Kp * 16);
    for (int i = tid; i < a.Kp; i += blockDim.x) reinterpret_cast<uint4*>(lut)[i] = src[i];
  }
  __syncthreads();

  if (SP && E > 0 && !(a.exp & 1)) {
    // touched points: buckets hold one entry per point (k_bucket_aggregate:
    // its products summed in the reference's ascending dim order), then
    // empty entries
    // four entries per thread per round: their code-row loads overlap
    constexpr int U = 4;
    for (uint32_t eb = 0; eb < E; eb += U * blockDim.x) {
      uint32_t sl[U], t[U];
      double acc[U];
      const uint32_t* row[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = eb + u * blockDim.x + tid;
        sl[u] = e < E ? qs[e] : 0xFFFFFFFFu;
        acc[u] = e < E ? qv[e] : 0.0;
        t[u] = 0;
        row[u] = reinterpret_cast<const uint32_t*>(
            a.pcodes + (int64_t)(sl[u] == 0xFFFFFFFFu ? 0u : sl[u]) * a.prow);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (sl[u] != 0xFFFFFFFFu) atomicOr(bm + (sl[u] >> 5), 1u << (sl[u] & 31));
      // the points' LUT16 totals from their codes (exact integer sums); rows
      // are read 16 bytes (32 subspaces) at a time
      for (int w = 0; w * 16 < a.npairs; ++w) {
        uint4 v4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v4[u] = __ldg(reinterpret_cast<const uint4*>(row[u]) + w);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int pair = w * 16 + h * 4 + bb;
            if (pair < a.npairs) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const uint32_t word = h == 0 ? v4[u].x : h == 1 ? v4[u].y : h == 2 ? v4[u].z : v4[u].w;
                const uint32_t byte = (word >> (8 * bb)) & 0xFFu;
                t[u] += lut[(2 * pair) * 16 + (byte & 15u)];
                t[u] += lut[(2 * pair + 1) * 16 + (byte >> 4)];  // padding row of odd K is zero
              }
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (sl[u] == 0xFFFFFFFFu) continue;
        Cand c;
        c.s = __dadd_rn(acc[u], dense_score(b, s, o, t[u]));
        if (!(c.s >= T)) continue;  // below the sample threshold (still marked touched)
        c.tie = __ldg(a.order + sl[u]);
        c.slot = sl[u];
        out[atomicAdd(&s_cnt, 1u)] = c;
      }
    }
  }
  __syncthreads();
  // dense candidates without a sparse part
  const uint2* lst = a.list + q * a.nseg * a.cap;
  for (uint32_t i = tid; i < ((a.exp & 2) ? 0u : nd); i += blockDim.x) {
    int lo = 0, hi = a.nseg;  // segment of flat index i: largest c with s_pre[c] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pre[mid] <= i) lo = mid;
      else hi = mid;
    }
    const uint2 pt = lst[(int64_t)lo * a.cap + (i - s_pre[lo])];
    if (SP && E > 0 && (bm[pt.x >> 5] >> (pt.x & 31) & 1u)) continue;
    Cand c;
    c.s = __dadd_rn(0.0, dense_score(b, s, o, pt.y));
    c.tie = __ldg(a.order + pt.x);
    c.slot = pt.x;
    out[atomicAdd(&s_cnt, 1u)] = c;
  }
  __syncthreads();
  if (SP && E > 0)
    for (uint32_t e = tid; e < E; e += blockDim.x) {
      const uint32_t sl = qs[e];
      if (sl != 0xFFFFFFFFu) bm[sl >> 5] = 0u;
    }
  if (tid == 0) a.out_cnt[q] = s_cnt;
}

// pair-major packed codes -> point-major rows of `prow` bytes
__global__ void k_to_pcodes(const uint8_t* __restrict__ packed, int64_t n, int npairs,
                            int64_t prow, uint8_t* __restrict__ pc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  for (int j = 0; j < prow; ++j) pc[p * prow + j] = j < npairs ? packed[(int64_t)j * n + p] : 0;
}

}  // namespace

// rows padded to 16 bytes: one 16-byte load per 32 subspaces
int64_t pcodes_row(int npairs) { return ((int64_t)npairs + 15) / 16 * 16; }

void launch_to_pcodes(const uint8_t* packed, int64_t n, int npairs, uint8_t* pc, cudaStream_t st) {
  if (n <= 0) return;
  k_to_pcodes<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(packed, n, npairs, pcodes_row(npairs), pc);
}

void launch_tlim(const Cand* cand_s, int64_t nq, int k, const double* btot, const double* scl,
                 const double* off, uint32_t* tlim, double* T, cudaStream_t st) {
  if (nq <= 0) return;
  k_tlim<<<(unsigned)ceil_div(nq, 128), 128, 0, st>>>(cand_s, nq, k, btot, scl, off, tlim, T);
}

void launch_sample_tlim(const uint16_t* tot_s, int64_t ld, int64_t m, int64_t nq, int k,
                        const int64_t* qptr, const double* qv, double wmin, double wmax,
                        const double* btot, const double* scl, const double* off,
                        uint32_t* tlim, double* T, cudaStream_t st) {
  if (nq <= 0) return;
  // sub-sample of the first selection, in 8-value groups (HSB200_TLIM_SUBGROUPS: test knob that
  // lets small samples take the two-level path)
  const char* e = std::getenv("HSB200_TLIM_SUBGROUPS");
  const int64_t sub_groups = e ? std::max<int64_t>(1, std::atoll(e)) : 8192;
  // bins of the direct histogram of the single full pass (the last one open-ended);
  // HSB200_TLIM_DIRECT: test knob that makes the open bin, and the two-pass fallback, common
  const char* e2 = std::getenv("HSB200_TLIM_DIRECT");
  const uint32_t direct_bins =
      e2 ? (uint32_t)std::min<int64_t>(4096, std::max<int64_t>(2, std::atoll(e2))) : 4096u;
  k_sample_tlim<<<(unsigned)nq, kTlThreads, 0, st>>>(tot_s, ld, m, k, sub_groups, direct_bins, qptr,
                                                     qv, wmin, wmax, btot, scl, off, tlim, T);
}

int launch_fuse_cands(const DeviceIndex& ix, int64_t nq, const uint8_t* luts, const double* btot,
                      const double* scl, const double* off, const uint2* list,
                      const uint32_t* cnt, int64_t cap, int nseg, const SparseBuckets* sb,
                      uint32_t* bitmap, Cand* out, int64_t M, uint32_t* out_cnt, int* fallback,
                      const double* T, cudaStream_t st) {
  if (nq <= 0) return HS_OK;
  FuseArgs a;
  a.T = T;
  a.exp = std::getenv("HSB200_FUSE_EXP") ? std::atoi(std::getenv("HSB200_FUSE_EXP")) : 0;
  a.n = ix.n;
  a.Kp = ix.Kp;
  a.npairs = ix.npairs;
  a.prow = pcodes_row(ix.npairs);
  a.pcodes = ix.pcodes;
  a.luts = luts;
  a.btot = btot;
  a.scl = scl;
  a.off = off;
  a.order = ix.order;
  a.list = list;
  a.cnt = cnt;
  a.cap = cap;
  a.nseg = nseg;
  if (nseg > kMaxSeg) HS_FAIL(HS_EINVAL, "too many list segments");
  a.bmode = sb ? sb->mode : nullptr;
  a.boff = sb ? sb->boff : nullptr;
  a.bslots = sb ? sb->slots : nullptr;
  a.bvals = sb ? sb->vals : nullptr;
  a.capq = sb ? sb->capq : 0;
  a.nchunks = sb ? sb->nchunks : 0;
  a.bitmap = bitmap;
  a.words = ceil_div(ix.n, 32);
  a.out = out;
  a.M = M;
  a.out_cnt = out_cnt;
  a.fallback = fallback;
  const size_t smem = (size_t)ix.Kp * 16;
  if (sb) {
    if (!ix.pcodes) HS_FAIL(HS_EUNSUPPORTED, "filtered stage 1 needs point-major codes");
    k_fuse_cands<true><<<(unsigned)nq, kFuseThreads, smem, st>>>(a);
  } else {
    k_fuse_cands<false><<<(unsigned)nq, kFuseThreads, smem, st>>>(a);
  }
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace hs
