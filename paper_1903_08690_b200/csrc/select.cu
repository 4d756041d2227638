// select.cu — K4 top-k selection and K7 shard merge.
//
// Exact top-k by (score desc, tie id asc), the ordering of select_topk
// (reference pipeline.py:165-189).  Candidates are 16-byte {score, tie, slot}
// entries.  One CTA per query sorts up to kCap entries in shared memory with
// a bitonic network; longer inputs are streamed through the same buffer
// (keep the best k, refill, re-sort).  Inputs with k > kCap/2 fall back to a
// global-memory bitonic sort (only reachable from exhaustive test settings).
#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kSelThreads = 512;
constexpr int kCap = 8192;  // 128 KB of candidates in shared memory

__global__ void __launch_bounds__(kSelThreads) k_select_smem(const Cand* __restrict__ in,
                                                             int64_t m_row, int k,
                                                             Cand* __restrict__ out,
                                                             const uint32_t* __restrict__ counts,
                                                             const int* __restrict__ qmask) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* buf = reinterpret_cast<Cand*>(smem_raw);
  const int64_t q = blockIdx.x;
  if (qmask && qmask[q] == 0) return;
  const Cand* src = in + q * m_row;
  const int64_t m = counts ? min((int64_t)counts[q], m_row) : m_row;
  int have = 0;
  int64_t pos = 0;
  do {
    const int64_t take = min((int64_t)(kCap - have), m - pos);
    const int tot = have + (int)take;
    int P = 1;
    while (P < tot) P <<= 1;
    for (int i = threadIdx.x; i < P - have; i += blockDim.x)
      buf[have + i] = (i < take) ? src[pos + i] : worst_cand();
    __syncthreads();
    bitonic_sort_block(buf, P);
    pos += take;
    have = tot < k ? tot : k;
  } while (pos < m);
  if (m == 0) have = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) out[q * k + i] = i < have ? buf[i] : worst_cand();
}

// Exact top-k of a variable-length row by radix select: 8-bit digits of the
// order-preserving score key from the top (early exit once the boundary bin
// is taken whole), then, for exact score ties at the boundary, digits of the
// tie id from the bottom; the k selected entries are gathered and sorted.
// Reads the row once per digit (typically 2-3), no full sort of the row.
constexpr int kRsThreads = 512;

__global__ void __launch_bounds__(kRsThreads) k_select_radix(const Cand* __restrict__ in,
                                                             int64_t m_row, int k,
                                                             Cand* __restrict__ out,
                                                             const uint32_t* __restrict__ counts,
                                                             const int* __restrict__ qmask) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* buf = reinterpret_cast<Cand*>(smem_raw);  // [P] selected entries
  __shared__ unsigned hist[256];
  __shared__ int ctl[16];
  __shared__ unsigned long long red[2 * (kRsThreads / 32)];
  const int64_t q = blockIdx.x;
  if (qmask && qmask[q] == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const Cand* src = in + q * m_row;
  const int64_t m = counts ? min((int64_t)counts[q], m_row) : m_row;
  int P = 1;
  while (P < k) P <<= 1;
  unsigned long long prefix = 0, pmask = 0;
  bool whole = true;
  uint32_t tie_lim = 0xFFFFFFFFu;
  if (m > k) {
    int need = k;
    whole = false;
    // The keys of one query's candidates share their leading bytes (sign,
    // exponent, often the top of the mantissa): a digit pass over such a byte
    // puts every candidate into one bin — m atomics on one shared-memory word
    // — and selects nothing.  One min/max reduction finds the first byte where
    // the keys differ; the passes start there.
    int shift0 = 56;
    {
      unsigned long long kmin = ~0ull, kmax = 0ull;
      for (int64_t i = tid; i < m; i += blockDim.x) {
        const unsigned long long key = score_key(src[i].s);
        kmin = key < kmin ? key : kmin;
        kmax = key > kmax ? key : kmax;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
      }
      if ((tid & 31) == 0) {
        red[2 * warp] = kmin;
        red[2 * warp + 1] = kmax;
      }
      __syncthreads();
      kmin = red[0];
      kmax = red[1];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        kmin = red[2 * w] < kmin ? red[2 * w] : kmin;
        kmax = red[2 * w + 1] > kmax ? red[2 * w + 1] : kmax;
      }
      __syncthreads();
      const unsigned long long diff = kmin ^ kmax;
      if (diff == 0ull) {  // every key equal: only the tie ids select
        prefix = kmax;
        pmask = ~0ull;
        shift0 = -8;
      } else {
        shift0 = ((63 - __clzll((long long)diff)) >> 3) << 3;  // first differing byte
        if (shift0 < 56) {
          pmask = ~0ull << (shift0 + 8);
          prefix = kmax & pmask;
        }
      }
    }
    for (int shift = shift0; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int64_t i = tid; i < m; i += blockDim.x) {
        const unsigned long long key = score_key(src[i].s);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
      }
      __syncthreads();
      if (warp == 0) find_bin(hist, need, true, ctl);
      __syncthreads();
      prefix |= (unsigned long long)ctl[0] << shift;
      pmask |= 0xFFull << shift;
      need = ctl[1];
      whole = ctl[2] == need;
      __syncthreads();
      if (whole) break;
    }
    if (!whole) {  // the `need` smallest tie ids among key == prefix
      uint32_t tpre = 0, tmask = 0;
      for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t i = tid; i < m; i += blockDim.x) {
          const Cand e = src[i];
          if (score_key(e.s) == prefix && (e.tie & tmask) == tpre)
            atomicAdd(&hist[(e.tie >> shift) & 255], 1u);
        }
        __syncthreads();
        if (warp == 0) find_bin(hist, need, false, ctl);
        __syncthreads();
        tpre |= (uint32_t)ctl[0] << shift;
        tmask |= 0xFFu << shift;
        need = ctl[1];
        __syncthreads();
      }
      tie_lim = tpre;
    }
  }
  if (tid == 0) ctl[8] = 0;
  __syncthreads();
  for (int64_t i = tid; i < m; i += blockDim.x) {
    const Cand e = src[i];
    bool keep = true;
    if (m > k) {
      const unsigned long long key = score_key(e.s) & pmask;
      keep = key > prefix || (key == prefix && (whole || e.tie <= tie_lim));
    }
    if (keep) buf[atomicAdd(&ctl[8], 1)] = e;
  }
  __syncthreads();
  const int kept = ctl[8];
  for (int i = kept + tid; i < P; i += blockDim.x) buf[i] = worst_cand();
  __syncthreads();
  bitonic_sort_block(buf, P);
  for (int i = tid; i < k; i += blockDim.x) out[q * k + i] = i < kept ? buf[i] : worst_cand();
}

__global__ void k_pad_copy(const Cand* __restrict__ in, int64_t m, int64_t P, int64_t nq,
                           Cand* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * P) return;
  const int64_t q = i / P, j = i % P;
  out[i] = j < m ? in[q * m + j] : worst_cand();
}

__global__ void k_bitonic_step(Cand* a, int64_t P, int64_t nq, int64_t kk, int64_t jj) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t half = P >> 1;
  if (t >= nq * half) return;
  const int64_t q = t / half, i = t % half;
  const int64_t lo = ((i & ~(jj - 1)) << 1) | (i & (jj - 1));
  const int64_t hi = lo + jj;
  Cand* s = a + q * P;
  const bool up = (lo & kk) == 0;
  Cand x = s[lo], y = s[hi];
  if (up ? better(y, x) : better(x, y)) {
    s[lo] = y;
    s[hi] = x;
  }
}

__global__ void k_take_prefix(const Cand* __restrict__ a, int64_t P, int64_t nq, int64_t k,
                              Cand* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * k) return;
  out[i] = a[(i / k) * P + (i % k)];
}

__global__ void k_scores_to_cands(const double* __restrict__ s, const int64_t* __restrict__ tie,
                                  int64_t nq, int64_t n, Cand* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * n) return;
  const int64_t j = i % n;
  Cand c;
  c.s = s[i];
  c.tie = tie ? (uint32_t)tie[j] : (uint32_t)j;
  c.slot = (uint32_t)j;
  out[i] = c;
}

__global__ void k_cands_to_positions(const Cand* __restrict__ c, int64_t total,
                                     int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) out[i] = (int64_t)c[i].slot;
}

// K7: per query, best h of the G*kh gathered (id, score) pairs by
// (score desc, id asc).  Shards own disjoint id ranges, so ids are unique.
__global__ void __launch_bounds__(kSelThreads) k_shard_merge(
    const int64_t* __restrict__ ids, const double* __restrict__ scores, int64_t G, int64_t nq,
    int64_t kh, int h, int64_t* __restrict__ out_ids, double* __restrict__ out_scores) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* buf = reinterpret_cast<Cand*>(smem_raw);
  const int64_t q = blockIdx.x;
  const int64_t m = G * kh;
  int P = 1;
  while (P < m) P <<= 1;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
    Cand c = worst_cand();
    if (i < m) {
      const int64_t g = i / kh, j = i % kh;
      const int64_t src = (g * nq + q) * kh + j;
      const int64_t id = ids[src];
      if (id >= 0) {
        c.s = scores[src];
        c.tie = (uint32_t)id;
        c.slot = (uint32_t)i;
      }
    }
    buf[i] = c;
  }
  __syncthreads();
  bitonic_sort_block(buf, P);
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const Cand c = buf[i];
    const bool ok = c.slot != 0xFFFFFFFFu;
    int64_t id = -1;
    if (ok) {
      const int64_t g = c.slot / kh, j = c.slot % kh;
      id = ids[(g * nq + q) * kh + j];
    }
    out_ids[q * h + i] = id;
    out_scores[q * h + i] = ok ? c.s : -INFINITY;
  }
}

}  // namespace

int launch_select_topk(const Cand* in, int64_t nq, int64_t m, int64_t k, Cand* out,
                       cudaStream_t st, const uint32_t* counts, const int* qmask) {
  if (nq <= 0 || k <= 0) return HS_OK;
  // radix select (O(m) per digit) for every k <= 4096; the streamed bitonic
  // k_select_smem re-sorts 8192 entries per refill (1.2 ms for the 40K
  // per-tile candidates of one 10M-point query) and is kept for reference
  if (counts || qmask || k <= kCap / 2) {
    if (k > kCap / 2) HS_FAIL(HS_EUNSUPPORTED, "variable-length selection needs k <= 4096");
    int P = 1;
    while (P < k) P <<= 1;
    const size_t smem = sizeof(Cand) * P;
    HS_CUDA(cudaFuncSetAttribute(k_select_radix, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_select_radix<<<(unsigned)nq, kRsThreads, smem, st>>>(in, m, (int)k, out, counts, qmask);
    HS_CUDA(cudaGetLastError());
    return HS_OK;
  }
  if (k <= kCap / 2) {
    const size_t smem = sizeof(Cand) * kCap;
    HS_CUDA(cudaFuncSetAttribute(k_select_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_select_smem<<<(unsigned)nq, kSelThreads, smem, st>>>(in, m, (int)k, out, counts, qmask);
    HS_CUDA(cudaGetLastError());
    return HS_OK;
  }
  // global bitonic fallback
  const int64_t P = next_pow2(m);
  Cand* tmp = nullptr;
  HS_CUDA(cudaMallocAsync(&tmp, sizeof(Cand) * nq * P, st));
  const int T = 256;
  k_pad_copy<<<(unsigned)ceil_div(nq * P, T), T, 0, st>>>(in, m, P, nq, tmp);
  for (int64_t kk = 2; kk <= P; kk <<= 1)
    for (int64_t jj = kk >> 1; jj > 0; jj >>= 1)
      k_bitonic_step<<<(unsigned)ceil_div(nq * (P >> 1), T), T, 0, st>>>(tmp, P, nq, kk, jj);
  k_take_prefix<<<(unsigned)ceil_div(nq * k, T), T, 0, st>>>(tmp, P, nq, k, out);
  HS_CUDA(cudaFreeAsync(tmp, st));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

void launch_scores_to_cands(const double* scores, const int64_t* tie_ids, int64_t nq, int64_t n,
                            Cand* out, cudaStream_t st) {
  if (nq * n <= 0) return;
  const int T = 256;
  k_scores_to_cands<<<(unsigned)ceil_div(nq * n, T), T, 0, st>>>(scores, tie_ids, nq, n, out);
}

void launch_cands_to_positions(const Cand* c, int64_t nq, int64_t k, int64_t* out,
                               cudaStream_t st) {
  if (nq * k <= 0) return;
  const int T = 256;
  k_cands_to_positions<<<(unsigned)ceil_div(nq * k, T), T, 0, st>>>(c, nq * k, out);
}

void launch_shard_merge(const int64_t* ids, const double* scores, int64_t G, int64_t nq,
                        int64_t kh, int h, int64_t* out_ids, double* out_scores,
                        cudaStream_t st) {
  if (nq <= 0) return;
  const int64_t P = next_pow2(G * kh);
  const size_t smem = sizeof(Cand) * P;
  cudaFuncSetAttribute(k_shard_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_shard_merge<<<(unsigned)nq, kSelThreads, smem, st>>>(ids, scores, G, nq, kh, h, out_ids,
                                                          out_scores);
}

}  // namespace hs
