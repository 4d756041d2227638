// devbuild.cu — the index build on the GPU, sparse
// half, plus the seeded on-device generator of the BASELINE data laws.
//
// Config 5 (10^8 points, 5*10^9 nonzeros over 10^9 dims, fp16 dense) fits
// neither the host nor the reference's Python build, so the dataset is
// generated where it is searched and the index is built in place.  The build
// restates the reference's integer products exactly:
//
//   _top_t_thresholds   sparse.py:66-80   per head dim (count > t) the t-th
//                       largest |v|: a 4-pass, 8-bit radix select over the
//                       |v| bit pattern with one 256-bin histogram per head
//                       dim (np.partition(col, nnz-t)[nnz-t]).
//   prune_split         sparse.py:83-103  data iff |v| >= eta[dim]; residual iff
//                       not data and |v| >= residual_min; kept as one flag bit
//                       per raw entry (the residual is read from the raw row).
//   cache_sort          sparse.py:106-163 (+ _refine_equal_runs): points sorted
//                       by their data-part activity over the dims ranked
//                       (nnz desc, dim asc), descending lexicographically,
//                       stably.  Equivalent order: each point's ascending rank
//                       list with a +inf terminator, compared ascending
//                       (a proper prefix sorts after its extensions; equal
//                       lists keep id order).  Built as an LSD-free iterative
//                       refinement: a stable radix sort on the first rank,
//                       then, depth by depth, a stable sort of the points
//                       still tied on (segment start, next rank).
//   build_inverted      sparse.py:219-235 postings (dim asc, layout slot asc):
//                       one radix sort of (dim << 32 | slot) keys.
//
// Generator: per row Poisson(mean) nonzeros with DISTINCT
// Zipf(s) ranks (inverse CDF: a table of the first 4096 ranks, the continuous
// tail integral beyond), mapped through the seeded Feistel bijection of
// [0, d_sparse) that the host generator (hostbuild.cpp) also uses, |N(0,1)| or
// lognormal(0,1) values, N(0,1) dense part, the row L2-normalised over the
// concatenation in f64, stored f32 (dense optionally rounded to fp16 after
// normalisation).  Every draw is a counter-based hash of (seed, global row,
// stream, index), so any id range [row0, row0 + n) generates the same rows
// whatever the sharding.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "kernels.cuh"

namespace hs {

int builder_tmp(Builder& b, size_t bytes) {
  if (bytes <= b.tmp_bytes) return HS_OK;
  if (b.tmp) {
    HS_CUDA(cudaStreamSynchronize(b.st));
    cudaFree(b.tmp);
    b.tmp = nullptr;
    b.tmp_bytes = 0;
  }
  HS_CUDA(cudaMalloc(&b.tmp, bytes));
  b.tmp_bytes = bytes;
  return HS_OK;
}

void builder_phase(Builder& b, const char* name, double sec) {
  b.tnames.push_back(name);
  b.tsec.push_back(sec);
}

void builder_free(Builder* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  if (b->st) cudaStreamSynchronize(b->st);
  void* ptrs[] = {b->indptr, b->indices, b->data, b->dense, b->dense_h, b->dmask, b->order,
                  b->post_dims, b->post_ptr, b->post, b->head_dims, b->head_thr, b->packed,
                  b->pcodes, b->sq, b->tmp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (b->st) cudaStreamDestroy(b->st);
}

namespace {

using Clock = std::chrono::steady_clock;
double secs_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

template <typename T>
int balloc(Builder& b, T** p, size_t count) {
  *p = nullptr;
  HS_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(count, 1)));
  return HS_OK;
}

// ---------------------------------------------------------------------------
// counter-based RNG and the seeded bijection
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t sm_mix(uint64_t z) {  // splitmix64 output
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// hostbuild.cpp mix64 (golden-ratio increment, then the finaliser)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  return sm_mix(z + 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ uint64_t row_key(uint64_t seed, uint64_t row, uint64_t stream) {
  return sm_mix(sm_mix(seed * 0x9E3779B97F4A7C15ULL + stream + 1) ^ ((row + 1) * 0xD1B54A32D192ED03ULL));
}
__device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t i) {
  return sm_mix(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ double unif(uint64_t z) {  // (0, 1)
  return ((double)(z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double normal_at(uint64_t key, uint64_t j) {
  const double u1 = unif(draw(key, 2 * j)), u2 = unif(draw(key, 2 * j + 1));
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

struct Feistel {  // hostbuild.cpp Feistel: 4 rounds on 2w bits + cycle walking
  uint64_t d, mask, keys[4];
  int half;
  __host__ __device__ uint64_t once(uint64_t x) const {
    uint64_t L = x >> half, R = x & mask;
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = mix64(R ^ keys[r]) & mask;
      const uint64_t nL = R;
      R = L ^ F;
      L = nL;
    }
    return (L << half) | R;
  }
  __host__ __device__ uint64_t operator()(uint64_t x) const {
    uint64_t y = once(x);
    while (y >= d) y = once(y);
    return y;
  }
};

Feistel make_feistel(uint64_t d, uint64_t seed) {
  Feistel f;
  f.d = d;
  int bits = 2;
  while ((1ULL << bits) < d) bits += 2;
  f.half = bits / 2;
  f.mask = (1ULL << f.half) - 1;
  for (int r = 0; r < 4; ++r) f.keys[r] = mix64(seed ^ (0xA5A5A5A5ULL + r));
  return f;
}

constexpr int kMaxRow = 256;      // nonzeros per generated row (Poisson tail clamp)
constexpr int kZipfTable = 4096;  // ranks with an explicit CDF entry
constexpr int kGenWarps = 8;

struct GenArgs {
  int64_t n, row0, d_sparse, d_dense;
  double mean, exp_neg_mean;
  int value_law, dense_fp16, table_n;
  uint64_t seed;
  double acc, tail, total, a_pow, s;  // Zipf: table mass, tail mass, a^(1-s)
  Feistel fe;
  const double* cdf;
};

__global__ void k_gen_counts(GenArgs a, int64_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int64_t k = 0;
  if (a.d_sparse > 0 && a.mean > 0) {
    const uint64_t key = row_key(a.seed, (uint64_t)(a.row0 + i), 0);
    if (a.mean > 500.0) {  // normal approximation (hostbuild.cpp)
      const double x = floor(a.mean + sqrt(a.mean) * normal_at(key, 0) + 0.5);
      k = x < 0 ? 0 : (int64_t)x;
    } else {  // Knuth: multiply uniforms until the product drops below e^-mean
      double p = 1.0;
      uint64_t c = 0;
      do {
        ++k;
        p *= unif(draw(key, c++));
      } while (p > a.exp_neg_mean);
      k -= 1;
    }
    k = min(k, (int64_t)kMaxRow);
    k = min(k, a.d_sparse);
  }
  counts[i] = k;
}

__device__ __forceinline__ uint32_t zipf_rank(const GenArgs& a, const double* cdf, double u01) {
  const double u = u01 * a.total;
  if (u < a.acc || a.tail == 0.0) {  // lower_bound in the CDF table
    int lo = 0, hi = a.table_n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    return (uint32_t)min(lo, a.table_n - 1);
  }
  // invert the continuous tail  int_{table_n+0.5}^{x} t^-s dt = u - acc
  const double x = pow(a.a_pow - (u - a.acc) * (a.s - 1.0), 1.0 / (1.0 - a.s));
  int64_t r = (int64_t)floor(x - 0.5);
  if (r < a.table_n) r = a.table_n;
  if (r >= a.d_sparse) r = a.d_sparse - 1;
  return (uint32_t)r;
}

// One warp per row.  Ranks: each round every lane draws one candidate; a
// candidate is taken if no accepted rank and no lower lane of the round has
// it (draw order decides), until the row's count is reached.
__global__ void __launch_bounds__(kGenWarps * 32)
k_gen_rows(GenArgs a, const int64_t* __restrict__ indptr, uint32_t* __restrict__ indices,
           float* __restrict__ data, float* __restrict__ dense, __half* __restrict__ dense_h) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_cdf = reinterpret_cast<double*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* s_val = s_cdf + a.table_n + warp * kMaxRow;
  uint32_t* s_dim = reinterpret_cast<uint32_t*>(s_cdf + a.table_n + kGenWarps * kMaxRow) + warp * kMaxRow;
  for (int i = threadIdx.x; i < a.table_n; i += blockDim.x) s_cdf[i] = a.cdf[i];
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * kGenWarps + warp; i < a.n;
       i += (int64_t)gridDim.x * kGenWarps) {
    const uint64_t row = (uint64_t)(a.row0 + i);
    const int64_t o = indptr[i];
    const int k = (int)(indptr[i + 1] - o);
    // ranks in draw order
    const uint64_t kr = row_key(a.seed, row, 1);
    int acc = 0;
    for (uint64_t round = 0; acc < k; ++round) {
      const uint32_t rank = zipf_rank(a, s_cdf, unif(draw(kr, round * 32 + lane)));
      bool dup = false;
      for (int j = 0; j < acc; ++j) dup |= s_dim[j] == rank;
      const unsigned same = __match_any_sync(FULL, rank);
      const bool take = !dup && (__ffs(same) - 1) == lane;
      const unsigned bal = __ballot_sync(FULL, take);
      const int at = acc + __popc(bal & lt);
      if (take && at < k) s_dim[at] = rank;
      acc = min(k, acc + __popc(bal));
      __syncwarp();
    }
    // dims through the bijection, values, squared norm (f64)
    const uint64_t kv = row_key(a.seed, row, 2), kd = row_key(a.seed, row, 3);
    double ss = 0.0;
    for (int j = lane; j < k; j += 32) {
      s_dim[j] = (uint32_t)a.fe((uint64_t)s_dim[j]);
      const double z = normal_at(kv, (uint64_t)j);
      double v = a.value_law == 1 ? exp(z) : fabs(z);
      if (v == 0.0) v = 1e-30;
      s_val[j] = v;
      ss = fma(v, v, ss);
    }
    for (int64_t j = lane; j < a.d_dense; j += 32) {
      const double z = normal_at(kd, (uint64_t)j);
      ss = fma(z, z, ss);
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) ss += __shfl_xor_sync(FULL, ss, m);
    const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 1.0;
    // sort the row by dim (bitonic over the next power of two)
    int P = 1;
    while (P < k) P <<= 1;
    for (int j = k + lane; j < P; j += 32) s_dim[j] = 0xFFFFFFFFu;
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < (P >> 1); t += 32) {
          const int x = 2 * t - (t & (stride - 1));
          const int y = x + stride;
          const bool asc = (x & size) == 0;
          const uint32_t dx = s_dim[x], dy = s_dim[y];
          if ((dx > dy) == asc) {
            s_dim[x] = dy;
            s_dim[y] = dx;
            const double vx = s_val[x];
            s_val[x] = s_val[y];
            s_val[y] = vx;
          }
        }
        __syncwarp();
      }
    }
    for (int j = lane; j < k; j += 32) {
      indices[o + j] = s_dim[j];
      float f = (float)(s_val[j] * inv);
      if (f == 0.0f) f = 1e-38f;
      data[o + j] = f;
    }
    for (int64_t j = lane; j < a.d_dense; j += 32) {
      const float f = (float)(normal_at(kd, (uint64_t)j) * inv);
      if (a.dense_fp16) dense_h[(int64_t)i * a.d_dense + j] = __float2half_rn(f);
      else dense[(int64_t)i * a.d_dense + j] = f;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// sparse build kernels
// ---------------------------------------------------------------------------
constexpr uint32_t kHeadTag = 0x80000000u;
constexpr uint32_t kInf = 0xFFFFFFFFu;

__global__ void k_dim_count(const uint32_t* __restrict__ idx, int64_t nnz, uint32_t* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + idx[e], 1u);
}

// dims with cnt[d] > t (unordered; sorted afterwards), or with cnt[d] > 0 when t < 0
__global__ void k_collect_dims(const uint32_t* __restrict__ cnt, int64_t d, int64_t t,
                               uint32_t* __restrict__ out, unsigned long long* __restrict__ nout) {
  __shared__ uint32_t s_buf[1024];
  __shared__ unsigned s_n;
  __shared__ unsigned long long s_base;
  for (int64_t b0 = (int64_t)blockIdx.x * 1024; b0 < d; b0 += (int64_t)gridDim.x * 1024) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < 1024; j += blockDim.x) {
      const int64_t x = b0 + j;
      if (x < d && (int64_t)cnt[x] > (t < 0 ? 0 : t)) s_buf[atomicAdd(&s_n, 1u)] = (uint32_t)x;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_n) s_base = atomicAdd(nout, (unsigned long long)s_n);
    __syncthreads();
    for (unsigned j = threadIdx.x; j < s_n; j += blockDim.x) out[s_base + j] = s_buf[j];
    __syncthreads();
  }
}

__global__ void k_tag_head(const uint32_t* __restrict__ hd, int64_t H, uint32_t* __restrict__ tab) {
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h < H) tab[hd[h]] = kHeadTag | (uint32_t)h;
}

__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// one 8-bit pass of the per-head-dim radix select
__global__ void k_head_hist(const uint32_t* __restrict__ idx, const float* __restrict__ val,
                            int64_t nnz, const uint32_t* __restrict__ tab,
                            const uint32_t* __restrict__ prefix, int shift,
                            uint32_t* __restrict__ hist) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = tab[idx[e]];
    if (!(t & kHeadTag)) continue;
    const uint32_t h = t & ~kHeadTag;
    const float v = val[e];
    if (isnan(v)) continue;
    const uint32_t key = mag_key(v);
    if (shift < 24 && (key >> (shift + 8)) != (prefix[h] >> (shift + 8))) continue;
    atomicAdd(hist + (int64_t)h * 256 + ((key >> shift) & 255u), 1u);
  }
}

// per head dim: pick the bin holding the rem-th largest, clear the histogram
__global__ void k_head_pick(int64_t H, int shift, uint32_t* __restrict__ hist,
                            uint32_t* __restrict__ prefix, uint32_t* __restrict__ rem) {
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  uint32_t* row = hist + h * 256;
  uint32_t r = rem[h], cum = 0;
  int b = 255;
  for (; b > 0; --b) {
    const uint32_t c = row[b];
    if (cum + c >= r) break;
    cum += c;
  }
  prefix[h] |= (uint32_t)b << shift;
  rem[h] = r - cum;
  for (int j = 0; j < 256; ++j) row[j] = 0;
}

// data-part flag per raw entry (one ballot word per 32 entries)
__global__ void k_data_mask(const uint32_t* __restrict__ idx, const float* __restrict__ val,
                            int64_t nnz, const uint32_t* __restrict__ tab,
                            const uint32_t* __restrict__ thr, int mode, double data_min,
                            uint32_t* __restrict__ mask) {
  // mode 0: top_t (head dims compare against thr, others keep all),
  // mode 1: constant data_min, mode 2: top_t == 0 (nothing is data)
  const int64_t words = (nnz + 31) / 32;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e = w * 32 + (threadIdx.x & 31);
    bool data = false;
    if (e < nnz && mode != 2) {
      const float v = val[e];
      if (!isnan(v)) {
        if (mode == 1) {
          data = fabs((double)v) >= data_min;
        } else {
          const uint32_t t = tab[idx[e]];
          data = (t & kHeadTag) ? mag_key(v) >= thr[t & ~kHeadTag] : true;
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, data);
    if ((threadIdx.x & 31) == 0) mask[w] = bal;
  }
}

__device__ __forceinline__ bool bit_of(const uint32_t* m, int64_t e) {
  return (m[e >> 5] >> (e & 31)) & 1u;
}

__global__ void k_data_count(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ mask,
                             int64_t nnz, uint32_t* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (bit_of(mask, e)) atomicAdd(cnt + idx[e], 1u);
}

__global__ void k_gather_u32(const uint32_t* __restrict__ tab, const uint32_t* __restrict__ at,
                             int64_t m, uint32_t* __restrict__ out, int complement) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = complement ? ~tab[at[i]] : tab[at[i]];
}

__global__ void k_scatter_rank(const uint32_t* __restrict__ ranked, int64_t m,
                               uint32_t* __restrict__ tab) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) tab[ranked[r]] = (uint32_t)r;
}

// data entries per row
__global__ void k_row_data_count(const int64_t* __restrict__ indptr, const uint32_t* __restrict__ mask,
                                 int64_t n, uint32_t* __restrict__ rc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    rc[n] = 0;
    return;
  }
  uint32_t c = 0;
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) c += bit_of(mask, e);
  rc[i] = c;
}

// per row: ascending ranks of its data entries (insertion sort in place)
__global__ void k_row_ranks(const int64_t* __restrict__ indptr, const uint32_t* __restrict__ idx,
                            const uint32_t* __restrict__ mask, const uint32_t* __restrict__ rank,
                            int64_t n, const uint32_t* __restrict__ rptr, uint32_t* __restrict__ rl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t* out = rl + rptr[i];
  int m = 0;
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
    if (!bit_of(mask, e)) continue;
    const uint32_t r = rank[idx[e]];
    int j = m++;
    while (j > 0 && out[j - 1] > r) {
      out[j] = out[j - 1];
      --j;
    }
    out[j] = r;
  }
}

__global__ void k_first_key(const uint32_t* __restrict__ rptr, const uint32_t* __restrict__ rl,
                            int64_t n, uint32_t* __restrict__ key, uint32_t* __restrict__ iota) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = rptr[i + 1] > rptr[i] ? rl[rptr[i]] : kInf;
  iota[i] = (uint32_t)i;
}

// depth 0: flag positions inside a run (length >= 2) of equal non-inf keys;
// head value = position where a run starts (max-scanned into run starts)
__global__ void k_runs32(const uint32_t* __restrict__ sk, int64_t m, uint8_t* __restrict__ flag,
                         uint32_t* __restrict__ head) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const uint32_t k = sk[p];
  const bool prev = p > 0 && sk[p - 1] == k, next = p + 1 < m && sk[p + 1] == k;
  flag[p] = (k != kInf) && (prev || next);
  head[p] = prev ? 0u : (uint32_t)p;
}

__global__ void k_runs64(const unsigned long long* __restrict__ sk, const uint32_t* __restrict__ pos,
                         int64_t m, uint8_t* __restrict__ flag, uint32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long k = sk[i];
  const bool prev = i > 0 && sk[i - 1] == k, next = i + 1 < m && sk[i + 1] == k;
  flag[i] = ((uint32_t)k != kInf) && (prev || next);
  head[i] = prev ? 0u : pos[i];
}

__global__ void k_depth_keys(const uint32_t* __restrict__ act_pos, const uint32_t* __restrict__ act_seg,
                             int64_t m, const uint32_t* __restrict__ perm,
                             const uint32_t* __restrict__ rptr, const uint32_t* __restrict__ rl,
                             uint32_t depth, unsigned long long* __restrict__ key,
                             uint32_t* __restrict__ row_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t row = perm[act_pos[i]];
  const uint32_t b = rptr[row], len = rptr[row + 1] - b;
  const uint32_t r = len > depth ? rl[b + depth] : kInf;
  key[i] = ((unsigned long long)act_seg[i] << 32) | r;
  row_out[i] = row;
}

__global__ void k_write_back(const uint32_t* __restrict__ act_pos, const uint32_t* __restrict__ rows,
                             int64_t m, uint32_t* __restrict__ perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) perm[act_pos[i]] = rows[i];
}

__global__ void k_gather_pair(const uint32_t* __restrict__ sel, int64_t m,
                              const uint32_t* __restrict__ a_in, const uint32_t* __restrict__ b_in,
                              uint32_t* __restrict__ a_out, uint32_t* __restrict__ b_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t s = sel[i];
  a_out[i] = a_in[s];
  b_out[i] = b_in[s];
}

__global__ void k_invert(const uint32_t* __restrict__ order, int64_t n, uint32_t* __restrict__ pos) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) pos[order[s]] = (uint32_t)s;
}

// (dim << 32 | slot, w) for every data entry, written at the row's data offset
__global__ void k_posting_keys(const int64_t* __restrict__ indptr, const uint32_t* __restrict__ idx,
                               const float* __restrict__ val, const uint32_t* __restrict__ mask,
                               int64_t n, const uint32_t* __restrict__ rptr,
                               const uint32_t* __restrict__ pos, unsigned long long* __restrict__ key,
                               float* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t o = rptr[i];
  const unsigned long long slot = pos[i];
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
    if (!bit_of(mask, e)) continue;
    key[o] = ((unsigned long long)idx[e] << 32) | slot;
    w[o] = val[e];
    ++o;
  }
}

__global__ void k_popc_total(const uint32_t* __restrict__ mask, int64_t words,
                             unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(mask[w]);
  for (int m = 16; m; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_interleave_post(const unsigned long long* __restrict__ key,
                                  const float* __restrict__ w, int64_t m, uint2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = make_uint2((uint32_t)key[i], __float_as_uint(w[i]));
  if (i == m) out[m] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // pad posting
}

__global__ void k_check_rows(const int64_t* __restrict__ indptr, const uint32_t* __restrict__ idx,
                             int64_t n, int64_t d, int* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = indptr[i], e = indptr[i + 1];
  if (e < b) {
    atomicOr(bad, 1);
    return;
  }
  for (int64_t x = b; x < e; ++x) {
    if ((int64_t)idx[x] >= d) atomicOr(bad, 2);
    if (x > b && idx[x] <= idx[x - 1]) atomicOr(bad, 4);
  }
}

struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};
struct MinF {
  __device__ __forceinline__ float operator()(float a, float b) const { return fminf(a, b); }
};
struct MaxF {
  __device__ __forceinline__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

unsigned grid_for(int64_t items, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, threads), 65535LL * 64));
}
unsigned stride_grid() { return kNumSMs * 16; }

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return std::max(b, 1);
}

// ---- cub wrappers (temp storage from the builder) ----
template <typename K, typename V>
int sort_pairs(Builder& b, const K* kin, K* kout, const V* vin, V* vout, int64_t m, int bb, int eb) {
  if (m <= 0) return HS_OK;
  if (m > INT32_MAX) HS_FAIL(HS_EUNSUPPORTED, "build: more than 2^31 items in one sort");
  size_t bytes = 0;
  HS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)m, bb, eb, b.st));
  HS_CHECK(builder_tmp(b, bytes));
  HS_CUDA(cub::DeviceRadixSort::SortPairs(b.tmp, bytes, kin, kout, vin, vout, (int)m, bb, eb, b.st));
  return HS_OK;
}
template <typename K>
int sort_keys(Builder& b, const K* kin, K* kout, int64_t m, int bb, int eb) {
  if (m <= 0) return HS_OK;
  if (m > INT32_MAX) HS_FAIL(HS_EUNSUPPORTED, "build: more than 2^31 items in one sort");
  size_t bytes = 0;
  HS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kin, kout, (int)m, bb, eb, b.st));
  HS_CHECK(builder_tmp(b, bytes));
  HS_CUDA(cub::DeviceRadixSort::SortKeys(b.tmp, bytes, kin, kout, (int)m, bb, eb, b.st));
  return HS_OK;
}
template <typename In, typename Out>
int excl_sum(Builder& b, In in, Out out, int64_t m) {
  if (m <= 0) return HS_OK;
  if (m > INT32_MAX) HS_FAIL(HS_EUNSUPPORTED, "build: more than 2^31 items in one scan");
  size_t bytes = 0;
  HS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)m, b.st));
  HS_CHECK(builder_tmp(b, bytes));
  HS_CUDA(cub::DeviceScan::ExclusiveSum(b.tmp, bytes, in, out, (int)m, b.st));
  return HS_OK;
}
int max_scan(Builder& b, const uint32_t* in, uint32_t* out, int64_t m) {
  if (m <= 0) return HS_OK;
  size_t bytes = 0;
  HS_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, in, out, MaxU32(), (int)m, b.st));
  HS_CHECK(builder_tmp(b, bytes));
  HS_CUDA(cub::DeviceScan::InclusiveScan(b.tmp, bytes, in, out, MaxU32(), (int)m, b.st));
  return HS_OK;
}
// indices i in [0, m) with flag[i] != 0, ascending
int select_flagged(Builder& b, const uint8_t* flag, int64_t m, uint32_t* out, int64_t* count) {
  *count = 0;
  if (m <= 0) return HS_OK;
  int64_t* d_cnt = nullptr;
  HS_CUDA(cudaMalloc(&d_cnt, sizeof(int64_t)));
  thrust::counting_iterator<uint32_t> it(0);
  size_t bytes = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, bytes, it, flag, out, d_cnt, (int)m, b.st);
  int rc = e == cudaSuccess ? builder_tmp(b, bytes) : HS_ECUDA;
  if (rc == HS_OK) {
    e = cub::DeviceSelect::Flagged(b.tmp, bytes, it, flag, out, d_cnt, (int)m, b.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(count, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, b.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(b.st);
  }
  cudaFree(d_cnt);
  if (rc != HS_OK) return rc;
  HS_CUDA(e);
  return HS_OK;
}
template <typename Op>
int reduce_f(Builder& b, const float* in, int64_t m, Op op, float init, float* host_out) {
  float* d_out = nullptr;
  HS_CUDA(cudaMalloc(&d_out, sizeof(float)));
  size_t bytes = 0;
  cudaError_t e = cub::DeviceReduce::Reduce(nullptr, bytes, in, d_out, (int)m, op, init, b.st);
  int rc = e == cudaSuccess ? builder_tmp(b, bytes) : HS_ECUDA;
  if (rc == HS_OK) {
    e = cub::DeviceReduce::Reduce(b.tmp, bytes, in, d_out, (int)m, op, init, b.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host_out, d_out, sizeof(float), cudaMemcpyDeviceToHost, b.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(b.st);
  }
  cudaFree(d_out);
  if (rc != HS_OK) return rc;
  HS_CUDA(e);
  return HS_OK;
}

// RAII device scratch freed at scope exit
struct Scratch {
  std::vector<void*> ptrs;
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  int get(T** p, size_t count) {
    *p = nullptr;
    HS_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(count, 1)));
    ptrs.push_back(*p);
    return HS_OK;
  }
  void drop(void* p) {
    auto it = std::find(ptrs.begin(), ptrs.end(), p);
    if (it != ptrs.end()) {
      cudaFree(p);
      ptrs.erase(it);
    }
  }
};

// the cache sort (see the file header); perm = order on return
int cache_sort_dev(Builder& b, const uint32_t* rptr, const uint32_t* rl, uint32_t* perm) {
  const int64_t n = b.n;
  const int T = 256;
  Scratch s;
  uint32_t *k0, *k1, *iota;
  HS_CHECK(s.get(&k0, n));
  HS_CHECK(s.get(&k1, n));
  HS_CHECK(s.get(&iota, n));
  k_first_key<<<grid_for(n), T, 0, b.st>>>(rptr, rl, n, k0, iota);
  HS_CHECK(sort_pairs(b, k0, k1, iota, perm, n, 0, 32));
  // depth-0 runs
  uint8_t* flag;
  uint32_t* head;
  HS_CHECK(s.get(&flag, n));
  HS_CHECK(s.get(&head, n));
  k_runs32<<<grid_for(n), T, 0, b.st>>>(k1, n, flag, head);
  uint32_t* runst = k0;  // reuse
  HS_CHECK(max_scan(b, head, runst, n));
  uint32_t *act_pos, *act_seg;
  HS_CHECK(s.get(&act_pos, n));
  HS_CHECK(s.get(&act_seg, n));
  int64_t m = 0;
  uint32_t* sel = iota;  // reuse
  HS_CHECK(select_flagged(b, flag, n, sel, &m));
  // active positions and the start of their run (segment)
  if (m) {
    HS_CUDA(cudaMemcpyAsync(act_pos, sel, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, b.st));
    k_gather_u32<<<grid_for(m), T, 0, b.st>>>(runst, sel, m, act_seg, 0);
  }
  s.drop(k1);
  unsigned long long *key, *key2;
  uint32_t *row, *row2, *pos2, *seg2;
  HS_CHECK(s.get(&key, std::max<int64_t>(m, 1)));
  HS_CHECK(s.get(&key2, std::max<int64_t>(m, 1)));
  HS_CHECK(s.get(&row, std::max<int64_t>(m, 1)));
  HS_CHECK(s.get(&row2, std::max<int64_t>(m, 1)));
  HS_CHECK(s.get(&pos2, std::max<int64_t>(m, 1)));
  HS_CHECK(s.get(&seg2, std::max<int64_t>(m, 1)));
  const int kb = 32 + bits_for((uint64_t)n);
  for (uint32_t depth = 1; m > 0; ++depth) {
    k_depth_keys<<<grid_for(m), T, 0, b.st>>>(act_pos, act_seg, m, perm, rptr, rl, depth, key, row);
    HS_CHECK(sort_pairs(b, key, key2, row, row2, m, 0, kb));
    k_write_back<<<grid_for(m), T, 0, b.st>>>(act_pos, row2, m, perm);
    k_runs64<<<grid_for(m), T, 0, b.st>>>(key2, act_pos, m, flag, head);
    HS_CHECK(max_scan(b, head, runst, m));
    int64_t m2 = 0;
    HS_CHECK(select_flagged(b, flag, m, sel, &m2));
    k_gather_pair<<<grid_for(m2), T, 0, b.st>>>(sel, m2, act_pos, runst, pos2, seg2);
    std::swap(act_pos, pos2);
    std::swap(act_seg, seg2);
    m = m2;
    if (depth > (1u << 30)) HS_FAIL(HS_ECUDA, "cache sort did not converge");
  }
  HS_CUDA(cudaStreamSynchronize(b.st));
  return HS_OK;
}

}  // namespace
}  // namespace hs

using namespace hs;

struct hs_builder : public hs::Builder {};

namespace {
void destroy_builder(hs_builder* b) {
  if (!b) return;
  hs::builder_free(b);
  delete b;
}
using BuilderPtr = std::unique_ptr<hs_builder, void (*)(hs_builder*)>;

int make_builder(int device, BuilderPtr* out) {
  HS_CUDA(cudaSetDevice(device));
  out->reset(new hs_builder());
  (*out)->device = device;
  HS_CUDA(cudaStreamCreateWithFlags(&(*out)->st, cudaStreamNonBlocking));
  return HS_OK;
}

int alloc_dataset(hs_builder& b) {
  HS_CUDA(cudaMalloc(&b.indptr, sizeof(int64_t) * (b.n + 1)));
  return HS_OK;
}

int alloc_entries(hs_builder& b) {
  HS_CUDA(cudaMalloc(&b.indices, sizeof(uint32_t) * std::max<int64_t>(b.nnz, 1)));
  HS_CUDA(cudaMalloc(&b.data, sizeof(float) * std::max<int64_t>(b.nnz, 1)));
  if (b.d_dense > 0) {
    const size_t cnt = (size_t)b.n * b.d_dense;
    if (b.dense_fp16) HS_CUDA(cudaMalloc(&b.dense_h, sizeof(__half) * std::max<size_t>(cnt, 1)));
    else HS_CUDA(cudaMalloc(&b.dense, sizeof(float) * std::max<size_t>(cnt, 1)));
  }
  return HS_OK;
}
}  // namespace

extern "C" {

int hs_builder_generate(const hs_gen_params* p, int device, hs_builder_t* out) {
  if (!p || !out) HS_FAIL(HS_EINVAL, "null argument");
  *out = nullptr;
  if (p->n < 0 || p->d_sparse < 0 || p->d_dense < 0 || p->row0 < 0)
    HS_FAIL(HS_EINVAL, "generator: negative size");
  if (p->n >= (int64_t)INT32_MAX) HS_FAIL(HS_EUNSUPPORTED, "generator: n must be < 2^31");
  if (p->d_sparse > (int64_t)0xFFFFFFFFLL) HS_FAIL(HS_EINVAL, "d_sparse must be < 2^32");
  if (p->d_sparse > 0 && !(p->zipf_s > 1.0)) HS_FAIL(HS_EINVAL, "generator: zipf_s must be > 1");
  BuilderPtr b(nullptr, destroy_builder);
  HS_CHECK(make_builder(device, &b));
  const auto t0 = std::chrono::steady_clock::now();
  b->n = p->n;
  b->d_sparse = p->d_sparse;
  b->d_dense = p->d_dense;
  b->dense_fp16 = p->dense_fp16 ? 1 : 0;
  // Zipf CDF table (host, sequential f64 sum) and tail constants
  GenArgs a{};
  a.n = p->n;
  a.row0 = p->row0;
  a.d_sparse = p->d_sparse;
  a.d_dense = p->d_dense;
  a.mean = p->mean_nnz;
  a.exp_neg_mean = std::exp(-p->mean_nnz);
  a.value_law = p->value_law;
  a.dense_fp16 = b->dense_fp16;
  a.seed = p->seed;
  a.s = p->zipf_s;
  const int64_t dsp = p->d_sparse > 1 ? p->d_sparse : 1;
  a.table_n = (int)(dsp < (int64_t)kZipfTable ? dsp : (int64_t)kZipfTable);
  std::vector<double> cdf(a.table_n);
  double acc = 0.0;
  for (int r = 0; r < a.table_n; ++r) {
    acc += std::pow((double)(r + 1), -p->zipf_s);
    cdf[r] = acc;
  }
  a.acc = acc;
  a.tail = 0.0;
  if (p->d_sparse > a.table_n) {
    const double lo = (double)a.table_n + 0.5, hi = (double)p->d_sparse + 0.5;
    a.a_pow = std::pow(lo, 1.0 - p->zipf_s);
    a.tail = (a.a_pow - std::pow(hi, 1.0 - p->zipf_s)) / (p->zipf_s - 1.0);
  }
  a.total = a.acc + a.tail;
  a.fe = make_feistel((uint64_t)std::max<int64_t>(p->d_sparse, 1), p->perm_seed);
  double* dcdf = nullptr;
  HS_CUDA(cudaMalloc(&dcdf, sizeof(double) * a.table_n));
  std::unique_ptr<double, decltype(&cudaFree)> gcdf(dcdf, cudaFree);
  HS_CUDA(cudaMemcpy(dcdf, cdf.data(), sizeof(double) * a.table_n, cudaMemcpyHostToDevice));
  a.cdf = dcdf;
  HS_CHECK(alloc_dataset(*b));
  // counts -> indptr
  if (b->n > 0) {
    int64_t* counts = nullptr;
    HS_CUDA(cudaMalloc(&counts, sizeof(int64_t) * b->n));
    std::unique_ptr<int64_t, decltype(&cudaFree)> gc(counts, cudaFree);
    k_gen_counts<<<grid_for(b->n), 256, 0, b->st>>>(a, counts);
    HS_CUDA(cudaMemsetAsync(b->indptr, 0, sizeof(int64_t), b->st));
    size_t bytes = 0;
    HS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, counts, b->indptr + 1, (int)b->n, b->st));
    HS_CHECK(builder_tmp(*b, bytes));
    HS_CUDA(cub::DeviceScan::InclusiveSum(b->tmp, bytes, counts, b->indptr + 1, (int)b->n, b->st));
    HS_CUDA(cudaMemcpyAsync(&b->nnz, b->indptr + b->n, sizeof(int64_t), cudaMemcpyDeviceToHost, b->st));
    HS_CUDA(cudaStreamSynchronize(b->st));
  } else {
    HS_CUDA(cudaMemset(b->indptr, 0, sizeof(int64_t)));
  }
  HS_CHECK(alloc_entries(*b));
  if (b->n > 0) {
    const size_t smem = sizeof(double) * a.table_n + (sizeof(double) + sizeof(uint32_t)) * kGenWarps * kMaxRow;
    HS_CUDA(cudaFuncSetAttribute(k_gen_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>(ceil_div(b->n, kGenWarps), (int64_t)kNumSMs * 8);
    k_gen_rows<<<(unsigned)blocks, kGenWarps * 32, smem, b->st>>>(a, b->indptr, b->indices, b->data,
                                                                   b->dense, b->dense_h);
    HS_CUDA(cudaGetLastError());
  }
  HS_CUDA(cudaStreamSynchronize(b->st));
  builder_phase(*b, "generate", secs_since(t0));
  *out = b.release();
  return HS_OK;
}

int hs_builder_upload(int64_t n, int64_t d_sparse, int64_t d_dense, const int64_t* indptr,
                      const uint32_t* indices, const float* data, const float* dense,
                      int32_t dense_fp16, int device, hs_builder_t* out) {
  if (!out || n < 0 || d_sparse < 0 || d_dense < 0 || !indptr) HS_FAIL(HS_EINVAL, "bad arguments");
  *out = nullptr;
  if (n >= (int64_t)INT32_MAX) HS_FAIL(HS_EUNSUPPORTED, "build: n must be < 2^31");
  if (d_sparse > (int64_t)0xFFFFFFFFLL) HS_FAIL(HS_EINVAL, "d_sparse must be < 2^32");
  if (indptr[0] != 0) HS_FAIL(HS_EINVAL, "dataset row pointers must start at 0");
  BuilderPtr b(nullptr, destroy_builder);
  HS_CHECK(make_builder(device, &b));
  const auto t0 = std::chrono::steady_clock::now();
  b->n = n;
  b->d_sparse = d_sparse;
  b->d_dense = d_dense;
  b->dense_fp16 = dense_fp16 ? 1 : 0;
  b->nnz = indptr[n];
  HS_CHECK(alloc_dataset(*b));
  HS_CHECK(alloc_entries(*b));
  HS_CUDA(cudaMemcpy(b->indptr, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  if (b->nnz) {
    HS_CUDA(cudaMemcpy(b->indices, indices, sizeof(uint32_t) * b->nnz, cudaMemcpyHostToDevice));
    HS_CUDA(cudaMemcpy(b->data, data, sizeof(float) * b->nnz, cudaMemcpyHostToDevice));
  }
  if (d_dense > 0 && n > 0) {
    if (!dense) HS_FAIL(HS_EINVAL, "dataset dense part missing");
    const size_t cnt = (size_t)n * d_dense;
    if (b->dense_fp16) {  // values must be fp16-exact (they are rounded here)
      std::vector<__half> h(cnt);
      for (size_t i = 0; i < cnt; ++i) h[i] = __float2half_rn(dense[i]);
      HS_CUDA(cudaMemcpy(b->dense_h, h.data(), sizeof(__half) * cnt, cudaMemcpyHostToDevice));
    } else {
      HS_CUDA(cudaMemcpy(b->dense, dense, sizeof(float) * cnt, cudaMemcpyHostToDevice));
    }
  }
  // canonical CSR: monotone row pointers, columns ascending and < d_sparse
  int* bad = nullptr;
  HS_CUDA(cudaMalloc(&bad, sizeof(int)));
  std::unique_ptr<int, decltype(&cudaFree)> gbad(bad, cudaFree);
  HS_CUDA(cudaMemset(bad, 0, sizeof(int)));
  if (n) k_check_rows<<<grid_for(n), 256, 0, b->st>>>(b->indptr, b->indices, n, d_sparse, bad);
  int hb = 0;
  HS_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, b->st));
  HS_CUDA(cudaStreamSynchronize(b->st));
  if (hb & 1) HS_FAIL(HS_EINVAL, "dataset row pointers not monotone");
  if (hb & 2) HS_FAIL(HS_EINVAL, "dataset column index out of range");
  if (hb & 4) HS_FAIL(HS_EINVAL, "dataset rows must have strictly ascending column indices");
  builder_phase(*b, "upload", secs_since(t0));
  *out = b.release();
  return HS_OK;
}

void hs_builder_destroy(hs_builder_t b) { destroy_builder(b); }

int hs_builder_info(hs_builder_t b, int64_t* info) {
  if (!b || !info) HS_FAIL(HS_EINVAL, "null argument");
  info[0] = b->n;
  info[1] = b->d_sparse;
  info[2] = b->d_dense;
  info[3] = b->nnz;
  info[4] = b->n_active;
  info[5] = b->nnz_post;
  info[6] = b->n_head;
  info[7] = b->dense_fp16;
  return HS_OK;
}

int hs_builder_phase_times(hs_builder_t b, double* sec, int32_t max_entries, int32_t* n_entries,
                           char* names, int32_t names_cap) {
  if (!b || !n_entries) HS_FAIL(HS_EINVAL, "null argument");
  const int32_t n = (int32_t)std::min<size_t>(b->tsec.size(), (size_t)max_entries);
  std::string joined;
  for (int32_t i = 0; i < n; ++i) {
    sec[i] = b->tsec[i];
    if (i) joined += ";";
    joined += b->tnames[i];
  }
  *n_entries = n;
  if (names && names_cap > 0) {
    std::strncpy(names, joined.c_str(), names_cap - 1);
    names[names_cap - 1] = 0;
  }
  return HS_OK;
}

// Rows [lo, hi) of the resident dataset: CSR (indptr relative to lo) and the
// dense part as f32 (fp16 values upcast exactly).  NULL outputs are skipped.
int hs_builder_download_rows(hs_builder_t b, int64_t lo, int64_t hi, int64_t* indptr,
                             uint32_t* indices, float* data, float* dense) {
  if (!b || lo < 0 || hi < lo || hi > b->n) HS_FAIL(HS_EINVAL, "row range out of range");
  HS_CUDA(cudaSetDevice(b->device));
  std::vector<int64_t> ptr(hi - lo + 1);
  HS_CUDA(cudaMemcpy(ptr.data(), b->indptr + lo, sizeof(int64_t) * (hi - lo + 1), cudaMemcpyDeviceToHost));
  const int64_t e0 = ptr[0], e1 = ptr[hi - lo];
  if (indptr)
    for (int64_t i = 0; i <= hi - lo; ++i) indptr[i] = ptr[i] - e0;
  if (indices && e1 > e0)
    HS_CUDA(cudaMemcpy(indices, b->indices + e0, sizeof(uint32_t) * (e1 - e0), cudaMemcpyDeviceToHost));
  if (data && e1 > e0)
    HS_CUDA(cudaMemcpy(data, b->data + e0, sizeof(float) * (e1 - e0), cudaMemcpyDeviceToHost));
  if (dense && b->d_dense > 0 && hi > lo) {
    const size_t cnt = (size_t)(hi - lo) * b->d_dense;
    if (b->dense_fp16) {
      std::vector<__half> h(cnt);
      HS_CUDA(cudaMemcpy(h.data(), b->dense_h + (size_t)lo * b->d_dense, sizeof(__half) * cnt,
                         cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < cnt; ++i) dense[i] = __half2float(h[i]);
    } else {
      HS_CUDA(cudaMemcpy(dense, b->dense + (size_t)lo * b->d_dense, sizeof(float) * cnt,
                         cudaMemcpyDeviceToHost));
    }
  }
  return HS_OK;
}

// The sparse half of build_index (pipeline.py:129-138): thresholds, data-part
// flags, layout order (cache_sort), postings.  top_t < 0 means top_t=None with
// the constant data_min (config.data_threshold); residual_min is the
// constant residual threshold.
int hs_builder_sparse(hs_builder_t bp, int64_t top_t, double data_min, double residual_min) {
  if (!bp) HS_FAIL(HS_EINVAL, "null builder");
  Builder& b = *bp;
  if (b.sparse_done) HS_FAIL(HS_EINVAL, "sparse part already built");
  HS_CUDA(cudaSetDevice(b.device));
  if (top_t < 0 && !(data_min == data_min)) HS_FAIL(HS_EINVAL, "need top_t or a data threshold");
  if (top_t < 0 && residual_min > data_min)
    HS_FAIL(HS_EINVAL, "residual_min must be <= data_min in every dimension");
  const auto t0 = std::chrono::steady_clock::now();
  const int T = 256;
  const int64_t n = b.n, nnz = b.nnz, D = std::max<int64_t>(b.d_sparse, 1);
  b.res_eps = residual_min;
  Scratch s;
  uint32_t* tab;  // per-dim table: counts, head tags, data counts, ranks
  HS_CHECK(s.get(&tab, D));
  HS_CUDA(cudaMemsetAsync(tab, 0, sizeof(uint32_t) * D, b.st));
  HS_CUDA(cudaMalloc(&b.dmask, sizeof(uint32_t) * std::max<int64_t>(ceil_div(nnz, 32), 1)));
  unsigned long long* d_cnt;
  HS_CHECK(s.get(&d_cnt, 1));
  // --- thresholds (_top_t_thresholds) and data-part flags (prune_split) ---
  int mode = top_t < 0 ? 1 : (top_t == 0 ? 2 : 0);
  // PruneThresholds.resolve (sparse.py:53-63): eps > eta in any dim raises;
  // with top_t every dim with <= t entries has eta = 0
  if (mode == 0 && residual_min > 0.0)
    HS_FAIL(HS_EINVAL, "residual_min must be <= data_min in every dimension");
  if (mode == 0) {
    if (nnz) k_dim_count<<<stride_grid(), T, 0, b.st>>>(b.indices, nnz, tab);
    HS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), b.st));
    uint32_t* hd_u;
    HS_CHECK(s.get(&hd_u, D));
    k_collect_dims<<<(unsigned)std::min<int64_t>(ceil_div(D, 1024), kNumSMs * 16), T, 0, b.st>>>(
        tab, b.d_sparse, top_t, hd_u, d_cnt);
    unsigned long long H = 0;
    HS_CUDA(cudaMemcpyAsync(&H, d_cnt, sizeof(H), cudaMemcpyDeviceToHost, b.st));
    HS_CUDA(cudaStreamSynchronize(b.st));
    b.n_head = (int64_t)H;
    HS_CUDA(cudaMalloc(&b.head_dims, sizeof(uint32_t) * std::max<int64_t>(H, 1)));
    HS_CUDA(cudaMalloc(&b.head_thr, sizeof(uint32_t) * std::max<int64_t>(H, 1)));
    if (H) {
      HS_CHECK(sort_keys(b, hd_u, b.head_dims, (int64_t)H, 0, 32));
      s.drop(hd_u);
      k_tag_head<<<grid_for(H), T, 0, b.st>>>(b.head_dims, (int64_t)H, tab);
      uint32_t *hist, *rem;
      HS_CHECK(s.get(&hist, (size_t)H * 256));
      HS_CHECK(s.get(&rem, H));
      HS_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * H * 256, b.st));
      HS_CUDA(cudaMemsetAsync(b.head_thr, 0, sizeof(uint32_t) * H, b.st));
      std::vector<uint32_t> r0(H, (uint32_t)top_t);
      HS_CUDA(cudaMemcpyAsync(rem, r0.data(), sizeof(uint32_t) * H, cudaMemcpyHostToDevice, b.st));
      for (int shift = 24; shift >= 0; shift -= 8) {
        k_head_hist<<<stride_grid(), T, 0, b.st>>>(b.indices, b.data, nnz, tab, b.head_thr, shift, hist);
        k_head_pick<<<grid_for(H), T, 0, b.st>>>((int64_t)H, shift, hist, b.head_thr, rem);
      }
      HS_CUDA(cudaStreamSynchronize(b.st));
    } else {
      s.drop(hd_u);
    }
  }
  if (nnz)
    k_data_mask<<<stride_grid(), T, 0, b.st>>>(b.indices, b.data, nnz, tab, b.head_thr, mode,
                                                data_min, b.dmask);
  // --- data-part counts per dim, active dims, ranking (cache_sort's ranked) ---
  HS_CUDA(cudaMemsetAsync(tab, 0, sizeof(uint32_t) * D, b.st));
  if (nnz) k_data_count<<<stride_grid(), T, 0, b.st>>>(b.indices, b.dmask, nnz, tab);
  HS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), b.st));
  uint32_t* act_u;
  HS_CHECK(s.get(&act_u, D));
  k_collect_dims<<<(unsigned)std::min<int64_t>(ceil_div(D, 1024), kNumSMs * 16), T, 0, b.st>>>(
      tab, b.d_sparse, -1, act_u, d_cnt);
  unsigned long long A = 0;
  HS_CUDA(cudaMemcpyAsync(&A, d_cnt, sizeof(A), cudaMemcpyDeviceToHost, b.st));
  HS_CUDA(cudaStreamSynchronize(b.st));
  b.n_active = (int64_t)A;
  HS_CUDA(cudaMalloc(&b.post_dims, sizeof(uint32_t) * std::max<int64_t>(A, 1)));
  HS_CUDA(cudaMalloc(&b.post_ptr, sizeof(uint32_t) * (A + 1)));
  HS_CHECK(sort_keys(b, act_u, b.post_dims, (int64_t)A, 0, 32));
  s.drop(act_u);
  uint32_t *acnt, *ncnt, *ranked;
  HS_CHECK(s.get(&acnt, A + 1));
  HS_CHECK(s.get(&ncnt, A + 1));
  HS_CHECK(s.get(&ranked, A + 1));
  HS_CUDA(cudaMemsetAsync(acnt, 0, sizeof(uint32_t) * (A + 1), b.st));
  k_gather_u32<<<grid_for(A), T, 0, b.st>>>(tab, b.post_dims, (int64_t)A, acnt, 0);
  HS_CHECK(excl_sum(b, acnt, b.post_ptr, (int64_t)A + 1));
  {  // data entries counted in 64 bits: the u32 offsets hold < 2^32 postings
    unsigned long long tot = 0;
    HS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), b.st));
    if (nnz) k_popc_total<<<stride_grid(), T, 0, b.st>>>(b.dmask, ceil_div(nnz, 32), d_cnt);
    HS_CUDA(cudaMemcpyAsync(&tot, d_cnt, sizeof(tot), cudaMemcpyDeviceToHost, b.st));
    HS_CUDA(cudaStreamSynchronize(b.st));
    if (tot >= 0xFFFFFFFFull) HS_FAIL(HS_EUNSUPPORTED, "build: 2^32 or more postings");
    b.nnz_post = (int64_t)tot;
  }
  // ranked = active dims by (count desc, dim asc): stable sort on ~count
  k_gather_u32<<<grid_for(A), T, 0, b.st>>>(tab, b.post_dims, (int64_t)A, ncnt, 1);
  HS_CHECK(sort_pairs(b, ncnt, acnt, b.post_dims, ranked, (int64_t)A, 0, 32));
  k_scatter_rank<<<grid_for(A), T, 0, b.st>>>(ranked, (int64_t)A, tab);
  s.drop(ncnt);
  s.drop(acnt);
  s.drop(ranked);
  // --- per-row rank lists -> cache sort ---
  uint32_t *rptr, *rl;
  HS_CHECK(s.get(&rptr, n + 1));
  uint32_t* rc;
  HS_CHECK(s.get(&rc, n + 1));
  k_row_data_count<<<grid_for(n + 1), T, 0, b.st>>>(b.indptr, b.dmask, n, rc);
  HS_CHECK(excl_sum(b, rc, rptr, n + 1));
  s.drop(rc);
  uint32_t total = 0;
  HS_CUDA(cudaMemcpyAsync(&total, rptr + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, b.st));
  HS_CUDA(cudaStreamSynchronize(b.st));
  if ((int64_t)total != b.nnz_post) HS_FAIL(HS_ECUDA, "build: posting counts disagree");
  HS_CHECK(s.get(&rl, std::max<int64_t>(b.nnz_post, 1)));
  if (n) k_row_ranks<<<grid_for(n), T, 0, b.st>>>(b.indptr, b.indices, b.dmask, tab, n, rptr, rl);
  s.drop(tab);
  HS_CUDA(cudaMalloc(&b.order, sizeof(uint32_t) * std::max<int64_t>(n, 1)));
  const auto t1 = std::chrono::steady_clock::now();
  if (n) HS_CHECK(cache_sort_dev(b, rptr, rl, b.order));
  builder_phase(b, "cache_sort", secs_since(t1));
  s.drop(rl);
  // --- postings (build_inverted) ---
  uint32_t* pos;
  HS_CHECK(s.get(&pos, n));
  if (n) k_invert<<<grid_for(n), T, 0, b.st>>>(b.order, n, pos);
  const int64_t E = b.nnz_post;
  unsigned long long *k0, *k1;
  float *w0, *w1;
  HS_CHECK(s.get(&k0, E));
  HS_CHECK(s.get(&w0, E));
  if (n) k_posting_keys<<<grid_for(n), T, 0, b.st>>>(b.indptr, b.indices, b.data, b.dmask, n, rptr, pos, k0, w0);
  s.drop(pos);
  s.drop(rptr);
  HS_CHECK(s.get(&k1, E));
  HS_CHECK(s.get(&w1, E));
  HS_CHECK(sort_pairs(b, k0, k1, w0, w1, E, 0, 32 + bits_for((uint64_t)D)));
  s.drop(k0);
  s.drop(w0);
  HS_CUDA(cudaMalloc(&b.post, sizeof(uint2) * (E + 1)));
  k_interleave_post<<<grid_for(E + 1), T, 0, b.st>>>(k1, w1, E, b.post);
  if (E) {
    HS_CHECK(reduce_f(b, w1, E, MinF(), INFINITY, &b.wmin));
    HS_CHECK(reduce_f(b, w1, E, MaxF(), -INFINITY, &b.wmax));
  }
  HS_CUDA(cudaStreamSynchronize(b.st));
  HS_CUDA(cudaGetLastError());
  b.sparse_done = 1;
  builder_phase(b, "sparse_build", secs_since(t0));
  return HS_OK;
}

// Download of the sparse build products (parity against the host build).
// order [n] (layout slot -> row), post_dims [n_active], post_ptr [n_active+1],
// post_ids / post_w [nnz_post], dmask [ceil(nnz/32)], head_dims / head_thr
// [n_head] (the top_t thresholds as f32 |v|).  NULL outputs are skipped.
int hs_builder_download_sparse(hs_builder_t b, int64_t* order, uint32_t* post_dims,
                               int64_t* post_ptr, uint32_t* post_ids, float* post_w,
                               uint32_t* dmask, uint32_t* head_dims, float* head_thr) {
  if (!b) HS_FAIL(HS_EINVAL, "null builder");
  if (!b->sparse_done) HS_FAIL(HS_EINVAL, "sparse part not built");
  HS_CUDA(cudaSetDevice(b->device));
  if (order && b->n) {
    std::vector<uint32_t> o(b->n);
    HS_CUDA(cudaMemcpy(o.data(), b->order, sizeof(uint32_t) * b->n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < b->n; ++i) order[i] = o[i];
  }
  if (post_dims && b->n_active)
    HS_CUDA(cudaMemcpy(post_dims, b->post_dims, sizeof(uint32_t) * b->n_active, cudaMemcpyDeviceToHost));
  if (post_ptr) {
    std::vector<uint32_t> p(b->n_active + 1);
    HS_CUDA(cudaMemcpy(p.data(), b->post_ptr, sizeof(uint32_t) * (b->n_active + 1), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= b->n_active; ++i) post_ptr[i] = p[i];
  }
  if ((post_ids || post_w) && b->nnz_post) {
    std::vector<uint2> p(b->nnz_post);
    HS_CUDA(cudaMemcpy(p.data(), b->post, sizeof(uint2) * b->nnz_post, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < b->nnz_post; ++i) {
      if (post_ids) post_ids[i] = p[i].x;
      if (post_w) std::memcpy(post_w + i, &p[i].y, 4);
    }
  }
  if (dmask && b->nnz)
    HS_CUDA(cudaMemcpy(dmask, b->dmask, sizeof(uint32_t) * ceil_div(b->nnz, 32), cudaMemcpyDeviceToHost));
  if (head_dims && b->n_head)
    HS_CUDA(cudaMemcpy(head_dims, b->head_dims, sizeof(uint32_t) * b->n_head, cudaMemcpyDeviceToHost));
  if (head_thr && b->n_head)
    HS_CUDA(cudaMemcpy(head_thr, b->head_thr, sizeof(uint32_t) * b->n_head, cudaMemcpyDeviceToHost));
  return HS_OK;
}

}  // extern "C"
