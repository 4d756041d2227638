// common.cuh — shared device/host helpers for the hsb200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "../../include/hsb200.h"

namespace hs {

// --------------------------------------------------------------------------
// error plumbing: thread-local last error, status codes from hsb200.h
// --------------------------------------------------------------------------
void set_error(const std::string& msg);
const char* last_error();

struct Status {
  int code = HS_OK;
  bool ok() const { return code == HS_OK; }
};

#define HS_FAIL(code_, msg_)            \
  do {                                  \
    ::hs::set_error(msg_);              \
    return (code_);                     \
  } while (0)

#define HS_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::hs::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                      " at " + __FILE__ + ":" + std::to_string(__LINE__));     \
      return _e == cudaErrorMemoryAllocation ? HS_ENOMEM : HS_ECUDA;           \
    }                                                                          \
  } while (0)

#define HS_CHECK(expr)          \
  do {                          \
    int _s = (expr);            \
    if (_s != HS_OK) return _s; \
  } while (0)

constexpr int kNumSMs = 148;

// Device bounds checks for the debug build (HSB200_DEBUG=1 => -DHS_DEBUG).
#ifdef HS_DEBUG
#define HS_DCHECK(cond, ...)                                                       \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("HS_DCHECK %s:%d (%s) block(%d,%d) thread %d\n", __FILE__, __LINE__,   \
             #cond, blockIdx.x, blockIdx.y, threadIdx.x);                          \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define HS_DCHECK(cond, ...) \
  do {                       \
  } while (0)
#endif

// --------------------------------------------------------------------------
// candidate entries and the reference ordering (pipeline.py:165-189):
// better = higher score, ties to the smaller tie id (original id).
// --------------------------------------------------------------------------
struct __align__(16) Cand {
  double s;       // score
  uint32_t tie;   // original id (within this index; shards add id_offset later)
  uint32_t slot;  // layout slot
};

__host__ __device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  return a.s > b.s || (a.s == b.s && a.tie < b.tie);
}

__host__ __device__ __forceinline__ Cand worst_cand() {
  Cand c;
  c.s = -INFINITY;
  c.tie = 0xFFFFFFFFu;
  c.slot = 0xFFFFFFFFu;
  return c;
}

// --------------------------------------------------------------------------
// OpenBLAS dgemv_t dot recipe (re-derived here):
// 4 FMA lanes over blocks of 4, lanes combined (L0+L2)+(L1+L3); a tail of one
// element is FMA'd onto the base, a longer tail is summed as
// fma(x0,y0,x1*y1) (+ fma for a third) and then added.  Matches numpy's
// `A @ v` for row-major A in the dev container (adc_table dense.py:219,
// whiten_apply dense.py:355-357).  Bit-exactness to a given host's BLAS is
// checked by the golden tests, not assumed.
// --------------------------------------------------------------------------
template <typename TX, typename TY>
__host__ __device__ __forceinline__ double dot_recipe(const TX* x, const TY* y, int w,
                                                      int sx = 1, int sy = 1) {
  double L0 = 0.0, L1 = 0.0, L2 = 0.0, L3 = 0.0;
  const int m = w & ~3;
  for (int i = 0; i < m; i += 4) {
    L0 = fma((double)x[(i + 0) * sx], (double)y[(i + 0) * sy], L0);
    L1 = fma((double)x[(i + 1) * sx], (double)y[(i + 1) * sy], L1);
    L2 = fma((double)x[(i + 2) * sx], (double)y[(i + 2) * sy], L2);
    L3 = fma((double)x[(i + 3) * sx], (double)y[(i + 3) * sy], L3);
  }
  const double base = (L0 + L2) + (L1 + L3);
  const int rem = w - m;
  if (rem == 0) return base;
  if (rem == 1) {
    const double xy = (double)x[m * sx];
    return m ? fma(xy, (double)y[m * sy], base) : xy * (double)y[m * sy];
  }
  double p = fma((double)x[m * sx], (double)y[m * sy],
                 (double)x[(m + 1) * sx] * (double)y[(m + 1) * sy]);
  for (int k = m + 2; k < w; ++k) p = fma((double)x[k * sx], (double)y[k * sy], p);
  return m ? base + p : p;
}

// numpy pairwise summation (QuantizedLUT.bias_total, dense.py:243-245),
// starting from the additive identity like np.sum.
__host__ __device__ inline double pairwise_block(const double* a, int n) {
  if (n < 8) {
    double s = n ? a[0] : 0.0;
    for (int i = 1; i < n; ++i) s += a[i];
    return s;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 += a[i + 0]; r1 += a[i + 1]; r2 += a[i + 2]; r3 += a[i + 3];
    r4 += a[i + 4]; r5 += a[i + 5]; r6 += a[i + 6]; r7 += a[i + 7];
  }
  double s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) s += a[i];
  return s;
}

// Splits while n > 128 at n/2 rounded down to a multiple of 8 (depth is tiny
// for the K of a PQ codebook).  Returns 0.0 + sum so an all -0.0 row gives +0.0.
__host__ __device__ inline double pairwise_rec(const double* a, int n) {
  if (n <= 128) return pairwise_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_rec(a, n2) + pairwise_rec(a + n2, n - n2);
}

__host__ __device__ inline double pairwise_sum(const double* a, int n) {
  return 0.0 + pairwise_rec(a, n);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int next_pow2(int64_t x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// --------------------------------------------------------------------------
// block-wide bitonic sort of `n` (power of two) candidates in shared memory,
// best first.  All threads of the block must call it.
// --------------------------------------------------------------------------
// Order-preserving 64-bit key of an f64 score (-0.0 folded into +0.0: the
// reference compares them equal and breaks the tie by id).
__device__ __forceinline__ unsigned long long score_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x + 0.0);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Warp 0 helper: among 256 bins, walking bins in the given direction (desc =
// from 255 down), find the bin where the running count reaches `need`.
// Writes bin, the count still needed inside it, and the bin's size to ctl[12..14].
__device__ __forceinline__ void find_bin(const unsigned* hist, int need, bool desc, int* out) {
  const int lane = threadIdx.x & 31;
  unsigned c[8];
  unsigned tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int bin = desc ? 255 - (lane * 8 + j) : lane * 8 + j;
    c[j] = hist[bin];
    tot += c[j];
  }
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned excl = incl - tot;
  const bool here = excl < (unsigned)need && incl >= (unsigned)need;
  if (here) {
    unsigned run = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (run + c[j] >= (unsigned)need) {
        out[0] = desc ? 255 - (lane * 8 + j) : lane * 8 + j;
        out[1] = need - (int)run;
        out[2] = (int)c[j];
        break;
      }
      run += c[j];
    }
  }
}

__device__ __forceinline__ void bitonic_sort_block(Cand* a, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        Cand x = a[lo], y = a[hi];
        const bool sw = up ? better(y, x) : better(x, y);
        if (sw) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// In-register LUT16 (the GPU analogue of the paper's PSHUFB table,
// PAPER.md:374-397): eight 16-entry u8 lookups with PRMT.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

// w: nibble j = code of point j; T: the u8 table (entries 0..15 in the bytes
// of T.x..T.w).  r0 = table bytes of points 0-3, r1 = points 4-7.  PRMT
// selects among 8 bytes by the low 3 bits of a selector nibble (bit 3 set =
// sign-replicate: garbage here, blended away), so entries 0-7 and 8-15 are
// looked up separately and blended by a byte mask of the codes' bit 3.  The
// mask is itself one PRMT in sign-replicate mode: the msb of byte j of w is
// bit 3 of point 2j+1, the msb of byte j of w << 4 is bit 3 of point 2j.
__device__ __forceinline__ void lut8(const uint4& T, uint32_t w, uint32_t& r0, uint32_t& r1) {
  const uint32_t x = w ^ 0x88888888u;  // entries 8..15 become selectors 0..7
  const uint32_t a0 = prmt(T.x, T.y, w), a1 = prmt(T.x, T.y, w >> 16);
  const uint32_t b0 = prmt(T.z, T.w, x), b1 = prmt(T.z, T.w, x >> 16);
  const uint32_t w4 = w << 4;
  const uint32_t k0 = prmt(w, w4, 0x9D8Cu), k1 = prmt(w, w4, 0xBFAEu);
  r0 = (b0 & k0) | (a0 & ~k0);
  r1 = (b1 & k1) | (a1 & ~k1);
}

}  // namespace hs
