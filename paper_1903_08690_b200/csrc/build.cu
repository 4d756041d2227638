// build.cu — GPU dense-part index build (dense slice):
// PQ encode + 4-bit pair-major pack + scalar-quantised residual, all in
// layout order, bit-identical to the reference's
//   codes = pq_encode(vectors, codebooks)[order]            pipeline.py:152, dense.py:138-153
//   PQCodes.from_codes -> pack_codes                         dense.py:156-170
//   sq_encode(vectors[order] - reconstruct(codes))           pipeline.py:154-157, dense.py:381-390
// (the arithmetic recipe is the host builder's, hostbuild.cpp hsb_pq_encode /
// hsb_sq_residual, which the golden build fixtures pin to the reference).
//
// Two HBM-bound kernels:
//   k_pq_encode_pack  persistent CTAs over tiles of 32 layout slots; a warp
//                     encodes a whole row order[i] (lane = subspace pair,
//                     contiguous loads), picks the nearest of the 16 centers
//                     per subspace in f64 (first minimum wins), stores the
//                     tile pair-major through a shared-memory transpose plus a
//                     point-major copy for the SQ pass, and keeps per-dim
//                     residual min/max in registers (ordered-key atomics once
//                     per CTA).
//   k_sq_encode       CTA per row, threads over dims: recomputes the residual
//                     from the point-major code and writes the u8 code.
// Bytes per point: 2*d*8 (vectors, read twice) + 3*ceil(K/2) + d.
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include <algorithm>
#include <chrono>
#include <memory>

#include "kernels.cuh"

namespace hs {
namespace {

constexpr int kEncThreads = 256;

// order-preserving map of a (non-NaN) double to u64, so that min/max over
// doubles is an integer atomicMin/atomicMax
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dunkey(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double x;
  memcpy(&x, &b, 8);
  return x;
#endif
}

struct SubTab {  // per-subspace geometry (device arrays)
  const int32_t* dim_off;   // [K]
  const int32_t* width;     // [K] 1 or 2
  const int32_t* cen_off;   // [K] float offset of centers[k]
};

constexpr int kTile = 32;  // layout slots per tile

// nearest of 16 centers for one subspace (hostbuild.cpp hsb_pq_encode recipe)
__device__ __forceinline__ int nearest(double x0, double x1, int w, const float2* c, int cs) {
  int best = 0;
  double bd = 0.0;
  if (w == 2) {
    const double sq = __dadd_rn(__dadd_rn(0.0, __dmul_rn(x0, x0)), __dmul_rn(x1, x1));
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 cf = c[j * cs];
      const double c0 = cf.x, c1 = cf.y;
      const double dot = __fma_rn(x1, c1, __dmul_rn(x0, c0));
      // |c|^2 as hsb_pq_encode: (0 + c0*c0) + c1*c1 (0 + v is exact)
      const double csq = __dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1));
      // 2*dot is exact, so fma(-2, dot, sq) == RN(sq - 2*dot)
      const double d2 = __dadd_rn(__fma_rn(-2.0, dot, sq), csq);
      if (j == 0 || d2 < bd) {
        bd = d2;
        best = j;
      }
    }
  } else {
    const double sq = __dadd_rn(0.0, __dmul_rn(x0, x0));
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double c0 = c[j * cs].x;
      const double dot = __dmul_rn(x0, c0);
      const double d2 = __dadd_rn(__fma_rn(-2.0, dot, sq), __dmul_rn(c0, c0));
      if (j == 0 || d2 < bd) {
        bd = d2;
        best = j;
      }
    }
  }
  return best;
}

// Persistent: a CTA walks tiles of kTile layout slots; each warp encodes whole
// rows (lane = subspace pair, so a warp's loads of one row are contiguous),
// the tile's codes are transposed in shared memory and stored pair-major
// (32 consecutive bytes per pair), and a point-major copy [n][npairs] feeds
// the SQ pass.  Residual min/max per dim stay in registers across tiles
// (lane-owned pairs), then shared-memory and global ordered-key atomics once
// per CTA.  M = ceil(npairs / 32).
template <int M>
__global__ void __launch_bounds__(kEncThreads)
k_pq_encode_pack(const double* __restrict__ vec, int64_t n, int64_t d,
                 const int64_t* __restrict__ order, int32_t K, SubTab t,
                 const float* __restrict__ centers, uint8_t* __restrict__ packed, int64_t ld,
                 uint8_t* __restrict__ codes_pm, int64_t prow,
                 unsigned long long* __restrict__ lo_key,
                 unsigned long long* __restrict__ hi_key) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int npairs = (K + 1) / 2;
  const int npad = 2 * ((K + 1) / 2);
  float2* s_c = reinterpret_cast<float2*>(smem);                         // [16][2][npairs]
  unsigned long long* s_lo = reinterpret_cast<unsigned long long*>(s_c + (size_t)npad * 16);  // [d]
  unsigned long long* s_hi = s_lo + d;                                   // [d]
  uint8_t* s_tile = reinterpret_cast<uint8_t*>(s_hi + d);                // [npairs][kTile]
  // f32 centers at [c][k & 1][k >> 1] (|c|^2 is recomputed in f64 from them):
  // the lanes of a warp (consecutive pairs) read consecutive entries, no bank
  // conflicts
  const int cstride = 2 * npairs;
  for (int e = threadIdx.x; e < K * 16; e += blockDim.x) {
    const int k = e >> 4, c = e & 15, w = t.width[k];
    const float* src = centers + t.cen_off[k] + c * w;
    const int at = c * cstride + (k & 1) * npairs + (k >> 1);
    s_c[at] = make_float2(src[0], w == 2 ? src[1] : 0.f);
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    s_lo[j] = ~0ull;
    s_hi[j] = 0ull;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double rmin[M][4], rmax[M][4];
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rmin[m][q] = INFINITY;
      rmax[m][q] = -INFINITY;
    }
  const int64_t ntiles = (n + kTile - 1) / kTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kTile;
    // S slots of this warp in flight: all their loads issue before the math
    constexpr int S = M >= 4 ? 1 : 4 / M;
    constexpr int kWarps = kEncThreads / 32;
    for (int s0 = warp; s0 < kTile; s0 += kWarps * S) {
      double xv[S][M][4];
#pragma unroll
      for (int u = 0; u < S; ++u) {
        const int64_t i = base + s0 + u * kWarps;
        const bool ok = s0 + u * kWarps < kTile && i < n;
        const double* row = vec + (ok ? (order ? order[i] : i) : 0) * d;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int p = lane + 32 * m;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * p + h;
            const bool live = ok && p < npairs && k < K;
            const int w = live ? t.width[k] : 1, off = live ? t.dim_off[k] : 0;
            xv[u][m][2 * h] = live ? row[off] : 0.0;
            xv[u][m][2 * h + 1] = live && w == 2 ? row[off + 1] : 0.0;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < S; ++u) {
        const int s = s0 + u * kWarps;
        const int64_t i = base + s;
        if (s >= kTile || i >= n) break;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int p = lane + 32 * m;
          if (p < npairs) {
            uint8_t byte = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k = 2 * p + h;
              if (k < K) {
                const int w = t.width[k];
                const double x0 = xv[u][m][2 * h], x1 = xv[u][m][2 * h + 1];
                const int at = h * npairs + p;
                const int c = nearest(x0, x1, w, s_c + at, cstride);
                byte |= (uint8_t)(c << (4 * h));
                const float2 cc = s_c[c * cstride + at];
                const double r0 = __dsub_rn(x0, (double)cc.x);
                rmin[m][2 * h] = fmin(rmin[m][2 * h], r0);
                rmax[m][2 * h] = fmax(rmax[m][2 * h], r0);
                if (w == 2) {
                  const double r1 = __dsub_rn(x1, (double)cc.y);
                  rmin[m][2 * h + 1] = fmin(rmin[m][2 * h + 1], r1);
                  rmax[m][2 * h + 1] = fmax(rmax[m][2 * h + 1], r1);
                }
              }
            }
            s_tile[p * kTile + s] = byte;
            codes_pm[i * prow + p] = byte;
          }
        }
      }
    }
    __syncthreads();
    const int live = (int)((n - base) < kTile ? (n - base) : kTile);
    for (int e = threadIdx.x; e < npairs * kTile; e += blockDim.x) {
      const int p = e / kTile, s = e % kTile;
      if (s < live) packed[(int64_t)p * ld + base + s] = s_tile[e];
    }
    __syncthreads();
  }
  // fold the lane-owned dims into shared memory, then once per CTA to global
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int p = lane + 32 * m;
    if (p >= npairs) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 2 * p + (q >> 1), tt = q & 1;
      if (k >= K || tt >= t.width[k] || !(rmin[m][q] <= rmax[m][q])) continue;
      const int dim = t.dim_off[k] + tt;
      atomicMin(s_lo + dim, dkey(rmin[m][q]));
      atomicMax(s_hi + dim, dkey(rmax[m][q]));
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    if (s_lo[j] != ~0ull) atomicMin(lo_key + j, s_lo[j]);
    if (s_hi[j] != 0ull) atomicMax(hi_key + j, s_hi[j]);
  }
}

// One CTA row at a time (grid-stride over layout slots), threads over dims:
// the row of vec and the slot's point-major codes are contiguous loads, the
// u8 output row a contiguous store.
__global__ void __launch_bounds__(256)
k_sq_encode(const double* __restrict__ vec, int64_t n, int64_t d,
            const int64_t* __restrict__ order, const int32_t* __restrict__ dim_k,
            const int32_t* __restrict__ dim_t, const int32_t* __restrict__ width,
            const int32_t* __restrict__ cen_off, const float* __restrict__ centers,
            const uint8_t* __restrict__ codes_pm, int64_t prow, const double* __restrict__ lo,
            const double* __restrict__ safe, uint8_t* __restrict__ sq) {
  constexpr int R = 4;  // rows in flight per CTA
  for (int64_t i0 = (int64_t)blockIdx.x * R; i0 < n; i0 += (int64_t)gridDim.x * R) {
    const double* rows[R];
    const uint8_t* crs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = i0 + r < n ? i0 + r : n - 1;
      rows[r] = vec + (order ? order[i] : i) * d;
      crs[r] = codes_pm + i * prow;
    }
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const int k = dim_k[j];
      const double l0 = lo[j], sf = safe[j], iv = 1.0 / sf;
      const float* cb = centers + cen_off[k] + dim_t[j];
      const int w = width[k];
      double x[R];
      int code[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[r] = rows[r][j];
        code[r] = (crs[r][k >> 1] >> (4 * (k & 1))) & 15;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (i0 + r >= n) break;
        const double res = __dsub_rn(x[r], (double)cb[code[r] * w]);
        // floor(RN(a / sf)) through the reciprocal when a*inv is not within
        // 1e-6 of an integer (|a*inv - RN(a/sf)| is a few ulp of a value
        // <= 256, far below that); the IEEE division otherwise
        const double a = __dsub_rn(res, l0);
        const double tq = a * iv;
        double q = floor(tq);
        const double fr = tq - q;
        if (!(fr > 1e-6 && fr < 1.0 - 1e-6)) q = floor(__ddiv_rn(a, sf));
        q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
        sq[(i0 + r) * d + j] = (uint8_t)q;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// GPU build from a resident dataset (hs_builder_*): dense rows as f64,
// optionally whitened, moments for whiten_fit
// ---------------------------------------------------------------------------
template <typename TIN>
__device__ __forceinline__ double dval(const TIN* p) { return (double)*p; }
template <>
__device__ __forceinline__ double dval<__half>(const __half* p) { return (double)__half2float(*p); }

__device__ __forceinline__ int64_t pick_row(const uint32_t* rows_u32, const int64_t* rows_i64,
                                            int64_t slot0, int64_t i) {
  return rows_u32 ? (int64_t)rows_u32[slot0 + i] : (rows_i64 ? rows_i64[i] : slot0 + i);
}

template <typename TIN>
__global__ void k_rows_f64(const TIN* __restrict__ src, int64_t d, const uint32_t* __restrict__ ru,
                           const int64_t* __restrict__ ri, int64_t slot0, int64_t m,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const TIN* row = src + pick_row(ru, ri, slot0, i) * d;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) out[i * d + j] = dval(row + j);
  }
}

// out[i][c] = sum_j fwd[c][j] * (x[row_i][j] - mean[j]), j ascending (one
// FMA chain per output; whiten_apply "data", dense.py:354).  64x64 output
// tiles, 16-wide k steps, 4x4 outputs per thread.
constexpr int kWB = 64, kWK = 16;
template <typename TIN>
__global__ void __launch_bounds__(256)
k_whiten_rows(const TIN* __restrict__ src, int64_t d, const uint32_t* __restrict__ ru,
              const int64_t* __restrict__ ri, int64_t slot0, int64_t m,
              const double* __restrict__ mean, const double* __restrict__ fwd,
              double* __restrict__ out) {
  __shared__ double As[kWK][kWB + 1];
  __shared__ double Bs[kWK][kWB + 1];
  __shared__ int64_t rowid[kWB];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * kWB;
  const int64_t c0 = (int64_t)blockIdx.y * kWB;
  if (threadIdx.x < kWB) {
    const int64_t i = r0 + threadIdx.x;
    rowid[threadIdx.x] = i < m ? pick_row(ru, ri, slot0, i) : -1;
  }
  __syncthreads();
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = 0; k0 < d; k0 += kWK) {
    for (int e = threadIdx.x; e < kWB * kWK; e += 256) {
      const int r = e / kWK, k = e % kWK;
      const int64_t j = k0 + k;
      const int64_t row = rowid[r];
      As[k][r] = (row >= 0 && j < d) ? __dsub_rn(dval(src + row * d + j), mean[j]) : 0.0;
      const int64_t c = c0 + r;
      Bs[k][r] = (c < d && j < d) ? fwd[c * d + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kWK; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[k][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[k][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = r0 + ty * 4 + a;
    if (i >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t c = c0 + tx * 4 + b;
      if (c < d) out[i * d + c] = acc[a][b];
    }
  }
}

// per-CTA column sums over a row range (sequential per thread, f64)
template <typename TIN>
__global__ void k_col_sums(const TIN* __restrict__ src, int64_t n, int64_t d, int64_t rows_per,
                           double* __restrict__ part) {
  const int64_t i0 = (int64_t)blockIdx.x * rows_per;
  const int64_t i1 = i0 + rows_per < n ? i0 + rows_per : n;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) s = __dadd_rn(s, dval(src + i * d + j));
    part[(int64_t)blockIdx.x * d + j] = s;
  }
}

// partial centred Gram tile (ta, tb) over a row chunk: 64x64 outputs
template <typename TIN>
__global__ void __launch_bounds__(256)
k_gram(const TIN* __restrict__ src, int64_t n, int64_t d, const double* __restrict__ mean,
       const int* __restrict__ pair_a, const int* __restrict__ pair_b, int64_t rows_per,
       double* __restrict__ part) {
  __shared__ double Xa[kWK][kWB + 1];
  __shared__ double Xb[kWK][kWB + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int pr = blockIdx.x;
  const int64_t a0 = (int64_t)pair_a[pr] * kWB, b0 = (int64_t)pair_b[pr] * kWB;
  const int64_t i0 = (int64_t)blockIdx.y * rows_per;
  const int64_t i1 = i0 + rows_per < n ? i0 + rows_per : n;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t r0 = i0; r0 < i1; r0 += kWK) {
    for (int e = threadIdx.x; e < kWB * kWK; e += 256) {
      const int k = e / kWB, c = e % kWB;
      const int64_t i = r0 + k;
      const int64_t ja = a0 + c, jb = b0 + c;
      Xa[k][c] = (i < i1 && ja < d) ? __dsub_rn(dval(src + i * d + ja), mean[ja]) : 0.0;
      Xb[k][c] = (i < i1 && jb < d) ? __dsub_rn(dval(src + i * d + jb), mean[jb]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kWK; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = Xa[k][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Xb[k][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  double* out = part + ((int64_t)blockIdx.y * gridDim.x + pr) * kWB * kWB;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) out[(ty * 4 + a) * kWB + tx * 4 + b] = acc[a][b];
}

// sum the chunk partials (chunk order) into the full symmetric matrix
__global__ void k_gram_reduce(const double* __restrict__ part, int npairs_t, int nchunks,
                              const int* __restrict__ pair_a, const int* __restrict__ pair_b,
                              int64_t d, double* __restrict__ cov) {
  const int pr = blockIdx.x;
  for (int e = threadIdx.x; e < kWB * kWB; e += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s = __dadd_rn(s, part[((int64_t)c * npairs_t + pr) * kWB * kWB + e]);
    const int64_t i = (int64_t)pair_a[pr] * kWB + e / kWB, j = (int64_t)pair_b[pr] * kWB + e % kWB;
    if (i < d && j < d) {
      cov[i * d + j] = s;
      cov[j * d + i] = s;
    }
  }
}

struct DBufs {  // frees everything on scope exit
  std::vector<void*> ptrs;
  ~DBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  template <class T>
  cudaError_t upload(T** p, const T* h, size_t count) {
    cudaError_t e = alloc(p, count);
    if (e == cudaSuccess && count) e = cudaMemcpy(*p, h, sizeof(T) * count, cudaMemcpyHostToDevice);
    return e;
  }
};

}  // namespace
}  // namespace hs

using namespace hs;

extern "C" int hs_dense_encode(const double* vec, int64_t n, int64_t d, const int64_t* order,
                               int32_t K, const int64_t* subdims, const float* centers, int32_t l,
                               uint8_t* packed, float* sq_lo, float* sq_step, uint8_t* sq_codes,
                               int device, double* seconds) {
  if (n < 0 || d <= 0 || K <= 0 || !vec || !order || !subdims || !centers || !packed)
    HS_FAIL(HS_EINVAL, "hs_dense_encode: bad arguments");
  if (l != 16) HS_FAIL(HS_EUNSUPPORTED, "hs_dense_encode: only 16-center (4-bit) codebooks");
  std::vector<int32_t> dim_off(K), width(K), cen_off(K), dim_k(d), dim_t(d);
  int64_t o = 0, co = 0;
  for (int32_t k = 0; k < K; ++k) {
    if (subdims[k] < 1 || subdims[k] > 2)
      HS_FAIL(HS_EUNSUPPORTED, "hs_dense_encode: subspaces wider than 2 dims");
    dim_off[k] = (int32_t)o;
    width[k] = (int32_t)subdims[k];
    cen_off[k] = (int32_t)co;
    for (int64_t t = 0; t < subdims[k]; ++t) {
      if (o + t >= d) HS_FAIL(HS_EINVAL, "hs_dense_encode: subdims exceed d");
      dim_k[o + t] = k;
      dim_t[o + t] = (int32_t)t;
    }
    o += subdims[k];
    co += subdims[k] * 16;
  }
  if (o != d) HS_FAIL(HS_EINVAL, "hs_dense_encode: subdims do not cover d");
  HS_CUDA(cudaSetDevice(device));
  const int npairs = (K + 1) / 2;
  DBufs b;
  double *dvec, *dlo, *dsafe;
  int64_t* dord;
  int32_t *ddo, *dw, *dco, *ddk, *ddt;
  float* dcen;
  uint8_t *dpk, *dpm, *dsq = nullptr;
  unsigned long long* dkeys;
  HS_CUDA(b.upload(&dvec, vec, (size_t)(n * d)));
  HS_CUDA(b.upload(&dord, order, (size_t)n));
  HS_CUDA(b.upload(&ddo, dim_off.data(), K));
  HS_CUDA(b.upload(&dw, width.data(), K));
  HS_CUDA(b.upload(&dco, cen_off.data(), K));
  HS_CUDA(b.upload(&ddk, dim_k.data(), (size_t)d));
  HS_CUDA(b.upload(&ddt, dim_t.data(), (size_t)d));
  HS_CUDA(b.upload(&dcen, centers, (size_t)co));
  HS_CUDA(b.alloc(&dpk, (size_t)(npairs * n)));
  HS_CUDA(b.alloc(&dpm, (size_t)(npairs * n)));
  HS_CUDA(b.alloc(&dkeys, (size_t)(2 * d)));
  HS_CUDA(b.alloc(&dlo, (size_t)d));
  HS_CUDA(b.alloc(&dsafe, (size_t)d));
  HS_CUDA(cudaMemset(dkeys, 0xff, sizeof(unsigned long long) * d));  // lo: max key
  HS_CUDA(cudaMemset(dkeys + d, 0x00, sizeof(unsigned long long) * d));  // hi: min key
  if (sq_codes) HS_CUDA(b.alloc(&dsq, (size_t)(n * d)));
  cudaEvent_t e0, e1;
  HS_CUDA(cudaEventCreate(&e0));
  HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaEventRecord(e0));
  if (n > 0) {
    SubTab t{ddo, dw, dco};
    const size_t smem = (size_t)(2 * npairs) * 16 * sizeof(float2) +
                        2 * sizeof(unsigned long long) * (size_t)d + (size_t)npairs * kTile;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const unsigned grid = (unsigned)(ntiles < kNumSMs * 4 ? ntiles : kNumSMs * 4);
    const int M = (npairs + 31) / 32;
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<grid, kEncThreads, smem>>>(dvec, n, d, dord, K, t, dcen, dpk, n, dpm, npairs, dkeys,
                                        dkeys + d);
      return cudaGetLastError();
    };
    if (smem > 200 * 1024) HS_FAIL(HS_EUNSUPPORTED, "hs_dense_encode: too many subspaces");
    if (M <= 1) HS_CUDA(go(k_pq_encode_pack<1>));
    else if (M <= 2) HS_CUDA(go(k_pq_encode_pack<2>));
    else if (M <= 4) HS_CUDA(go(k_pq_encode_pack<4>));
    else if (M <= 8) HS_CUDA(go(k_pq_encode_pack<8>));
    else HS_FAIL(HS_EUNSUPPORTED, "hs_dense_encode: more than 512 subspaces");
  }
  std::vector<double> lo(d), step(d), safe(d);
  if (sq_codes || sq_lo || sq_step) {
    std::vector<unsigned long long> keys(2 * d);
    HS_CUDA(cudaMemcpy(keys.data(), dkeys, sizeof(unsigned long long) * 2 * d,
                       cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < d; ++j) {  // hostbuild.cpp hsb_sq_residual
      double a = dunkey(keys[j]), z = dunkey(keys[d + j]);
      if (n == 0) a = z = 0.0;
      lo[j] = a;
      step[j] = (z - a) / 256.0;
      safe[j] = step[j] > 0 ? step[j] : 1.0;
      if (sq_lo) sq_lo[j] = (float)lo[j];
      if (sq_step) sq_step[j] = (float)step[j];
    }
  }
  if (sq_codes && n > 0) {
    HS_CUDA(cudaMemcpy(dlo, lo.data(), sizeof(double) * d, cudaMemcpyHostToDevice));
    HS_CUDA(cudaMemcpy(dsafe, safe.data(), sizeof(double) * d, cudaMemcpyHostToDevice));
    const int threads = d >= 256 ? 256 : (int)((d + 31) / 32 * 32);
    const int64_t rows4 = (n + 3) / 4;
    const unsigned blocks = (unsigned)(rows4 < kNumSMs * 16 ? rows4 : kNumSMs * 16);
    k_sq_encode<<<blocks, threads>>>(dvec, n, d, dord, ddk, ddt, dw, dco, dcen, dpm,
                                     (int64_t)npairs, dlo, dsafe, dsq);
    HS_CUDA(cudaGetLastError());
  }
  HS_CUDA(cudaEventRecord(e1));
  HS_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (seconds) *seconds = ms * 1e-3;
  HS_CUDA(cudaMemcpy(packed, dpk, (size_t)(npairs * n), cudaMemcpyDeviceToHost));
  if (sq_codes && n > 0) HS_CUDA(cudaMemcpy(sq_codes, dsq, (size_t)(n * d), cudaMemcpyDeviceToHost));
  return HS_OK;
}

// ---------------------------------------------------------------------------
// dense half of the GPU build from a resident dataset (hs_builder_*)
// ---------------------------------------------------------------------------
namespace hs {

int launch_dense_rows(const Builder& b, const uint32_t* rows_u32, const int64_t* rows_i64,
                      int64_t slot0, int64_t m, const double* mean, const double* fwd,
                      double* out, cudaStream_t st) {
  if (m <= 0) return HS_OK;
  const int64_t d = b.d_dense;
  if (fwd) {
    dim3 grid((unsigned)ceil_div(m, kWB), (unsigned)ceil_div(d, kWB));
    if (b.dense_fp16)
      k_whiten_rows<__half><<<grid, 256, 0, st>>>(b.dense_h, d, rows_u32, rows_i64, slot0, m, mean, fwd, out);
    else
      k_whiten_rows<float><<<grid, 256, 0, st>>>(b.dense, d, rows_u32, rows_i64, slot0, m, mean, fwd, out);
  } else {
    const unsigned grid = (unsigned)std::min<int64_t>(m, (int64_t)kNumSMs * 32);
    if (b.dense_fp16)
      k_rows_f64<__half><<<grid, 256, 0, st>>>(b.dense_h, d, rows_u32, rows_i64, slot0, m, out);
    else
      k_rows_f64<float><<<grid, 256, 0, st>>>(b.dense, d, rows_u32, rows_i64, slot0, m, out);
  }
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace hs

struct hs_builder : public hs::Builder {};

namespace {
double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

int hs_builder_dense_moments(hs_builder_t bp, double* mean, double* cov) {
  if (!bp || !mean) HS_FAIL(HS_EINVAL, "null argument");
  Builder& b = *bp;
  const int64_t n = b.n, d = b.d_dense;
  if (d <= 0) HS_FAIL(HS_EINVAL, "dataset has no dense part");
  HS_CUDA(cudaSetDevice(b.device));
  const auto t0 = std::chrono::steady_clock::now();
  DBufs buf;
  // column means: per-CTA sequential sums, CTAs summed in order on the host
  const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)kNumSMs * 8));
  const int64_t rows_per = std::max<int64_t>(1, ceil_div(n, nblk));
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, rows_per));
  double* part;
  HS_CUDA(buf.alloc(&part, (size_t)(nb * d)));
  const int th = d >= 256 ? 256 : (int)((d + 31) / 32 * 32);
  if (n > 0) {
    if (b.dense_fp16) k_col_sums<__half><<<(unsigned)nb, th, 0, b.st>>>(b.dense_h, n, d, rows_per, part);
    else k_col_sums<float><<<(unsigned)nb, th, 0, b.st>>>(b.dense, n, d, rows_per, part);
  }
  std::vector<double> hp((size_t)(nb * d), 0.0);
  if (n > 0) HS_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * nb * d, cudaMemcpyDeviceToHost, b.st));
  HS_CUDA(cudaStreamSynchronize(b.st));
  for (int64_t j = 0; j < d; ++j) {
    double sacc = 0.0;
    for (int64_t c = 0; c < nb; ++c) sacc += hp[(size_t)(c * d + j)];
    mean[j] = n > 0 ? sacc / (double)n : 0.0;
  }
  if (cov) {
    double* dmean;
    HS_CUDA(buf.upload(&dmean, mean, (size_t)d));
    const int nt = (int)ceil_div(d, kWB);
    std::vector<int> pa, pb;
    for (int a = 0; a < nt; ++a)
      for (int c = a; c < nt; ++c) {
        pa.push_back(a);
        pb.push_back(c);
      }
    const int np = (int)pa.size();
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 4096), ceil_div((int64_t)kNumSMs * 4, np)));
    const int64_t rp = std::max<int64_t>(1, ceil_div(n, nchunks));
    int *dpa, *dpb;
    double *gpart, *dcov;
    HS_CUDA(buf.upload(&dpa, pa.data(), pa.size()));
    HS_CUDA(buf.upload(&dpb, pb.data(), pb.size()));
    HS_CUDA(buf.alloc(&gpart, (size_t)(nchunks * np) * kWB * kWB));
    HS_CUDA(buf.alloc(&dcov, (size_t)(d * d)));
    dim3 grid((unsigned)np, (unsigned)nchunks);
    if (b.dense_fp16) k_gram<__half><<<grid, 256, 0, b.st>>>(b.dense_h, n, d, dmean, dpa, dpb, rp, gpart);
    else k_gram<float><<<grid, 256, 0, b.st>>>(b.dense, n, d, dmean, dpa, dpb, rp, gpart);
    k_gram_reduce<<<np, 256, 0, b.st>>>(gpart, np, (int)nchunks, dpa, dpb, d, dcov);
    HS_CUDA(cudaGetLastError());
    HS_CUDA(cudaMemcpyAsync(cov, dcov, sizeof(double) * d * d, cudaMemcpyDeviceToHost, b.st));
    HS_CUDA(cudaStreamSynchronize(b.st));
    for (int64_t i = 0; i < d * d; ++i) cov[i] = n > 0 ? cov[i] / (double)n : 0.0;
  }
  builder_phase(b, "dense_moments", since(t0));
  return HS_OK;
}

int hs_builder_gather_dense(hs_builder_t bp, const int64_t* rows, int64_t m, const double* mean,
                            const double* fwd, double* out) {
  if (!bp || (!rows && m > 0) || !out) HS_FAIL(HS_EINVAL, "null argument");
  Builder& b = *bp;
  const int64_t d = b.d_dense;
  if (d <= 0) HS_FAIL(HS_EINVAL, "dataset has no dense part");
  for (int64_t i = 0; i < m; ++i)
    if (rows[i] < 0 || rows[i] >= b.n) HS_FAIL(HS_EINVAL, "sample row out of range");
  if (fwd && !mean) HS_FAIL(HS_EINVAL, "whitening needs the mean");
  HS_CUDA(cudaSetDevice(b.device));
  DBufs buf;
  int64_t* dr;
  double *dm = nullptr, *df = nullptr, *dout;
  HS_CUDA(buf.upload(&dr, rows, (size_t)m));
  if (fwd) {
    HS_CUDA(buf.upload(&dm, mean, (size_t)d));
    HS_CUDA(buf.upload(&df, fwd, (size_t)(d * d)));
  }
  HS_CUDA(buf.alloc(&dout, (size_t)(m * d)));
  HS_CHECK(launch_dense_rows(b, nullptr, dr, 0, m, dm, df, dout, b.st));
  if (m) HS_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * m * d, cudaMemcpyDeviceToHost, b.st));
  HS_CUDA(cudaStreamSynchronize(b.st));
  return HS_OK;
}

int hs_builder_dense_encode(hs_builder_t bp, int32_t K, const int32_t* subdims,
                            const float* centers, int32_t l, const double* wh_mean,
                            const double* wh_fwd, const double* wh_inverse_t) {
  if (!bp || K <= 0 || !subdims || !centers) HS_FAIL(HS_EINVAL, "bad arguments");
  Builder& b = *bp;
  const int64_t n = b.n, d = b.d_dense;
  if (d <= 0) HS_FAIL(HS_EINVAL, "dataset has no dense part");
  if (!b.sparse_done) HS_FAIL(HS_EINVAL, "build the sparse part (layout order) first");
  if (b.dense_done) HS_FAIL(HS_EINVAL, "dense part already built");
  if (l != 16) HS_FAIL(HS_EUNSUPPORTED, "GPU dense build: only 16-center (4-bit) codebooks");
  if ((wh_fwd != nullptr) != (wh_mean != nullptr) || (wh_fwd != nullptr) != (wh_inverse_t != nullptr))
    HS_FAIL(HS_EINVAL, "whitening needs mean, forward and inverse_t");
  std::vector<int32_t> dim_off(K), width(K), cen_off(K), dim_k(d), dim_t(d);
  int64_t o = 0, co = 0;
  for (int32_t k = 0; k < K; ++k) {
    if (subdims[k] < 1 || subdims[k] > 2)
      HS_FAIL(HS_EUNSUPPORTED, "GPU dense build: subspaces wider than 2 dims");
    dim_off[k] = (int32_t)o;
    width[k] = subdims[k];
    cen_off[k] = (int32_t)co;
    for (int32_t t = 0; t < subdims[k]; ++t) {
      if (o + t >= d) HS_FAIL(HS_EINVAL, "subdims exceed d");
      dim_k[o + t] = k;
      dim_t[o + t] = t;
    }
    o += subdims[k];
    co += (int64_t)subdims[k] * 16;
  }
  if (o != d) HS_FAIL(HS_EINVAL, "subdims do not cover d");
  HS_CUDA(cudaSetDevice(b.device));
  const auto t0 = std::chrono::steady_clock::now();
  const int npairs = (K + 1) / 2;
  const int64_t prow = pcodes_row(npairs);
  DBufs buf;
  int32_t *ddo, *dw, *dco, *ddk, *ddt;
  float* dcen;
  double *dmean = nullptr, *dfwd = nullptr, *dvec, *dlo, *dsafe;
  unsigned long long* dkeys;
  HS_CUDA(buf.upload(&ddo, dim_off.data(), K));
  HS_CUDA(buf.upload(&dw, width.data(), K));
  HS_CUDA(buf.upload(&dco, cen_off.data(), K));
  HS_CUDA(buf.upload(&ddk, dim_k.data(), (size_t)d));
  HS_CUDA(buf.upload(&ddt, dim_t.data(), (size_t)d));
  HS_CUDA(buf.upload(&dcen, centers, (size_t)co));
  if (wh_fwd) {
    HS_CUDA(buf.upload(&dmean, wh_mean, (size_t)d));
    HS_CUDA(buf.upload(&dfwd, wh_fwd, (size_t)(d * d)));
  }
  const int64_t C = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)1 << 20));
  HS_CUDA(buf.alloc(&dvec, (size_t)(C * d)));
  HS_CUDA(buf.alloc(&dkeys, (size_t)(2 * d)));
  HS_CUDA(buf.alloc(&dlo, (size_t)d));
  HS_CUDA(buf.alloc(&dsafe, (size_t)d));
  HS_CUDA(cudaMemsetAsync(dkeys, 0xff, sizeof(unsigned long long) * d, b.st));
  HS_CUDA(cudaMemsetAsync(dkeys + d, 0x00, sizeof(unsigned long long) * d, b.st));
  HS_CUDA(cudaMalloc(&b.packed, std::max<size_t>((size_t)npairs * n, 1)));
  HS_CUDA(cudaMalloc(&b.pcodes, std::max<size_t>((size_t)prow * n, 1)));
  HS_CUDA(cudaMalloc(&b.sq, std::max<size_t>((size_t)n * d, 1)));
  if (prow > npairs && n > 0) HS_CUDA(cudaMemsetAsync(b.pcodes, 0, (size_t)prow * n, b.st));
  SubTab t{ddo, dw, dco};
  const size_t smem = (size_t)(2 * npairs) * 16 * sizeof(float2) +
                      2 * sizeof(unsigned long long) * (size_t)d + (size_t)npairs * kTile;
  if (smem > 200 * 1024) HS_FAIL(HS_EUNSUPPORTED, "GPU dense build: too many subspaces");
  const int M = (npairs + 31) / 32;
  if (M > 8) HS_FAIL(HS_EUNSUPPORTED, "GPU dense build: more than 512 subspaces");
  // pass 1: PQ codes (pair-major + point-major) and residual min/max
  for (int64_t s0 = 0; s0 < n; s0 += C) {
    const int64_t c = std::min(C, n - s0);
    HS_CHECK(launch_dense_rows(b, b.order, nullptr, s0, c, dmean, dfwd, dvec, b.st));
    const int64_t ntiles = (c + kTile - 1) / kTile;
    const unsigned grid = (unsigned)(ntiles < kNumSMs * 4 ? ntiles : kNumSMs * 4);
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<grid, kEncThreads, smem, b.st>>>(dvec, c, d, nullptr, K, t, dcen, b.packed + s0, n,
                                              b.pcodes + s0 * prow, prow, dkeys, dkeys + d);
      return cudaGetLastError();
    };
    if (M <= 1) HS_CUDA(go(k_pq_encode_pack<1>));
    else if (M <= 2) HS_CUDA(go(k_pq_encode_pack<2>));
    else if (M <= 4) HS_CUDA(go(k_pq_encode_pack<4>));
    else HS_CUDA(go(k_pq_encode_pack<8>));
  }
  // sq_encode's lo / step (hostbuild.cpp hsb_sq_residual recipe)
  std::vector<unsigned long long> keys(2 * d);
  HS_CUDA(cudaMemcpyAsync(keys.data(), dkeys, sizeof(unsigned long long) * 2 * d,
                          cudaMemcpyDeviceToHost, b.st));
  HS_CUDA(cudaStreamSynchronize(b.st));
  std::vector<double> lo(d), safe(d);
  b.sq_lo.assign(d, 0.f);
  b.sq_step.assign(d, 0.f);
  for (int64_t j = 0; j < d; ++j) {
    double a = dunkey(keys[j]), z = dunkey(keys[d + j]);
    if (n == 0) a = z = 0.0;
    lo[j] = a;
    const double step = (z - a) / 256.0;
    safe[j] = step > 0 ? step : 1.0;
    b.sq_lo[j] = (float)a;
    b.sq_step[j] = (float)step;
  }
  HS_CUDA(cudaMemcpyAsync(dlo, lo.data(), sizeof(double) * d, cudaMemcpyHostToDevice, b.st));
  HS_CUDA(cudaMemcpyAsync(dsafe, safe.data(), sizeof(double) * d, cudaMemcpyHostToDevice, b.st));
  // pass 2: SQ codes of the residual (rows recomputed)
  const int threads = d >= 256 ? 256 : (int)((d + 31) / 32 * 32);
  for (int64_t s0 = 0; s0 < n; s0 += C) {
    const int64_t c = std::min(C, n - s0);
    HS_CHECK(launch_dense_rows(b, b.order, nullptr, s0, c, dmean, dfwd, dvec, b.st));
    const int64_t rows4 = (c + 3) / 4;
    const unsigned blocks = (unsigned)(rows4 < kNumSMs * 16 ? rows4 : kNumSMs * 16);
    k_sq_encode<<<blocks, threads, 0, b.st>>>(dvec, c, d, nullptr, ddk, ddt, dw, dco, dcen,
                                              b.pcodes + s0 * prow, prow, dlo, dsafe, b.sq + s0 * d);
    HS_CUDA(cudaGetLastError());
  }
  HS_CUDA(cudaStreamSynchronize(b.st));
  b.K = K;
  b.l = l;
  b.subdims.assign(subdims, subdims + K);
  b.centers.assign(centers, centers + co);
  b.has_wh = wh_fwd ? 1 : 0;
  if (wh_fwd) {
    b.wh_mean.assign(wh_mean, wh_mean + d);
    b.wh_inv_t.assign(wh_inverse_t, wh_inverse_t + d * d);
  }
  b.dense_done = 1;
  builder_phase(b, "dense_encode", since(t0));
  return HS_OK;
}

int hs_builder_download_dense(hs_builder_t bp, uint8_t* packed, float* sq_lo, float* sq_step,
                              uint8_t* sq_codes) {
  if (!bp) HS_FAIL(HS_EINVAL, "null builder");
  Builder& b = *bp;
  if (!b.dense_done) HS_FAIL(HS_EINVAL, "dense part not built");
  HS_CUDA(cudaSetDevice(b.device));
  const int64_t n = b.n, d = b.d_dense;
  if (packed && n) HS_CUDA(cudaMemcpy(packed, b.packed, (size_t)((b.K + 1) / 2) * n, cudaMemcpyDeviceToHost));
  if (sq_lo) std::copy(b.sq_lo.begin(), b.sq_lo.end(), sq_lo);
  if (sq_step) std::copy(b.sq_step.begin(), b.sq_step.end(), sq_step);
  if (sq_codes && n) HS_CUDA(cudaMemcpy(sq_codes, b.sq, (size_t)n * d, cudaMemcpyDeviceToHost));
  return HS_OK;
}

}  // extern "C"
