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

#include "common.cuh"

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
                 const float* __restrict__ centers, uint8_t* __restrict__ packed,
                 uint8_t* __restrict__ codes_pm, unsigned long long* __restrict__ lo_key,
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
        const double* row = vec + (ok ? order[i] : 0) * d;
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
            codes_pm[i * npairs + p] = byte;
          }
        }
      }
    }
    __syncthreads();
    const int live = (int)((n - base) < kTile ? (n - base) : kTile);
    for (int e = threadIdx.x; e < npairs * kTile; e += blockDim.x) {
      const int p = e / kTile, s = e % kTile;
      if (s < live) packed[(int64_t)p * n + base + s] = s_tile[e];
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
            const uint8_t* __restrict__ codes_pm, int npairs, const double* __restrict__ lo,
            const double* __restrict__ safe, uint8_t* __restrict__ sq) {
  constexpr int R = 4;  // rows in flight per CTA
  for (int64_t i0 = (int64_t)blockIdx.x * R; i0 < n; i0 += (int64_t)gridDim.x * R) {
    const double* rows[R];
    const uint8_t* crs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = i0 + r < n ? i0 + r : n - 1;
      rows[r] = vec + order[i] * d;
      crs[r] = codes_pm + i * npairs;
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
      kern<<<grid, kEncThreads, smem>>>(dvec, n, d, dord, K, t, dcen, dpk, dpm, dkeys, dkeys + d);
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
    k_sq_encode<<<blocks, threads>>>(dvec, n, d, dord, ddk, ddt, dw, dco, dcen, dpm, npairs, dlo,
                                     dsafe, dsq);
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
