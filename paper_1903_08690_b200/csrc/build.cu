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
//   k_pq_encode_pack  grid (slot chunks, subspace pairs): one thread per
//                     (layout slot, pair) reads the pair's <= 4 f64 values of
//                     row order[i] (one 32-byte sector), picks the nearest of
//                     the 16 centers per subspace in f64 (first minimum wins),
//                     writes the packed byte (coalesced along slots) and folds
//                     the residuals into per-dimension min/max (block
//                     reduction, then one ordered-key atomic per dim).
//   k_sq_encode       one thread per (slot, dim), dims fastest: recomputes the
//                     residual from the packed nibble and writes the u8 code.
// Bytes per point: d*8 (vectors, read twice) + ceil(K/2) + d (codes out).
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
  const double* csq;        // [K][16] |c|^2 in the host recipe
};

__global__ void __launch_bounds__(kEncThreads)
k_pq_encode_pack(const double* __restrict__ vec, int64_t n, int64_t d,
                 const int64_t* __restrict__ order, int32_t K, SubTab t,
                 const float* __restrict__ centers, uint8_t* __restrict__ packed,
                 unsigned long long* __restrict__ lo_key, unsigned long long* __restrict__ hi_key) {
  const int p = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * kEncThreads + threadIdx.x;
  __shared__ float s_c[2][16][2];
  __shared__ double s_csq[2][16];
  __shared__ double s_red[2][4][kEncThreads / 32];  // [min|max][dim][warp]
  int ks[2] = {2 * p, 2 * p + 1};
  const int nk = (2 * p + 1 < K) ? 2 : 1;
  for (int e = threadIdx.x; e < nk * 16; e += blockDim.x) {
    const int s = e >> 4, c = e & 15, k = ks[s], w = t.width[k];
    s_c[s][c][0] = centers[t.cen_off[k] + c * w];
    s_c[s][c][1] = w == 2 ? centers[t.cen_off[k] + c * w + 1] : 0.f;
    s_csq[s][c] = t.csq[k * 16 + c];
  }
  __syncthreads();
  const bool live = i < n;
  double rmin[4], rmax[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    rmin[q] = INFINITY;
    rmax[q] = -INFINITY;
  }
  uint8_t byte = 0;
  if (live) {
    const double* row = vec + order[i] * d;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s < nk) {
        const int k = ks[s], w = t.width[k];
        const double x0 = row[t.dim_off[k]];
        const double x1 = w == 2 ? row[t.dim_off[k] + 1] : 0.0;
        int best = 0;
        double bd = 0.0;
        if (w == 2) {
          const double sq = __dadd_rn(__dadd_rn(0.0, __dmul_rn(x0, x0)), __dmul_rn(x1, x1));
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const double dot = __fma_rn(x1, (double)s_c[s][c][1], __dmul_rn(x0, (double)s_c[s][c][0]));
            const double d2 = __dadd_rn(__dsub_rn(sq, __dmul_rn(2.0, dot)), s_csq[s][c]);
            if (c == 0 || d2 < bd) {
              bd = d2;
              best = c;
            }
          }
        } else {
          const double sq = __dadd_rn(0.0, __dmul_rn(x0, x0));
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const double dot = __dmul_rn(x0, (double)s_c[s][c][0]);
            const double d2 = __dadd_rn(__dsub_rn(sq, __dmul_rn(2.0, dot)), s_csq[s][c]);
            if (c == 0 || d2 < bd) {
              bd = d2;
              best = c;
            }
          }
        }
        byte |= (uint8_t)(best << (4 * s));
        const double r0 = __dsub_rn(x0, (double)s_c[s][best][0]);
        rmin[2 * s] = rmax[2 * s] = r0;
        if (w == 2) {
          const double r1 = __dsub_rn(x1, (double)s_c[s][best][1]);
          rmin[2 * s + 1] = rmax[2 * s + 1] = r1;
        }
      }
    }
    packed[(int64_t)p * n + i] = byte;
  }
  // block min/max per dim of this pair (<= 4 dims)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double a = rmin[q], b = rmax[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      s_red[0][q][warp] = a;
      s_red[1][q][warp] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int q = threadIdx.x & 3, mx = threadIdx.x >> 2;
    const int s = q >> 1, tt = q & 1;
    if (s < nk && tt < t.width[ks[s]]) {
      double v = s_red[mx][q][0];
      for (int w = 1; w < kEncThreads / 32; ++w)
        v = mx ? fmax(v, s_red[mx][q][w]) : fmin(v, s_red[mx][q][w]);
      if (isfinite(v)) {
        const int dim = t.dim_off[ks[s]] + tt;
        if (mx) atomicMax(hi_key + dim, dkey(v));
        else atomicMin(lo_key + dim, dkey(v));
      }
    }
  }
}

__global__ void k_sq_encode(const double* __restrict__ vec, int64_t n, int64_t d,
                            const int64_t* __restrict__ order, const int32_t* __restrict__ dim_k,
                            const int32_t* __restrict__ dim_t, const int32_t* __restrict__ width,
                            const int32_t* __restrict__ cen_off, const float* __restrict__ centers,
                            const uint8_t* __restrict__ packed, const double* __restrict__ lo,
                            const double* __restrict__ safe, uint8_t* __restrict__ sq) {
  const int64_t total = n * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int j = (int)(e - i * d);
    const int k = dim_k[j];
    const int code = (packed[(int64_t)(k >> 1) * n + i] >> (4 * (k & 1))) & 15;
    const double r = __dsub_rn(vec[order[i] * d + j],
                               (double)centers[cen_off[k] + code * width[k] + dim_t[j]]);
    double q = floor(__ddiv_rn(__dsub_rn(r, lo[j]), safe[j]));
    q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
    sq[e] = (uint8_t)q;
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
  std::vector<double> csq((size_t)K * 16);
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
    for (int c = 0; c < 16; ++c) {  // hostbuild.cpp hsb_pq_encode's |c|^2
      double s = 0.0;
      for (int64_t t = 0; t < subdims[k]; ++t) {
        const double v = (double)centers[co + c * subdims[k] + t];
        s = s + v * v;
      }
      csq[(size_t)k * 16 + c] = s;
    }
    o += subdims[k];
    co += subdims[k] * 16;
  }
  if (o != d) HS_FAIL(HS_EINVAL, "hs_dense_encode: subdims do not cover d");
  HS_CUDA(cudaSetDevice(device));
  const int npairs = (K + 1) / 2;
  DBufs b;
  double *dvec, *dcsq, *dlo, *dsafe;
  int64_t* dord;
  int32_t *ddo, *dw, *dco, *ddk, *ddt;
  float* dcen;
  uint8_t *dpk, *dsq = nullptr;
  unsigned long long* dkeys;
  HS_CUDA(b.upload(&dvec, vec, (size_t)(n * d)));
  HS_CUDA(b.upload(&dord, order, (size_t)n));
  HS_CUDA(b.upload(&ddo, dim_off.data(), K));
  HS_CUDA(b.upload(&dw, width.data(), K));
  HS_CUDA(b.upload(&dco, cen_off.data(), K));
  HS_CUDA(b.upload(&ddk, dim_k.data(), (size_t)d));
  HS_CUDA(b.upload(&ddt, dim_t.data(), (size_t)d));
  HS_CUDA(b.upload(&dcsq, csq.data(), csq.size()));
  HS_CUDA(b.upload(&dcen, centers, (size_t)co));
  HS_CUDA(b.alloc(&dpk, (size_t)(npairs * n)));
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
    SubTab t{ddo, dw, dco, dcsq};
    dim3 grid((unsigned)((n + kEncThreads - 1) / kEncThreads), (unsigned)npairs);
    k_pq_encode_pack<<<grid, kEncThreads>>>(dvec, n, d, dord, K, t, dcen, dpk, dkeys, dkeys + d);
    HS_CUDA(cudaGetLastError());
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
    const int64_t total = n * d;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    const unsigned blocks = (unsigned)(want < kNumSMs * 32 ? want : kNumSMs * 32);
    k_sq_encode<<<blocks, threads>>>(dvec, n, d, dord, ddk, ddt, dw, dco, dcen, dpk, dlo, dsafe, dsq);
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
