// lut.cu — K1: per-query LUT build.
//
// Replaces _dense_query + adc_table + quantize_lut (reference
// pipeline.py:206-223, dense.py:212-260, dense.py:351-357).  One CTA per
// query: weighted f64 query, whitening GEMV, ADC table in f64 with the BLAS
// dot recipe, per-row min bias, shared scale, round-half-even u8 table and
// the numpy-pairwise bias_total.  Arithmetic is IEEE double with explicit
// rounding where the reference does not contract (see common.cuh).
#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kLutThreads = 256;

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? red[lane] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// Shared quantisation of a K x l f64 table held in shared memory
// (dense.py:248-260): bias = row min, spread = max(T - bias),
// scale = spread / 255, q = clip(rint((T - bias) / scale), 0, 255).
__device__ void quantize_rows(const double* T, int K, int l, int Kp, double* bias_s,
                              double* red, uint8_t* table_out, double* bias_out,
                              double* scale_out, double* bias_total_out, int* bad_out) {
  const int tid = threadIdx.x;
  int nonfinite = 0;
  for (int i = tid; i < K * l; i += blockDim.x) nonfinite |= !isfinite(T[i]);
  nonfinite = __syncthreads_or(nonfinite);
  if (nonfinite) {
    if (tid == 0 && bad_out) *bad_out = 1;
    // still produce a defined (all-zero) table
  }
  for (int k = tid; k < K; k += blockDim.x) {
    double m = T[k * l];
    for (int c = 1; c < l; ++c) m = fmin(m, T[k * l + c]);
    bias_s[k] = m;
  }
  __syncthreads();
  double mx = -INFINITY;
  for (int i = tid; i < K * l; i += blockDim.x) mx = fmax(mx, __dsub_rn(T[i], bias_s[i / l]));
  mx = block_max(mx, red);
  const double spread = (K * l) ? mx : 0.0;
  const double scale = __ddiv_rn(spread, 255.0);
  for (int i = tid; i < Kp * l; i += blockDim.x) {
    uint8_t q = 0;
    if (i < K * l && scale != 0.0 && !nonfinite) {
      double r = rint(__ddiv_rn(__dsub_rn(T[i], bias_s[i / l]), scale));
      r = fmin(fmax(r, 0.0), 255.0);
      q = (uint8_t)r;
    }
    table_out[i] = q;
  }
  if (bias_out)
    for (int k = tid; k < K; k += blockDim.x) bias_out[k] = bias_s[k];
  if (tid == 0) {
    *scale_out = scale;
    *bias_total_out = pairwise_sum(bias_s, K);
  }
}

// One CTA per query.  smem: qd[d], qw[d], T[K*16], bias[K], red[32].
__global__ void __launch_bounds__(kLutThreads) k_lut_build(
    const float* __restrict__ qdense, int64_t d, double dense_weight, int has_wh,
    const double* __restrict__ inv_t, const double* __restrict__ mean,
    const float* __restrict__ centers, const int32_t* __restrict__ subdims,
    const int32_t* __restrict__ dim_off, const int32_t* __restrict__ cen_off, int K, int Kp,
    double* __restrict__ qd_out, double* __restrict__ qw_out, uint8_t* __restrict__ luts,
    double* __restrict__ bias_total, double* __restrict__ scale, double* __restrict__ offset,
    int* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* qd = reinterpret_cast<double*>(smem);
  double* qw = qd + d;
  double* T = qw + d;
  double* bias_s = T + (size_t)K * 16;
  double* red = bias_s + K;
  const int64_t q = blockIdx.x;
  const int tid = threadIdx.x;

  // qd = f64(query.dense) * dense_weight  (pipeline.py:209)
  for (int64_t i = tid; i < d; i += blockDim.x)
    qd[i] = __dmul_rn((double)qdense[q * d + i], dense_weight);
  __syncthreads();
  // qw = qd @ inverse_t.T ; offset = qd @ mean  (pipeline.py:220-223)
  if (has_wh) {
    // inv_t is stored transposed: element (r, c) at inv_t[c * d + r]
    for (int64_t r = tid; r < d; r += blockDim.x) qw[r] = dot_recipe(inv_t + r, qd, (int)d, (int)d);
    if (tid == 0) offset[q] = dot_recipe(qd, mean, (int)d);
  } else {
    for (int64_t i = tid; i < d; i += blockDim.x) qw[i] = qd[i];
    if (tid == 0) offset[q] = 0.0;
  }
  __syncthreads();
  for (int64_t i = tid; i < d; i += blockDim.x) {
    qd_out[q * d + i] = qd[i];
    qw_out[q * d + i] = qw[i];
  }
  // ADC table T[k][c] = centers_k[c] . qw[slice k]  (dense.py:218-219)
  for (int i = tid; i < K * 16; i += blockDim.x) {
    const int k = i >> 4, c = i & 15;
    const int w = subdims[k];
    T[i] = dot_recipe(centers + cen_off[k] + c * w, qw + dim_off[k], w);
  }
  __syncthreads();
  quantize_rows(T, K, 16, Kp, bias_s, red, luts + q * (int64_t)Kp * 16, nullptr, scale + q,
                bias_total + q, bad);
}

__global__ void __launch_bounds__(kLutThreads) k_adc_table(
    const float* __restrict__ centers, const int32_t* __restrict__ subdims,
    const int32_t* __restrict__ dim_off, const int32_t* __restrict__ cen_off, int K, int l,
    const double* __restrict__ qw, int64_t d, double* __restrict__ T) {
  const int64_t q = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)K * l) return;
  const int k = (int)(i / l), c = (int)(i % l);
  const int w = subdims[k];
  T[q * K * l + i] = dot_recipe(centers + cen_off[k] + (int64_t)c * w, qw + q * d + dim_off[k], w);
}

__global__ void __launch_bounds__(kLutThreads) k_quantize(const double* __restrict__ Tg, int K,
                                                          int l, int Kp, uint8_t* table,
                                                          double* bias, double* scale,
                                                          double* bias_total, int* bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* T = reinterpret_cast<double*>(smem);
  double* bias_s = T + (size_t)K * l;
  double* red = bias_s + K;
  const int64_t q = blockIdx.x;
  for (int i = threadIdx.x; i < K * l; i += blockDim.x) T[i] = Tg[q * K * l + i];
  __syncthreads();
  quantize_rows(T, K, l, Kp, bias_s, red, table + q * (int64_t)Kp * l, bias + q * K, scale + q,
                bias_total + q, bad + q);
}

}  // namespace

void launch_lut_build(const DeviceIndex& ix, const float* qdense, int64_t nq, double* qd_out,
                      double* qw_out, uint8_t* luts, double* bias_total, double* scale,
                      double* offset, int* bad, cudaStream_t st) {
  if (nq <= 0) return;
  const size_t smem = sizeof(double) * (2 * ix.d_dense + (size_t)ix.K * 16 + ix.K + 32);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_lut_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_lut_build<<<(unsigned)nq, kLutThreads, smem, st>>>(
      qdense, ix.d_dense, ix.dense_weight, ix.has_wh, ix.wh_inv_t, ix.wh_mean, ix.centers,
      ix.subdims, ix.dim_off, ix.cen_off, ix.K, ix.Kp, qd_out, qw_out, luts, bias_total, scale,
      offset, bad);
}

void launch_adc_table(const float* centers, const int32_t* subdims, const int32_t* dim_off,
                      const int32_t* cen_off, int K, int l, const double* qw, int64_t nq,
                      int64_t d, double* T, cudaStream_t st) {
  if (nq <= 0 || K <= 0) return;
  dim3 grid((unsigned)ceil_div((int64_t)K * l, kLutThreads), (unsigned)nq);
  k_adc_table<<<grid, kLutThreads, 0, st>>>(centers, subdims, dim_off, cen_off, K, l, qw, d, T);
}

void launch_quantize(const double* T, int64_t nq, int K, int l, int Kp, uint8_t* table,
                     double* bias, double* scale, double* bias_total, int* bad,
                     cudaStream_t st) {
  if (nq <= 0) return;
  const size_t smem = sizeof(double) * ((size_t)K * l + K + 32);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_quantize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_quantize<<<(unsigned)nq, kLutThreads, smem, st>>>(T, K, l, Kp, table, bias, scale,
                                                      bias_total, bad);
}

}  // namespace hs
