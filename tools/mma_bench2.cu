// Dev microbenchmark (not part of the product): issue rate of back-to-back
// tcgen05.mma kind::i8 with A from TMEM, single CTA (M=128) vs CTA pair
// (cta_group::2, M=256), for the N values the LUT16 tensor-core kernel uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench2 tools/mma_bench2.cu
// Prints cycles per MMA (operands resident, contents irrelevant) and, timed
// with CUDA events over all 148 SMs, the u8 op rate that issue cadence amounts
// to (one JSON line per configuration): the tensor-pipe ceiling bench.py's
// `roofline.issue_peak` restates analytically.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_u8(int m, int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <bool PAIR>
__global__ void k_bench(int iters, int N, int nacc, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (tid < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const int M = PAIR ? 256 : 128;
  const int NL = PAIR ? N / 2 : N;
  const uint32_t idesc = idesc_u8(M, N);
  const uint64_t bd = desc(smem_u32(sm), (uint32_t)(NL * 16), 128);
  const uint32_t ta = tmem + (uint32_t)(nacc * N);  // A after the accumulators
  if (tid < 32 && (!PAIR || rank == 0)) {
    long long t0 = clock64();
    uint32_t pred0 = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred0));
    if (pred0) {
      // 16 MMAs per loop trip, one elected thread, no per-MMA warp sync
      for (int it0 = 0; it0 < iters; it0 += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int it = it0 + u;
          const uint32_t d = tmem + (uint32_t)(u % 2 == 0 || nacc == 1 ? 0 : 1) * (uint32_t)N;
          const uint32_t a = ta + 8u * (uint32_t)(u & 3);
          const uint64_t b = bd + (uint64_t)(u * 2 * NL);
          const int acc = it >= 2 ? 1 : 0;
          if (PAIR)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
        }
      }
    }
    __syncwarp();
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    if (pred) {
      if (PAIR)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  } else if (PAIR && rank != 0 && tid < 32) {
    asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 4);
  const int iters = 4096;
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k_bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct C { int N, nacc; };
  for (C c : {C{96, 1}, C{96, 2}, C{192, 1}, C{192, 2}}) {
    long long h = 0;
    k_bench<false><<<148, 128, smem>>>(iters, c.N, c.nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cta_group::1 M=128 N=%3d acc=%d: %7.1f cycles/MMA (floor %5.1f) %s\n", c.N, c.nacc,
           (double)h / iters, 128.0 * c.N / 256.0, cudaGetErrorString(e));
  }
  for (C c : {C{96, 1}, C{96, 2}, C{192, 1}, C{192, 2}}) {
    long long h = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_bench<true>, iters, c.N, c.nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cta_group::2 M=256 N=%3d acc=%d: %7.1f cycles/MMA (floor %5.1f) %s\n", c.N, c.nacc,
           (double)h / iters, 256.0 * c.N / 512.0, cudaGetErrorString(e));
    // whole-chip rate: a longer launch between two events
    const int long_iters = 1 << 18;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k_bench<true>, long_iters, c.N, c.nacc, d);  // warm
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_bench<true>, long_iters, c.N, c.nacc, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 74.0 * long_iters * 2.0 * 256.0 * c.N * 32.0;
    printf("{\"kind\": \"tcgen05.mma.cta_group::2.kind::i8\", \"M\": 256, \"N\": %d, \"acc_buffers\": %d, "
           "\"ms\": %.3f, \"u8_tops\": %.1f}\n", c.N, c.nacc, ms, ops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
