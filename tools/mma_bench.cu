// Dev microbenchmark (not part of the product): tcgen05.mma issue rate for
// the operand modes the LUT16 tensor-core kernel can use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
// Prints cycles per MMA for each variant (one CTA per SM, back-to-back MMAs
// into one accumulator, operands resident, contents irrelevant).
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int KIND, bool TS, int LAYOUT, int N, int MODE>
__global__ void k_bench(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  __shared__ volatile int done;
  if (tid == 0) done = 0;
  __syncthreads();
  const int warp = tid >> 5;
  if (warp >= 1 && warp <= 4 && (MODE == 2 || MODE == 4)) {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = j * tid;
    const uint32_t lb = (uint32_t)(((warp & 3) * 32) << 16);
    long long cnt = 0;
    while (!done) {
      ++cnt;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + lb + 448),
        "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if ((tid & 31) == 0 && blockIdx.x == 0) out[150 + warp] = cnt;
  }
  if (warp >= 5 && warp <= 8 && (MODE == 3 || MODE == 4)) {
    uint32_t acc = 0;
    const uint32_t lb = (uint32_t)(((warp & 3) * 32) << 16);
    while (!done) {
      uint32_t r[4];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]) : "r"(tmem + lb + 480));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r[0] ^ r[3];
    }
    if (acc == 12345) out[148] = acc;
  }
  if (tid == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);           // i8 -> s32
    else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);  // bf16 -> f32
    const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 32 * 1024);
    uint64_t ad, bd;
    if (LAYOUT == 0) {
      ad = desc(a_addr, 128 * 16, 128, 0);
      bd = desc(b_addr, N * 16, 128, 0);
    } else {
      ad = desc(a_addr, 16, 1024, 2);
      bd = desc(b_addr, 16, 1024, 2);
    }
    const uint32_t d = tmem, ta = tmem + 256;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      if (TS) {
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      if (MODE == 1 && (i & 3) == 3)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
        smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, bool TS, int LAYOUT, int N, int MODE = 0>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 160);
  cudaMemset(d, 0, sizeof(long long) * 160);
  auto k = k_bench<KIND, TS, LAYOUT, N, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  k<<<148, 288, 100 * 1024>>>(iters, d);
  k<<<148, 288, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[160];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double floor = 128.0 * N / 256.0;
  printf("mode %d %-30s N=%3d  %7.1f cyc/MMA  (floor %5.1f)  sttm/warp %lld -> %.1f cyc/STTM.x32 %s\n", MODE, name, N, avg / iters, floor,
         h[151], h[151] ? (double)h[0] / h[151] : 0.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, true, 0, 192, 0>("i8  TS  B no-swizzle");
  run<0, true, 0, 192, 1>("i8  TS  + commit/4");
  run<0, true, 0, 192, 2>("i8  TS  + STTM warps");
  run<0, true, 0, 192, 3>("i8  TS  + LDTM warps");
  run<0, true, 0, 192, 4>("i8  TS  + STTM+LDTM");
  run<0, true, 1, 192, 4>("i8  TS  SW128 + STTM+LDTM");
  run<0, false, 0, 256, 4>("i8  SS  + STTM+LDTM");
  return 0;
}
