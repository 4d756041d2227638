// lut16_tc.cu — K2 on the 5th-generation tensor cores: batched LUT16 totals.
//
// For a group of 128 queries and a block of 256 points the LUT16 totals
// (reference lut16_scan, dense.py:263-317: total = sum_k table[k][code_k])
// are an integer matrix product
//
//     T[q][n] = sum_{k,c} LUT[q][k][c] * onehot(code_k(n) == c)
//
// with A = the queries' u8 tables (128 x 16K, K-major: one 16-byte row per
// (query, subspace) — exactly the LUT layout) and B = the one-hot expansion of
// the points' 4-bit codes (256 x 16K, K-major: one 16-byte row per (point,
// subspace) with a single 1).  tcgen05.mma kind::i8 (u8 x u8 -> s32) computes
// it exactly in TMEM (K*255 < 2^31), so totals are bit-identical to the scalar
// semantics; the epilogue narrows them to u16 (K <= 257 keeps them < 2^16)
// for the fused stage-1 kernel, which adds the sparse part and selects.
//
// Shared-memory operand layout (SWIZZLE_NONE, K-major "interleave" canonical
// layout): 16-byte column block b (= subspace) holds all MN rows
// contiguously, 16 B per row, so 8-row core matrices are 128 B apart
// (SBO = 128 B) and the two 16-byte K halves of one MMA are MN*16 B apart
// (LBO).  One MMA consumes 32 B of K = 2 subspaces.
//
// Pipeline per CTA (query group g, a range of point blocks): K is walked in
// chunks of kKC subspaces through two shared-memory stages; all 256 threads
// write a stage (LUT rows + one-hot rows), fence the async proxy, and thread 0
// issues the chunk's MMAs and commits them to the stage's mbarrier, so the
// next chunk is produced while the tensor core consumes this one.  After the
// last chunk of a block the epilogue warps read the 128x256 s32 accumulator
// (warp w reads TMEM lanes 32*(w%4).. of columns 128*(w/4)..) and store u16
// totals row-major [query][point].
#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kTM = 128;      // queries per group (MMA M)
constexpr int kTN = 256;      // points per block (MMA N)
constexpr int kKC = 8;        // subspaces per K chunk (= 4 MMAs of K=32 B)
constexpr int kTThreads = 256;
constexpr int kStageA = kKC * kTM * 16;  // 16 KB
constexpr int kStageB = kKC * kTN * 16;  // 32 KB
constexpr int kStages = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  // base offset 0, lbo mode 0, layout type SWIZZLE_NONE (0)
  return d;
}

// kind::i8 instruction descriptor: u8 x u8 -> s32, K-major A and B, M=128, N=256
__host__ __device__ constexpr uint32_t idesc_u8() {
  return (2u << 4)               // c_format = S32
         | (0u << 7) | (0u << 10)  // a/b format = unsigned 8-bit
         | ((uint32_t)(kTN >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

#define TMEM_LD32(taddr, r)                                                                      \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr))

struct TcArgs {
  int64_t n;          // points
  int64_t nq;         // queries in this batch
  int K, Kp;          // subspaces (codes), padded LUT rows
  const uint32_t* vcodes;
  int64_t vstride;    // u32 words per subspace plane
  const uint8_t* luts;  // [nq][Kp][16]
  uint16_t* tot;      // [nq][ld] u16 totals
  int64_t ld;
  int blocks_per_cta;
};

__global__ void __launch_bounds__(kTThreads, 1) k_lut16_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sA = smem_raw;                      // [stage][kKC][128][16]
  unsigned char* sB = sA + kStages * kStageA;        // [stage][kKC][256][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kStageB);  // [kStages]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t g = blockIdx.x;  // query group
  const int64_t q0 = g * kTM;
  const int64_t nblocks = (a.n + kTN - 1) / kTN;
  const int64_t blk0 = (int64_t)blockIdx.y * a.blocks_per_cta;
  const int64_t blk1 = min(nblocks, blk0 + a.blocks_per_cta);
  const int nkc = (a.K + kKC - 1) / kKC;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_u8();
  uint32_t phase[kStages] = {0u, 0u};
  bool pending[kStages] = {false, false};  // a commit on this stage not yet waited for

  // Producer registers: this thread's 4 LUT rows (A) and 8 code words (B) of
  // the next K chunk are loaded one chunk ahead so global-load latency hides
  // behind the current chunk's shared-memory writes and MMAs.
  constexpr int kArows = kTM * kKC / kTThreads;  // 4
  uint4 ra[kArows];
  uint32_t rc[kKC];
  auto load_chunk = [&](int64_t blk, int kc) {
    const int s0 = kc * kKC;
#pragma unroll
    for (int r = 0; r < kArows; ++r) {
      const int i = tid + r * kTThreads;
      const int q = i & (kTM - 1), s = i >> 7;
      ra[r] = (q0 + q < a.nq && s0 + s < a.Kp)
                  ? __ldg(reinterpret_cast<const uint4*>(a.luts + ((q0 + q) * a.Kp + s0 + s) * 16))
                  : make_uint4(0u, 0u, 0u, 0u);
    }
    const int64_t p = blk * kTN + tid;
#pragma unroll
    for (int s = 0; s < kKC; ++s)
      rc[s] = (s0 + s < a.K && p < a.n) ? __ldg(a.vcodes + (int64_t)(s0 + s) * a.vstride + (p >> 3))
                                        : 0u;
  };
  if (blk0 < blk1) load_chunk(blk0, 0);

  for (int64_t blk = blk0; blk < blk1; ++blk) {
    const int64_t p0 = blk * kTN;
    for (int kc = 0; kc < nkc; ++kc) {
      const int st = kc & 1;
      // the MMAs that last read this stage must be done before overwriting it
      if (pending[st]) {
        mbar_wait(&bars[st], phase[st]);
        phase[st] ^= 1u;
        pending[st] = false;
      }
      unsigned char* A = sA + st * kStageA;
      unsigned char* B = sB + st * kStageB;
#pragma unroll
      for (int r = 0; r < kArows; ++r) {
        const int i = tid + r * kTThreads;
        *reinterpret_cast<uint4*>(A + (i >> 7) * (kTM * 16) + (i & (kTM - 1)) * 16) = ra[r];
      }
      {
        const int sh = 4 * (int)((p0 + tid) & 7);
#pragma unroll
        for (int s = 0; s < kKC; ++s) {
          const uint32_t code = (rc[s] >> sh) & 15u;
          const uint32_t bit = 1u << (8 * (code & 3u));
          const uint32_t c4 = code >> 2;
          uint4 v;
          v.x = c4 == 0 ? bit : 0u;
          v.y = c4 == 1 ? bit : 0u;
          v.z = c4 == 2 ? bit : 0u;
          v.w = c4 == 3 ? bit : 0u;
          if (kc * kKC + s >= a.K) v = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(B + s * (kTN * 16) + tid * 16) = v;
        }
      }
      // prefetch the next chunk (possibly of the next block) into registers
      if (kc + 1 < nkc) load_chunk(blk, kc + 1);
      else if (blk + 1 < blk1) load_chunk(blk + 1, 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_addr = smem_u32(A), b_addr = smem_u32(B);
#pragma unroll
        for (int m = 0; m < kKC / 2; ++m) {
          const uint64_t ad = smem_desc(a_addr + m * 2 * (kTM * 16), kTM * 16, 128);
          const uint64_t bd = smem_desc(b_addr + m * 2 * (kTN * 16), kTN * 16, 128);
          mma_u8(tmem, ad, bd, idesc, (kc > 0 || m > 0) ? 1u : 0u);
        }
        mma_commit(&bars[st]);
      }
      pending[st] = true;
    }
    // wait for the block's last chunk (commit tracks all earlier MMAs too)
#pragma unroll
    for (int st = 0; st < kStages; ++st) {
      if (pending[st]) {
        mbar_wait(&bars[st], phase[st]);
        phase[st] ^= 1u;
        pending[st] = false;
      }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warp w reads lanes 32*(w%4).. (queries) and columns 128*(w/4)..
    {
      const int quad = warp & 3, half = warp >> 2;
      const int64_t q = q0 + quad * 32 + (tid & 31);
      uint16_t* row = a.tot + q * a.ld + p0 + half * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * 128 + c * 32);
        TMEM_LD32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (q < a.nq) {
          uint4 w[4];
          uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int j = 0; j < 16; ++j) wp[j] = (r[2 * j] & 0xFFFFu) | (r[2 * j + 1] << 16);
          uint4* dst = reinterpret_cast<uint4*>(row + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = w[j];
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM reads done before the next block's MMAs overwrite it
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTN));
}

}  // namespace

size_t lut16_tc_smem() {
  return kStages * (kStageA + kStageB) + kStages * sizeof(uint64_t) + 16;
}

int64_t lut16_tc_ld(int64_t n) { return ((n + kTN - 1) / kTN) * kTN; }

int launch_lut16_tc(const DeviceIndex& ix, const uint8_t* luts, int64_t nq, uint16_t* tot,
                    int64_t ld, cudaStream_t st) {
  if (nq <= 0 || ix.n <= 0) return HS_OK;
  if (ix.K > 257) HS_FAIL(HS_EUNSUPPORTED, "tensor-core LUT16 needs K <= 257");
  TcArgs a;
  a.n = ix.n;
  a.nq = nq;
  a.K = ix.K;
  a.Kp = ix.Kp;
  a.vcodes = ix.vcodes;
  a.vstride = ix.vstride;
  a.luts = luts;
  a.tot = tot;
  a.ld = ld;
  const int64_t groups = ceil_div(nq, kTM);
  const int64_t nblocks = ceil_div(ix.n, kTN);
  // ~2 CTAs per SM worth of work items over (groups x point ranges)
  int64_t ranges = ceil_div(2LL * kNumSMs, groups);
  if (ranges > nblocks) ranges = nblocks;
  if (ranges < 1) ranges = 1;
  a.blocks_per_cta = (int)ceil_div(nblocks, ranges);
  ranges = ceil_div(nblocks, a.blocks_per_cta);
  const size_t smem = lut16_tc_smem();
  HS_CUDA(cudaFuncSetAttribute(k_lut16_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)groups, (unsigned)ranges);
  k_lut16_tc<<<grid, kTThreads, smem, st>>>(a);
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace hs
