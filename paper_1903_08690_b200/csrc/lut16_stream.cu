// lut16_stream.cu — HBM-bound LUT16 scan for small query batches (K2').
//
// Replaces lut16_scan (reference dense.py:263-317) for batches too small for
// the tensor-core pass (lut16_tc.cu): each query streams every packed code of
// the index once, so the kernel is bound by the code stream out of HBM
// (N * ceil(K/2) bytes per query) and by the in-register lookups.
//
// Codes: blocked vertical nibble planes, vcodes[block][k][512] u32 — block =
// 4096 consecutive layout slots, word w of row k holds the 4-bit codes of
// points 8w..8w+7 of the block (nibble j = point 8w+j).  Any run of subspace
// rows of one block is contiguous, so a stage of the shared-memory ring
// (kSlice rows = 16 KB) is ONE 1-D bulk copy (cp.async.bulk, TMA) issued by a
// producer warp and counted on an mbarrier; 256 consumer threads own 16
// points each, pull their codes of a stage into registers (one LDS.64 per
// row), release the stage, and look the codes up in the query's u8 tables
// with PRMT (the GPU analogue of the paper's in-register PSHUFB LUT16,
// PAPER.md:374-397).  Three CTAs per SM (4-stage rings, 12 x 16 KB in flight
// per SM).  Blocks are handed out by ticket: a CTA starts on block blockIdx.x
// and draws the following ones from a per-query counter (the next ticket is
// in flight while the current block streams), so SMs that run ahead take
// more blocks; the last CTA to finish re-arms the counter for the next launch.
// (The kernel ends about half a block's time after the tickets run out —
// ~6 of the 78 us a 320 MB query takes.  Half-block work units — ring stages
// of 16 rows x 1 KB, one bulk copy per row, 8 points per thread — were
// measured slower: 88 vs 80 us at 320 MB, 166 vs 145 us at 640 MB; the 1 KB
// copies 2 KB apart stream at 4.1 instead of 5.0 TB/s.)
//
// Accumulation: a PRMT result register holds 4 points' bytes.  `all` adds
// the registers as plain 32-bit integers (a base-256 sum with carries), `odd`
// adds bytes 1 and 3 as two u16 lanes; with S_j = the sum of byte j,
//   all = S0 + 2^8 S1 + 2^16 S2 + 2^24 S3 (mod 2^32),  odd = S1 | S3 << 16,
// so S0 + 2^16 S2 = all - 2^8 S1 - 2^24 S3 exactly (every S_j <= 255*256 <
// 2^16 for K <= 256).  Totals are exact integers (dense.py:297-317).
//
// Modes: TOTALS writes u16 totals of points [0, m) (the sample of the
// threshold pass, fuse.cu); FILTER appends (point, total) with total >=
// tlim[q] to the CTA's private list segment — the same contract as
// launch_lut16_filter (kernels.cuh), consumed by k_fuse_cands.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kSP = 4096;             // points per code block (= the stage-1 chunk)
constexpr int kRowWords = kSP / 8;    // u32 per subspace row of a block (2 KB)
constexpr int kSlice = 8;             // subspace rows per ring stage
constexpr int kStageBytes = kSlice * kRowWords * 4;  // 16 KB
#ifndef HS_STREAM_STAGES
#define HS_STREAM_STAGES 4
#endif
constexpr int kStages = HS_STREAM_STAGES;
constexpr int kConsumers = 256;       // 16 points each
#ifndef HS_STREAM_CTAS
#define HS_STREAM_CTAS 3
#endif
constexpr int kCtasPerSM = HS_STREAM_CTAS;
constexpr int kSchedQueries = 4096;   // scheduler slots after the code planes

bool env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] && e[0] != '0';
}

struct StreamArgs {
  const uint32_t* vcodes;
  int K, K8;            // subspaces; K rounded up to a multiple of kSlice
  int Kp;               // rows per query in `luts`
  int64_t n;            // points scanned: [0, n)
  int64_t nblocks;      // ceil(n / kSP)
  const uint8_t* luts;  // [nq][Kp][16]
  // totals
  uint16_t* tot;
  int64_t ld;
  // filter
  const uint32_t* tlim;
  uint2* list;
  uint32_t* cnt;
  int64_t cap;
  // dynamic block scheduling: sched[2q] = next block of query q, sched[2q+1]
  // = CTAs done (the last one re-arms both for the next launch)
  uint32_t* sched;
  // opaque multiplier (1): accumulator adds issue as IMAD on the FMA pipe,
  // which the lookups leave idle (PRMT, LOP3, SHF and IADD3 all share the
  // half-rate ALU pipe that bounds this kernel)
  uint32_t one;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// PRMT, LOP3, SHF and IADD3 all issue on the half-rate ALU pipe, which bounds
// this kernel (ncu: ALU pipe 85% active, FMA pipe 17%, LSU 14%), so whatever
// can issue elsewhere does: the accumulator adds are IMADs by an opaque 1 and
// the << 4 an IMUL by an opaque 16 (FMA pipe; ptxas would turn literal
// constants back into IADD3 / SHF).
__device__ __forceinline__ uint32_t add_fma(uint32_t x, uint32_t acc, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(acc));
  return r;
}
__device__ __forceinline__ uint32_t mul_fma(uint32_t x, uint32_t m) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m));
  return r;
}

// One subspace row, 8 points (one code word w, nibble j = point j): the two
// result registers (points 0-3, 4-7; byte = table entry) are added into the
// base-256 sums all0/all1 and, bytes 1 and 3 only, into the u16 lanes of
// odd0/odd1.  PRMT picks among 8 pool bytes by the low 3 bits of a selector
// nibble, so entries 0-7 (T.x, T.y) and 8-15 (T.z, T.w) are both looked up
// with the selector s = code & 7 and blended by a byte mask of the codes'
// bit 3 — one more PRMT in sign-replicate mode: the msb of byte j of w is bit
// 3 of point 2j+1, the msb of byte j of w << 4 that of point 2j.  12 ALU-pipe
// instructions per 8 codes.
__device__ __forceinline__ void row8(const uint4& T, uint32_t w, uint32_t one, uint32_t sixteen,
                                     uint32_t& all0, uint32_t& all1, uint32_t& odd0,
                                     uint32_t& odd1) {
  const uint32_t s = w & 0x77777777u;
  const uint32_t sh = s >> 16;
  const uint32_t a0 = prmt(T.x, T.y, s), a1 = prmt(T.x, T.y, sh);
  const uint32_t b0 = prmt(T.z, T.w, s), b1 = prmt(T.z, T.w, sh);
  const uint32_t w4 = mul_fma(w, sixteen);
  const uint32_t k0 = prmt(w, w4, 0x9D8Cu), k1 = prmt(w, w4, 0xBFAEu);
  const uint32_t r0 = (b0 & k0) | (a0 & ~k0);
  const uint32_t r1 = (b1 & k1) | (a1 & ~k1);
  all0 = add_fma(r0, all0, one);
  all1 = add_fma(r1, all1, one);
  odd0 = add_fma(prmt(r0, 0u, 0x4341u), odd0, one);
  odd1 = add_fma(prmt(r1, 0u, 0x4341u), odd1, one);
}

template <int MODE>  // 0 totals, 1 filter
__global__ void __launch_bounds__(kConsumers + 32, kCtasPerSM) k_lut16_stream(StreamArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;
  uint4* lut = reinterpret_cast<uint4*>(smem_raw + (size_t)kStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(lut + a.K8);
  uint64_t* empty = full + kStages;
  int32_t* s_blk = reinterpret_cast<int32_t*>(empty + kStages);  // [kStages] block of the stage
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_blk + kStages);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t q = blockIdx.y;
  const int seg = blockIdx.x, nseg = gridDim.x;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumers / 32);
    }
    *s_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers / 32) {
    // ---- producer: one bulk copy per (block, slice of kSlice rows); starts
    // streaming while the consumers stage the query's tables ----
    if (lane == 0) {
      uint32_t s = 0, ph = 1;  // stage, parity of its `empty` barrier (first pass: free)
      const bool dyn = a.sched != nullptr;
      // first block: the CTA's own index; then tickets nseg, nseg+1, ...
      int64_t b = seg;
      while (b < a.nblocks) {
        // the next block's ticket is in flight while this block streams
        const int64_t bn = dyn ? (int64_t)atomicAdd(&a.sched[2 * q], 1u) + nseg : b + nseg;
        const uint32_t* blk = a.vcodes + b * (int64_t)a.K * kRowWords;
        for (int k0 = 0; k0 < a.K; k0 += kSlice) {
          const uint32_t bytes = (uint32_t)min(kSlice, a.K - k0) * (kRowWords * 4);
          mbar_wait(&empty[s], ph);
          s_blk[s] = (int32_t)b;
          mbar_arrive_tx(&full[s], bytes);
          bulk_g2s(ring + (size_t)s * kStageBytes, blk + (int64_t)k0 * kRowWords, bytes, &full[s]);
          if (++s == kStages) s = 0, ph ^= 1u;
        }
        b = bn;
      }
      // end marker
      mbar_wait(&empty[s], ph);
      s_blk[s] = -1;
      mbar_arrive(&full[s]);
      if (dyn) {
        __threadfence();
        if (atomicAdd(&a.sched[2 * q + 1], 1u) == (uint32_t)nseg - 1u) {
          a.sched[2 * q] = 0u;  // every CTA has drawn its last ticket: re-arm
          a.sched[2 * q + 1] = 0u;
        }
      }
    }
    return;
  }

  // ---- consumers ----
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.luts + q * (int64_t)a.Kp * 16);
    for (int i = tid; i < a.K8; i += kConsumers) {
      lut[i] = i < a.K ? src[i] : make_uint4(0u, 0u, 0u, 0u);  // rows past K add 0
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
  const uint32_t tl = MODE == 1 ? a.tlim[q] : 0u;
  uint2* seg_list = MODE == 1 ? a.list + (q * nseg + seg) * a.cap : nullptr;
  const uint32_t one = a.one, sixteen = a.one << 4;
  uint32_t s = 0, ph = 0;  // stage, parity of its `full` barrier
  for (;;) {
    uint32_t all[4] = {0u, 0u, 0u, 0u}, odd[4] = {0u, 0u, 0u, 0u};
    int64_t b = 0;
    for (int k0 = 0; k0 < a.K; k0 += kSlice) {
      mbar_wait(&full[s], ph);
      if (k0 == 0) {
        b = s_blk[s];
        if (b < 0) break;
      }
      // every stage is read as kSlice rows: rows past K hold stale codes and
      // look up all-zero tables
      const uint2* src = reinterpret_cast<const uint2*>(ring + (size_t)s * kStageBytes) + tid;
      uint2 w[kSlice];
#pragma unroll
      for (int r = 0; r < kSlice; ++r) w[r] = src[r * (kRowWords / 2)];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // codes are in registers: release the stage
#pragma unroll
      for (int r = 0; r < kSlice; ++r) {
        const uint4 T = lut[k0 + r];
        row8(T, w[r].x, one, sixteen, all[0], all[1], odd[0], odd[1]);
        row8(T, w[r].y, one, sixteen, all[2], all[3], odd[2], odd[3]);
      }
      if (++s == kStages) s = 0, ph ^= 1u;
    }
    if (b < 0) break;
    // totals of this thread's 16 points: point 4i+j = S_j of register i
    uint32_t t[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t s1 = odd[i] & 0xFFFFu, s3 = odd[i] >> 16;
      const uint32_t e = all[i] - (s1 << 8) - (s3 << 24);
      t[4 * i + 0] = e & 0xFFFFu;
      t[4 * i + 1] = s1;
      t[4 * i + 2] = e >> 16;
      t[4 * i + 3] = s3;
    }
    const int64_t p0 = b * kSP + (int64_t)tid * 16;
    if constexpr (MODE == 0) {
      if (p0 + 16 <= a.n) {
        uint4 o0, o1;
        o0.x = t[0] | t[1] << 16;
        o0.y = t[2] | t[3] << 16;
        o0.z = t[4] | t[5] << 16;
        o0.w = t[6] | t[7] << 16;
        o1.x = t[8] | t[9] << 16;
        o1.y = t[10] | t[11] << 16;
        o1.z = t[12] | t[13] << 16;
        o1.w = t[14] | t[15] << 16;
        uint4* dst = reinterpret_cast<uint4*>(a.tot + q * a.ld + p0);
        dst[0] = o0;
        dst[1] = o1;
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (p0 + j < a.n) a.tot[q * a.ld + p0 + j] = (uint16_t)t[j];
      }
    } else {
      uint32_t mx = t[0];
#pragma unroll
      for (int j = 1; j < 16; ++j) mx = max(mx, t[j]);
      if (mx >= tl) {  // ~k1 * n / sample passes per query in all
        const int lim = (int)min((int64_t)16, a.n - p0);  // < 16 in the last block only
        uint32_t pm = 0u;
#pragma unroll
        for (int j = 0; j < 16; ++j) pm |= (t[j] >= tl && j < lim) ? (1u << j) : 0u;
        uint32_t pos = atomicAdd(s_cnt, (uint32_t)__popc(pm));  // one shared atomic per thread
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if ((pm >> j) & 1u) {
            if (pos < (uint32_t)a.cap) seg_list[pos] = make_uint2((uint32_t)(p0 + j), t[j]);
            ++pos;
          }
        }
      }
    }
  }
  if constexpr (MODE == 1) {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    if (tid == 0) a.cnt[q * nseg + seg] = *s_cnt;  // > cap: overflow (k_fuse_cands falls back)
  }
}

// pair-major packed codes (dense.py:156-170) -> blocked vertical nibble planes
__global__ void k_to_vertical(const uint8_t* __restrict__ packed, int64_t n, int K,
                              int64_t nblocks, uint32_t* __restrict__ v) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // word (8 points), global
  const int k = blockIdx.y;
  if (g >= nblocks * kRowWords) return;
  const uint8_t* row = packed + (int64_t)(k >> 1) * n;
  const int sh = (k & 1) ? 4 : 0;
  uint32_t w = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t pt = g * 8 + j;
    const uint32_t c = pt < n ? ((row[pt] >> sh) & 0xFu) : 0u;
    w |= c << (4 * j);
  }
  const int64_t b = g / kRowWords, wi = g % kRowWords;
  v[(b * K + k) * kRowWords + wi] = w;
}

size_t stream_smem(int K8) {
  return (size_t)kStages * kStageBytes + (size_t)K8 * 16 + sizeof(uint64_t) * 2 * kStages +
         sizeof(int32_t) * kStages + 16;
}

int launch_stream(const DeviceIndex& ix, int mode, StreamArgs& a, int64_t nq, int64_t nseg,
                  cudaStream_t st) {
  if (nq <= 0 || a.n <= 0) return HS_OK;
  if (!lut16_stream_supported(ix)) HS_FAIL(HS_EUNSUPPORTED, "streamed LUT16 unsupported for this index");
  a.vcodes = ix.vcodes;
  a.K = ix.K;
  a.K8 = (ix.K + kSlice - 1) / kSlice * kSlice;
  a.Kp = ix.Kp;
  a.nblocks = ceil_div(a.n, kSP);
  const size_t smem = stream_smem(a.K8);
  a.one = 1u;
  a.sched = env_flag("HSB200_STREAM_STATIC")
                ? nullptr
                : ix.vcodes + ceil_div(ix.n, kSP) * (int64_t)ix.K * kRowWords;
  if (nq > kSchedQueries) a.sched = nullptr;
  auto kern = mode == 0 ? k_lut16_stream<0> : k_lut16_stream<1>;
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)nseg, (unsigned)nq);
  kern<<<grid, kConsumers + 32, smem, st>>>(a);
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace

// the code planes, then the scheduler words of k_lut16_stream (zeroed here,
// re-armed by every launch)
int64_t vertical_words(int64_t n, int K) {
  return ceil_div(n, kSP) * (int64_t)K * kRowWords + 2 * kSchedQueries;
}

void launch_to_vertical(const uint8_t* packed, int64_t n, int K, uint32_t* v, cudaStream_t st) {
  if (K <= 0 || n <= 0) return;
  const int64_t nblocks = ceil_div(n, kSP);
  dim3 grid((unsigned)ceil_div(nblocks * kRowWords, 256), (unsigned)K);
  k_to_vertical<<<grid, 256, 0, st>>>(packed, n, K, nblocks, v);
  cudaMemsetAsync(v + nblocks * (int64_t)K * kRowWords, 0, sizeof(uint32_t) * 2 * kSchedQueries, st);
}

bool lut16_stream_supported(const DeviceIndex& ix) {
  return ix.vcodes != nullptr && ix.K > 0 && ix.K <= 256 && ix.l == 16;
}

int64_t lut16_stream_segments(const DeviceIndex& ix, int64_t n_limit) {
  const int64_t n = n_limit >= 0 ? std::min(n_limit, ix.n) : ix.n;
  return std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kSP), (int64_t)kCtasPerSM * kNumSMs));
}

void lut16_stream_layout(const DeviceIndex& ix, int64_t* nseg, double* frac) {
  const int64_t nblocks = ceil_div(ix.n, kSP);
  *nseg = lut16_stream_segments(ix, -1);
  *frac = std::min(1.0, (double)(ceil_div(nblocks, *nseg) * kSP) / (double)std::max<int64_t>(ix.n, 1));
}

int launch_lut16_stream_totals(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                               uint16_t* tot, int64_t ld, cudaStream_t st, int64_t n_limit) {
  StreamArgs a{};
  a.n = n_limit >= 0 ? std::min(n_limit, ix.n) : ix.n;
  a.luts = luts;
  a.tot = tot;
  a.ld = ld;
  return launch_stream(ix, 0, a, nq, lut16_stream_segments(ix, a.n), st);
}

int launch_lut16_stream_filter(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                               const uint32_t* tlim, uint2* list, uint32_t* cnt, int64_t cap,
                               cudaStream_t st) {
  StreamArgs a{};
  a.n = ix.n;
  a.luts = luts;
  a.tlim = tlim;
  a.list = list;
  a.cnt = cnt;
  a.cap = cap;
  return launch_stream(ix, 1, a, nq, lut16_stream_segments(ix, -1), st);
}

}  // namespace hs
