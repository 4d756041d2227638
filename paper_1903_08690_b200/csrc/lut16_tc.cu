// lut16_tc.cu — K2 on the 5th-generation tensor cores: batched LUT16 totals.
//
// For a block of 128 points and a group of NQ queries the LUT16 totals
// (reference lut16_scan, dense.py:263-317: total = sum_k table[k][code_k])
// are an integer matrix product
//
//     T[n][q] = sum_{k,c} onehot(code_k(n) == c) * LUT[q][k][c]
//
// issued as tcgen05.mma kind::i8 (u8 x u8 -> s32, exact: K*255 < 2^31) in the
// "A in tensor memory" form:
//   A (128 points x 16K, K-major) = the one-hot expansion of the points'
//     4-bit codes, generated in registers and written straight into TMEM with
//     tcgen05.st (no shared-memory round trip for the expanded operand);
//   B (NQ queries x 16K, K-major) = the group's u8 tables, resident in shared
//     memory while the CTA walks the group's point blocks (one 16-byte row per
//     (query, subspace) — exactly the LUT layout), so the only shared-memory
//     traffic in the steady state is the tensor core reading B;
//   D (128 x NQ s32) in TMEM, double-buffered so the epilogue of block i
//     overlaps the MMAs of block i+1.
// Totals are bit-identical to the scalar semantics; the epilogue narrows them
// to u16 (K <= 257 keeps them < 2^16) row-major [query][point] for the fused
// stage-1 kernel, which adds the sparse part and selects.
//
// Warp roles (672 threads, one CTA per SM — it owns all 512 TMEM columns):
//   warps 0-11  producers: thread = point lane (three warps per TMEM lane
//               quadrant, K chunks round-robin — the one-hot generation is
//               latency-bound per warp, so it needs the warps); per 8
//               subspaces one coalesced u32 load (8 codes, one block ahead),
//               32 one-hot words (one clamped funnel shift each), one
//               tcgen05.st.32x32b.x32 into an A ring slot, arrive `afull`;
//   warps 12-19 epilogue (two per lane quadrant, alternate 32-column
//               tiles): tcgen05.ld the finished
//               accumulator, then either transpose through shared memory +
//               TMA tensor store of u16 tiles (totals mode) or compare
//               against the queries' thresholds and append the passes
//               (filter mode); arrive `dempty`;
//   warp 20     TMEM allocation; one elected lane issues the MMAs (<= 8 per
//               chunk, K = 32 B = 2 subspaces each) and the commits.
//
// Shared-memory B layout (SWIZZLE_NONE, K-major canonical): 16-byte column
// block k (= subspace) holds the NQ query rows contiguously, so 8-row core
// matrices are 128 B apart (SBO) and the two subspaces of one MMA are NQ*16 B
// apart (LBO).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.cuh"

// dev A/B switches (build with HSB200_EXTRA_NVFLAGS=-D...=0 and a library tag)
#ifndef HS_TC_WARP_ARRIVE
#define HS_TC_WARP_ARRIVE 1  // one barrier arrive per warp instead of per thread
#endif
#ifndef HS_TC_FWD
#define HS_TC_FWD 1          // pair: the peer's producers arrive locally; forwarding warps relay
#endif
#ifndef HS_TC_LDMODE
#define HS_TC_LDMODE 0       // producers' code loads: 0 nc+no_allocate asm, 1 plain ld.global, 2 __ldg
#endif
#ifndef HS_TC_PREGEN
#define HS_TC_PREGEN 1       // producers generate a chunk's one-hot before waiting for its slot
#endif
#ifndef HS_TC_ASYNC
#define HS_TC_ASYNC 1        // pair: the peer's producers signal the leader's `afull` with st.async
                             // (transaction bytes, non-blocking) instead of forwarded remote arrives
#endif
#ifndef HS_TC_ROLLED
#define HS_TC_ROLLED 1       // producers' chunk loop rolled (one copy of the chunk code)
#endif

namespace hs {

namespace {

constexpr int kPM = 128;       // points per block (MMA M, TMEM lanes)
constexpr int kKC = 8;         // subspaces per code word (8 nibbles)
constexpr int kProd = HS_TC_WARP_ARRIVE ? 4 : 128;  // arrivals per A chunk (4 producer warps)
#ifndef HS_TC_NPAR
#define HS_TC_NPAR 3
#endif
constexpr int kNPar = HS_TC_NPAR;  // producer warps per TMEM lane quadrant (round-robin over chunks)
#ifndef HS_TC_EPIPAR
#define HS_TC_EPIPAR 2
#endif
constexpr int kEpiPar = HS_TC_EPIPAR;  // epilogue warps per lane quadrant (alternate 32-column tiles)
constexpr int kProdWarps = 4 * kNPar;
constexpr int kEpiWarp0 = kProdWarps;      // a multiple of 4: warp & 3 = lane quadrant
constexpr int kMmaWarp = kEpiWarp0 + 4 * kEpiPar;
constexpr int kEpi = (HS_TC_WARP_ARRIVE ? 4 : 128) * kEpiPar;  // dempty arrivals per block
constexpr int kThreadsTc = 32 * (kMmaWarp + 1);  // 12 producer, 8 epilogue, 1 MMA warps
// pair mode: the leader's `afull` / `dempty` barriers also count the peer
// CTA's producers / epilogue.  A cluster-scope remote mbarrier arrive blocks
// the issuing warp for ~1000 cycles (measured, HS_TCPROF), and relaying
// through forwarding warps (HS_TC_ASYNC=0: kFwd warps, slot s by warp
// s % kFwd) still left the relay latency in every slot's turnaround.  The
// peer therefore signals with st.async (HS_TC_ASYNC=1): a 4-byte asynchronous
// store into the leader's shared memory that completes 4 transaction bytes on
// the leader's barrier — non-blocking — while the leader's own warp of the
// same lane quadrant arrives with expect_tx(4).  cfg5-law filter pass 26.1 ->
// 22.4 ms per 1920 queries x 10^7 points.
constexpr int kFwd = (HS_TC_FWD && !HS_TC_ASYNC) ? 4 : 0;
constexpr int kFwdWarp0 = kMmaWarp + 1;
constexpr int kThreadsPair = 32 * (kFwdWarp0 + kFwd);
static_assert(kEpiWarp0 % 4 == 0, "epilogue warps must start on a lane-quadrant boundary");
constexpr int kTmemCols = 512;
constexpr int kMaxNQ = 224;    // 2*NQ accumulator + >= 2 A slots of 32 columns <= 512
constexpr size_t kStageBytes = 4 * kEpiPar * 2 * 32 * 32 * 2;  // epilogue staging: 2 x 32x32 u16 per warp
constexpr size_t kSmemBudget = 194 * 1024;          // resident B (the group's tables)

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

// kind::i8 instruction descriptor: u8 x u8 -> s32, K-major A and B, M=128, N=n
__device__ __forceinline__ uint32_t idesc_u8(int n) {
  return (2u << 4)                 // c_format = S32
         | (0u << 7) | (0u << 10)  // a/b format = unsigned 8-bit
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kPM >> 4) << 24);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// The suspend-time hint lets a waiting warp sleep until the phase completes
// instead of re-polling: without it the waiting epilogue / MMA / producer
// warps' retry loops took ~30% of the issue slots the producers need.
#ifndef HS_TC_SPIN
#define HS_TC_SPIN 0  // 1: waits without the suspend-time hint (dev A/B)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if HS_TC_SPIN
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
#endif
}

// Polling wait with a sleep between probes, for warps whose wait is long and
// not latency-critical: at cfg5 the suspend-hint loops of idle epilogue /
// producer warps executed ~38% of the kernel's instructions (ncu), issue
// slots the producers need.
#ifndef HS_TC_SLEEP_EPI
#define HS_TC_SLEEP_EPI 256  // ns between probes of the epilogue's dfull wait (0: hint loop)
#endif
#ifndef HS_TC_SLEEP_PROD
#define HS_TC_SLEEP_PROD 0   // ns between probes of the producers' aempty wait (0: hint loop)
#endif
// busy poll without the suspend hint (the MMA issuer: react at once)
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

#ifndef HS_TC_MMASPIN
#define HS_TC_MMASPIN 0  // 1: the MMA issuer polls without the suspend hint
#endif
__device__ __forceinline__ void mbar_wait_mma(uint64_t* bar, uint32_t parity) {
#if HS_TC_MMASPIN
  mbar_wait_spin(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, int ns) {
  if (ns <= 0) {
    mbar_wait(bar, parity);
    return;
  }
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// TMA tensor store of one 32x32 u16 tile (rows = queries, cols = points)
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* map, const void* ssrc, int x,
                                               int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(ssrc)), "r"(x), "r"(y)
      : "memory");
}

// ---- CTA-pair (cta_group::2) helpers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// shared::cluster address of the same shared variable in CTA `rank`
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// one arrival that also expects `bytes` of asynchronous-store transactions
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 4-byte asynchronous store into another CTA's shared memory that completes 4
// transaction bytes on that CTA's mbarrier: a non-blocking remote signal (a
// remote mbarrier.arrive.release.cluster stalls the issuing warp ~1000 cycles)
__device__ __forceinline__ void st_async_signal(uint32_t cluster_dst, uint32_t cluster_bar) {
  asm volatile(
      "st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(
          cluster_dst),
      "r"(1u), "r"(cluster_bar)
      : "memory");
}

// leader CTA only: D[256 x N] (+)= A[256 x 32 B] (TMEM, 128 rows per CTA) * B (smem,
// N/2 columns per CTA)
__device__ __forceinline__ void mma_ts2(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// completion of the leader's MMAs signalled to the barrier at the same
// shared-memory offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
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

#define TMEM_LD16(taddr, r)                                                                      \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15}, [%16];"                                                                             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15])                                                                 \
      : "r"(taddr))

#define TMEM_ST32(taddr, r)                                                                        \
  asm volatile(                                                                                    \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr), \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),      \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),            \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),          \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),          \
      "r"(r[29]), "r"(r[30]), "r"(r[31])                                                           \
      : "memory")

struct TcArgs {
  int64_t n;               // points
  int64_t nq;              // queries in this batch
  int K, Kp;               // subspaces (codes), LUT rows per query (even)
  int nq_grp;              // NQ: queries per group (MMA N, multiple of 32)
  int slots;               // A ring slots
  const uint32_t* hcodes;  // blocked: [n/128][ceil(K/8)][128], nibble s = code of subspace 8c+s
  const uint8_t* luts;     // [nq][Kp][16]
  uint16_t* tot;           // [nq][ld] u16 totals (totals mode)
  int64_t ld;
  int nwords;              // ceil(K/8): code words per point
  // filter mode: emit (point, total) with total >= tlim[q] into CTA-private
  // segments list[q][cta][cap] with counts cnt[q][cta] (> cap: overflow)
  const uint32_t* tlim;    // [nq]
  uint2* list;             // [nq][nseg][cap]
  uint32_t* cnt;           // [nq][nseg]
  int64_t cap;
  int nseg;                // segment stride (>= grid size)
  int rot;                 // producers take chunks by global index (see first_of)
  int exp;                 // dev profiling knobs (HSB200_TC_EXP: 1 epilogue drain only, 2 no TMEM
                           // stores, 8 no MMAs, 16 unused, 32 no code loads, 64 no pass appends; build with -DHS_TCPROF for per-warp wait cycles), results invalid when set
  uint32_t tmax;           // 255*K + 1: no total reaches it
  int64_t ngroups;
  int64_t nblocks;         // point blocks of 128
  int64_t items_per_cta;   // contiguous (group, block) items per CTA
};

// One-hot words of 8 full subspaces: word 4s + i = 1 << (8*code - 32*i) when
// that shift is in [0, 32), else 0 — one clamped funnel shift per word (an
// out-of-range or "negative" unsigned shift clamps to 32 and yields the zero
// low half).
__device__ __forceinline__ void onehot8_full(uint32_t w, uint32_t* r) {
#pragma unroll
  for (int s = 0; s < kKC; ++s) {
    const uint32_t c8 = s == 0 ? (w << 3) & 0x78u : (w >> (4 * s - 3)) & 0x78u;
#pragma unroll
    for (int i = 0; i < 4; ++i) r[4 * s + i] = __funnelshift_lc(0u, 1u, c8 - 32u * i);
  }
}

// One-hot words of 8 subspaces: word 4s + i has byte (code & 3) = 1 when
// (code >> 2) == i, for the code of subspace s (its 16-byte K row); subspaces
// at or past `valid` are all zero.
__device__ __forceinline__ void onehot8(uint32_t w, int valid, uint32_t* r) {
#pragma unroll
  for (int s = 0; s < kKC; ++s) {
    const uint32_t code = (w >> (4 * s)) & 15u;
    const uint32_t bit = s < valid ? 1u << (8 * (code & 3u)) : 0u;
    const uint32_t c4 = code >> 2;
    r[4 * s + 0] = c4 == 0 ? bit : 0u;
    r[4 * s + 1] = c4 == 1 ? bit : 0u;
    r[4 * s + 2] = c4 == 2 ? bit : 0u;
    r[4 * s + 3] = c4 == 3 ? bit : 0u;
  }
}

// MAXC >= code words (8 subspaces each) per point; KC = subspaces per A ring
// slot (8: 32 TMEM columns, 4 MMAs; 16: 64 columns, 8 MMAs — fewer handoffs
// per MMA when N is small)
//
// PAIR (cta_group::2): a cluster of two CTAs on the SMs of one TPC works on
// 256-point blocks — each CTA generates the one-hot rows of its 128 points
// into its own TMEM — against NQ queries, each CTA holding the tables of NQ/2
// of them; the leader (rank 0) issues M=256 x N=NQ MMAs that read A from both
// CTAs' TMEM and B from both CTAs' shared memory, and each CTA's accumulator
// holds its 128 points x all NQ queries.  The one-hot expansion (the
// producers' work) is thus shared by twice the queries a single CTA's shared
// memory can hold.  Barriers: afull / dempty live in the leader (the peer's
// producers / epilogue arrive remotely), aempty / dfull in both (multicast
// commits).
template <int MAXC, bool FILTER, int KC, bool PAIR>
__global__ void __launch_bounds__(PAIR ? kThreadsPair : kThreadsTc, 1)
    k_lut16_tc(TcArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int NQ = a.nq_grp;                 // MMA N (queries per group)
  const int NQL = PAIR ? NQ / 2 : NQ;      // queries whose tables this CTA holds
  constexpr int PB = PAIR ? 2 * kPM : kPM; // points per block (item)
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  unsigned char* sB = smem_raw;  // [Kp][NQL][16]
  uint16_t* sStage = reinterpret_cast<uint16_t*>(sB + (size_t)a.Kp * NQL * 16);  // epilogue staging
  // filter mode: the staging area holds each epilogue warp's totals for the
  // (rare) pass appends; per-query 65536 - threshold and segment counts follow
  uint32_t* sNt = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sStage) + kStageBytes);
  uint32_t* sCnt = sNt + kMaxNQ;                           // filter mode: [NQ] segment counts
  uint64_t* bars = reinterpret_cast<uint64_t*>(sCnt + kMaxNQ);
  uint64_t* afull = bars;              // [slots] producers -> MMA (count 128)
  uint64_t* aempty = afull + a.slots;  // [slots] MMA commit -> producers
  uint64_t* dfull = aempty + a.slots;  // [2]     MMA commit -> epilogue
  uint64_t* dempty = dfull + 2;        // [2]     epilogue -> MMA (count 128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);
  uint32_t* sink = tmem_slot + 4;  // [slots][4] + [2][kEpi] landing words of the peer's st.async signals

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t cta_item = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t it0 = cta_item * a.items_per_cta;
  const int64_t it1 = min(a.ngroups * a.nblocks, it0 + a.items_per_cta);
  if (it0 >= it1) return;
  constexpr int NW = KC / kKC;       // code words per chunk
  constexpr int SC = 4 * KC;         // TMEM columns per A slot
  const int nkc = (a.Kp + KC - 1) / KC;  // chunks per block
  const int nwords = (a.Kp + kKC - 1) / kKC;

  if (warp == kMmaWarp) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    for (int s = 0; s < a.slots; ++s) {
      // pair: the leader's afull counts its own producer warps plus either
      // the peer's (remote arrives) or the peer's forwarding warp (one)
      mbar_init(&afull[s], PAIR && rank == 0 && !HS_TC_ASYNC ? kProd + (HS_TC_FWD ? 1 : kProd) : kProd);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], PAIR && !HS_TC_ASYNC ? 2 * kEpi : kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync_all();  // both CTAs' barriers and TMEM exist before any remote arrive
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // where this CTA's producers / epilogue arrive: the leader's barriers
  const uint32_t afull_r = PAIR ? peer_addr(afull, 0) : 0u;
  const uint32_t dempty_r = PAIR ? peer_addr(dempty, 0) : 0u;
  const uint32_t sink_r = PAIR ? peer_addr(sink, 0) : 0u;
  const bool remote = PAIR && rank != 0;
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + 2u * (uint32_t)NQ;  // A ring after the two accumulators

  // Items are (group, block) pairs in group-major order; a CTA's contiguous
  // range spans few groups.  Per group segment: load the group's tables into
  // shared memory, then stream its blocks through the pipeline.  Pipeline
  // counters run across segments so the barrier parities stay in step.
#ifdef HS_TCPROF  // per-role wait cycles, printed for two CTAs (dev builds only)
  long long tw0 = 0, tw1 = 0, tw2 = 0, tw3 = 0, tw4 = 0, tw5 = 0;
  const long long tstart = clock64();
#define TC_T0() const long long t0 = clock64()
#define TC_ACC(v) v += clock64() - t0
#else
#define TC_T0() (void)0
#define TC_ACC(v) (void)0
#endif
  int64_t blk_it = 0;
  int slot = 0;          // A ring position (the issuer walks every chunk)
  uint32_t round = 0;    // completed passes over the ring
  int pslot = 0;         // producers: ring position of global chunk pg
  uint32_t pround = 0;
  int64_t pg = 0;
  int64_t ep_tile = 0;  // epilogue tiles issued by this thread (staging parity)
  for (int64_t seg = it0; seg < it1;) {
    const int64_t g = seg / a.nblocks;
    const int64_t b0 = seg % a.nblocks;
    const int64_t b1 = min(a.nblocks, b0 + (it1 - seg));
    const int64_t q0 = g * NQ;
    const int64_t nblk = b1 - b0;
    // this CTA's list segment among the CTAs covering group g
    const int64_t seg_id = PAIR ? 2 * (cta_item - (g * a.nblocks) / a.items_per_cta) + rank
                                : cta_item - (g * a.nblocks) / a.items_per_cta;
    // ---- B: the group's tables, [k][q][16] (this CTA's half in PAIR mode).
    // Safe to overwrite: the previous segment's epilogue (both CTAs') waited
    // for its last dfull commit, which tracks every earlier MMA, before
    // reaching this barrier.
    if (PAIR) cluster_sync_all();
    else __syncthreads();
    {
      const int rows = a.Kp * NQL;
      const int64_t qb = q0 + (int64_t)rank * NQL;
      for (int i = tid; i < rows; i += blockDim.x) {
        const int k = i / NQL, q = i - k * NQL;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (qb + q < a.nq)
          v = __ldg(reinterpret_cast<const uint4*>(a.luts + ((qb + q) * a.Kp + k) * 16));
        *reinterpret_cast<uint4*>(sB + (size_t)i * 16) = v;
      }
      if (FILTER)  // 65536 - threshold (host guarantees tmax = 255*K + 1 <= 0xFFFF)
        for (int i = tid; i < NQ; i += blockDim.x) {
          const int64_t q = q0 + i;
          const uint32_t t = q < a.nq ? min(__ldg(a.tlim + q), a.tmax) : a.tmax;
          sNt[i] = 65536u - t;
        }
      if (FILTER)
        for (int i = tid; i < NQ; i += blockDim.x) sCnt[i] = 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (PAIR) cluster_sync_all();  // both halves of B in place before the leader's MMAs
    else __syncthreads();

    if (warp < kProdWarps) {
      // ---- producers: one-hot A chunks into the TMEM ring ----
      // kNPar warps per TMEM lane quadrant take K chunks round-robin, so one
      // warp's tcgen05.st / barrier latency overlaps the others' generation.
      const int quad = warp & 3, par = warp >> 2;
      const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
      // this warp's code words of a block (words of its chunks; others 0),
      // loaded one block ahead so the load latency hides behind the MMAs
      constexpr int NCH = (MAXC + NW - 1) / NW;              // max chunks per block
      constexpr int OW = ((NCH + kNPar - 1) / kNPar) * NW;   // words of this warp's chunks
      uint32_t nxt[OW];  // own chunk oc = c/kNPar: words oc*NW + h
      // A quadrant's kNPar warps take the chunks c = par (mod kNPar) of every
      // block.  The parity wait on a slot's `aempty` barrier is exact only
      // while a warp revisits the ring at most `slots` chunks after its
      // previous chunk; across a block boundary the fixed residue can leave a
      // longer gap (14 chunks per block: chunks 11 -> 2 of the next block are
      // 5 apart on a 4-slot ring).  For such shapes (a.rot, decided by the
      // host) chunks go by their GLOBAL index (block * nkc + c) mod kNPar —
      // always kNPar apart.  (Not by default: 2-3% slower at K = 128.)
      // first_of(bi) = this warp's first chunk of block bi.
      auto first_of = [&](int64_t bi) -> int {
        if constexpr (NW == 1 && HS_TC_PREGEN && HS_TC_ROLLED) {
          if (!a.rot) return par;  // the fixed residue is safe for this shape (and measured faster)
          const int base = (int)(((blk_it + bi) * (int64_t)nkc) % kNPar);
          return (par - base + kNPar) % kNPar;
        } else {
          return par;
        }
      };
      auto load_block = [&](int64_t bi) {
        const int64_t p = (b0 + bi) * PB + rank * kPM + quad * 32 + lane;
        const bool live = bi < nblk && p < a.n;
        const int role = first_of(bi);
#pragma unroll
        for (int i = 0; i < OW; ++i) {
          const int w = (kNPar * (i / NW) + role) * NW + (i % NW);
          if (a.exp & 32) {
            nxt[i] = (uint32_t)(p * 2654435761u + w);
          } else {
            // volatile asm: the load issues HERE, a block ahead of its use
            // (the compiler sank plain __ldg loads to the point of use, so
            // every block start waited a full memory latency)
            uint32_t v = 0u;
            const uint32_t* src = a.hcodes + ((p >> 7) * a.nwords + w) * kPM + (p & (kPM - 1));
            if (live && w < nwords) {
#if HS_TC_LDMODE == 0
              asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(src));
#elif HS_TC_LDMODE == 1
              asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(src));
#else
              v = __ldg(src);
#endif
            }
            nxt[i] = v;
          }
        }
      };
      load_block(0);
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t p = (b0 + bi) * PB + rank * kPM + quad * 32 + lane;
        const bool live = p < a.n;
        uint32_t cur[OW];
        {
          TC_T0();
#pragma unroll
          for (int i = 0; i < OW; ++i) cur[i] = nxt[i];
#ifdef HS_TCPROF
          // make the timer see the loads' completion
          uint32_t acc = 0;
#pragma unroll
          for (int i = 0; i < OW; ++i) acc ^= cur[i];
          if (acc == 0x12345678u) tw4 += 1;
#endif
          TC_ACC(tw4);
        }
        {
          TC_T0();
          load_block(bi + 1);
          TC_ACC(tw5);
        }
        // ring position of chunk c of this block: global chunk index g =
        // (blocks so far) * nkc + c, slot = g mod slots, round = g / slots —
        // advanced incrementally over this warp's own chunks only
        const int64_t g0 = (blk_it + bi) * (int64_t)nkc;
        if constexpr (NW == 1 && HS_TC_PREGEN && HS_TC_ROLLED) {
          // This warp's own chunks c = par, par + kNPar, ... in a ROLLED loop:
          // one copy of the chunk code.  (Unrolled over the 16 chunks of a
          // block the producers' code ran to ~40 KB, each warp walking a
          // different third of it — ncu showed as many instruction-fetch
          // stalls as issued instructions.)  The chunk's code word is always
          // cur[0]; the remaining words shift down.
#pragma unroll 1
          for (int c = first_of(bi); c < nkc; c += kNPar) {
            const uint32_t w = cur[0];
#pragma unroll
            for (int i = 0; i + 1 < OW; ++i) cur[i] = cur[i + 1];
            const int64_t gch = g0 + c;
            pslot += (int)(gch - pg);
            pg = gch;
            while (pslot >= a.slots) {
              pslot -= a.slots;
              ++pround;
            }
            const int slot = pslot;
            const uint32_t round = pround;
            uint32_t r[32];
            {
              TC_T0();
              if (live && (c + 1) * kKC <= a.K) onehot8_full(w, r);
              else onehot8(w, live ? min(kKC, a.K - c * kKC) : 0, r);
#ifdef HS_TCPROF
              uint32_t acc = 0;
#pragma unroll
              for (int i = 0; i < 32; ++i) acc ^= r[i];
              if (acc == 0x12345678u) tw3 += 1;
#endif
              TC_ACC(tw3);
            }
            if (round > 0) {
              TC_T0();
              mbar_wait_sleep(&aempty[slot], (round - 1) & 1u, HS_TC_SLEEP_PROD);
              TC_ACC(tw0);
              asm volatile("tcgen05.fence::after_thread_sync;");
            }
            {
              TC_T0();
              if (!(a.exp & 2)) TMEM_ST32(tmem_a + lane_base + (uint32_t)(slot * SC), r);
              if (!(a.exp & 2)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              TC_ACC(tw1);
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();  // the warp's stores are complete (wait::st is warp-wide): one arrive
            {
              TC_T0();
              if (!HS_TC_WARP_ARRIVE || lane == 0) {
                if (PAIR && HS_TC_ASYNC) {
                  if (remote)
                    st_async_signal(sink_r + 4u * (uint32_t)(slot * 4 + quad),
                                    afull_r + 8u * (uint32_t)slot);
                  else
                    mbar_arrive_expect(&afull[slot], 4u);  // + the peer quadrant's 4 bytes
                } else if (remote && !HS_TC_FWD) mbar_arrive_remote(afull_r + 8u * (uint32_t)slot);
                else mbar_arrive(&afull[slot]);
              }
              __syncwarp();
              TC_ACC(tw2);
            }
          }
        } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c >= nkc) break;
          if ((c % kNPar) == par) {
            const int64_t gch = g0 + c;
            pslot += (int)(gch - pg);
            pg = gch;
            while (pslot >= a.slots) {
              pslot -= a.slots;
              ++pround;
            }
            const int slot = pslot;
            const uint32_t round = pround;
            if (NW == 1 && HS_TC_PREGEN) {
              // one 32-column store per chunk: generate the one-hot words
              // first, then wait for the slot — the generation overlaps the
              // wait, and a freed slot is refilled with one store + arrive
              uint32_t r[32];
              {
                TC_T0();
                if (live && (c + 1) * kKC <= a.K) {
                  onehot8_full(cur[c / kNPar], r);
                } else {
                  onehot8(cur[c / kNPar], live ? min(kKC, a.K - c * kKC) : 0, r);
                }
#ifdef HS_TCPROF
                uint32_t acc = 0;
#pragma unroll
                for (int i = 0; i < 32; ++i) acc ^= r[i];
                if (acc == 0x12345678u) tw3 += 1;
#endif
                TC_ACC(tw3);
              }
              if (round > 0) {
                TC_T0();
                mbar_wait_sleep(&aempty[slot], (round - 1) & 1u, HS_TC_SLEEP_PROD);
                TC_ACC(tw0);
                asm volatile("tcgen05.fence::after_thread_sync;");
              }
              {
                TC_T0();
                if (!(a.exp & 2)) TMEM_ST32(tmem_a + lane_base + (uint32_t)(slot * SC), r);
                if (!(a.exp & 2)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                TC_ACC(tw1);
              }
            } else {
            if (round > 0) {
              TC_T0();
              mbar_wait_sleep(&aempty[slot], (round - 1) & 1u, HS_TC_SLEEP_PROD);
              TC_ACC(tw0);
              asm volatile("tcgen05.fence::after_thread_sync;");
            }
#pragma unroll
            for (int h = 0; h < NW; ++h) {  // 32 columns (8 subspaces) per store
              uint32_t r[32];
              if (live && (c * NW + h + 1) * kKC <= a.K) {
                onehot8_full(cur[(c / kNPar) * NW + h], r);
              } else {
                onehot8(cur[(c / kNPar) * NW + h], live ? min(kKC, a.K - (c * NW + h) * kKC) : 0, r);
              }
              if (!(a.exp & 2)) TMEM_ST32(tmem_a + lane_base + (uint32_t)(slot * SC + 32 * h), r);
            }
            }
            if (!(a.exp & 2)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();  // the warp's stores are complete (wait::st is warp-wide): one arrive
            {
              TC_T0();
              if (!HS_TC_WARP_ARRIVE || lane == 0) {
                if (PAIR && HS_TC_ASYNC) {
                  if (remote)
                    st_async_signal(sink_r + 4u * (uint32_t)(slot * 4 + quad),
                                    afull_r + 8u * (uint32_t)slot);
                  else
                    mbar_arrive_expect(&afull[slot], 4u);  // + the peer quadrant's 4 bytes
                } else if (remote && !HS_TC_FWD) mbar_arrive_remote(afull_r + 8u * (uint32_t)slot);
                else mbar_arrive(&afull[slot]);
              }
              __syncwarp();
              TC_ACC(tw2);
            }
          }
        }
        }  // unrolled form (wide slots / no pre-generation)
      }
    } else if (warp < kMmaWarp) {
      // ---- epilogue: accumulator -> u16 totals [query][point] ----
      // kEpiPar warps per TMEM lane quadrant take alternate 32-column tiles.
      // Per 32x32 tile (32 points of this warp's lanes x 32 queries): the
      // tile is transposed through shared memory (conflict-free u16 stores,
      // one query row per 64 B) and one lane hands it to the TMA engine as a
      // 2-D tensor store; two staging buffers per warp.
      const int quad = warp & 3, half = (warp - kEpiWarp0) >> 2;
      const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
      uint16_t* stg = sStage + (warp - kEpiWarp0) * 2 * 1024;
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t bt = blk_it + bi;
        const int buf = (int)(bt & 1);
        TC_T0();
        mbar_wait_sleep(&dfull[buf], (uint32_t)((bt >> 1) & 1), HS_TC_SLEEP_EPI);
        TC_ACC(tw0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int64_t pbase = (b0 + bi) * PB + rank * kPM + quad * 32;
        if (half * 32 >= NQ) {  // no tile of this block for this warp
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (!HS_TC_WARP_ARRIVE || lane == 0) {
            if (PAIR && HS_TC_ASYNC) {
              if (remote)
                st_async_signal(sink_r + 4u * (uint32_t)(4 * a.slots + buf * kEpi + (warp - kEpiWarp0)),
                                dempty_r + 8u * (uint32_t)buf);
              else
                mbar_arrive_expect(&dempty[buf], 4u);  // + the peer warp's 4 bytes
            } else if (remote) mbar_arrive_remote(dempty_r + 8u * (uint32_t)buf);
            else mbar_arrive(&dempty[buf]);
          }
        }
        for (int c = half * 32; c < NQ; c += 32 * kEpiPar) {
          if (FILTER) {
            // emit the (point, total) pairs at or above the query's
            // threshold, 16 columns at a time.  Totals are < 2^16, so s_j =
            // total_j + (65536 - t_q) has bit 16 set iff total_j >= t_q: one
            // add per column, OR-reduced (in place: r[j] becomes s_j; the
            // rare path recovers the total)
            const int64_t p = pbase + lane;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int c16 = c + 16 * hh;
              uint32_t r[16];
              TMEM_LD16(tmem + lane_base + (uint32_t)(buf * NQ + c16), r);
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
              if (hh == 1 && c + 32 * kEpiPar >= NQ) {  // this warp's part read: release
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();  // wait::ld is warp-wide: one arrive per warp
                if (!HS_TC_WARP_ARRIVE || lane == 0) {
                  if (PAIR && HS_TC_ASYNC) {
                    if (remote)
                      st_async_signal(sink_r + 4u * (uint32_t)(4 * a.slots + buf * kEpi + (warp - kEpiWarp0)),
                                      dempty_r + 8u * (uint32_t)buf);
                    else
                      mbar_arrive_expect(&dempty[buf], 4u);  // + the peer warp's 4 bytes
                  } else if (remote) mbar_arrive_remote(dempty_r + 8u * (uint32_t)buf);
                  else mbar_arrive(&dempty[buf]);
                }
              }
              if (a.exp & 1) continue;  // profiling knob: drain only
              uint32_t og[4];  // per group of 4 columns: OR of the s_j
              const uint4* nt4 = reinterpret_cast<const uint4*>(sNt + c16);
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const uint4 t4 = nt4[g];
                r[4 * g + 0] += t4.x;
                r[4 * g + 1] += t4.y;
                r[4 * g + 2] += t4.z;
                r[4 * g + 3] += t4.w;
                og[g] = (r[4 * g + 0] | r[4 * g + 1]) | (r[4 * g + 2] | r[4 * g + 3]);
              }
              const uint32_t orr = (og[0] | og[1]) | (og[2] | og[3]);
              if ((orr & 0x10000u) != 0u && p < a.n && !(a.exp & 64)) {  // rare: this lane's passes
                // (a warp enters when any of its 32 lanes has a pass in these 16
                // columns — a quarter of the time at config 5 — so the path is
                // short: group ORs narrow the search to 4 columns, every
                // register index is static, the total is s_j minus the staged
                // 65536 - t_q)
                const int64_t lstride = (int64_t)a.nseg * a.cap;  // list entries per query
                uint2* lq = a.list + ((q0 + c16) * a.nseg + seg_id) * a.cap;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                  if (!(og[g] & 0x10000u)) continue;
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const int j = 4 * g + i;
                    if (!(r[j] & 0x10000u)) continue;
                    const uint32_t val = r[j] - sNt[c16 + j];
                    const uint32_t pos = atomicAdd(sCnt + c16 + j, 1u);  // this CTA's segment of q
                    if (pos < (uint32_t)a.cap) lq[j * lstride + pos] = make_uint2((uint32_t)p, val);
                  }
                }
              }
            }
            continue;
          }
          uint32_t r[32];
          TMEM_LD32(tmem + lane_base + (uint32_t)(buf * NQ + c), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 32 * kEpiPar >= NQ) {  // this warp's part of the accumulator read: release
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();  // wait::ld is warp-wide: one arrive per warp
            if (!HS_TC_WARP_ARRIVE || lane == 0) {
              if (PAIR && HS_TC_ASYNC) {
                if (remote)
                  st_async_signal(sink_r + 4u * (uint32_t)(4 * a.slots + buf * kEpi + (warp - kEpiWarp0)),
                                  dempty_r + 8u * (uint32_t)buf);
                else
                  mbar_arrive_expect(&dempty[buf], 4u);  // + the peer warp's 4 bytes
              } else if (remote) mbar_arrive_remote(dempty_r + 8u * (uint32_t)buf);
              else mbar_arrive(&dempty[buf]);
            }
          }
          if (a.exp & 1) continue;  // profiling knob: drain only
          const int sb = (int)(ep_tile & 1);
          if (ep_tile >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          uint16_t* t = stg + sb * 1024;
#pragma unroll
          for (int j = 0; j < 32; ++j) t[j * 32 + lane] = (uint16_t)r[j];
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (q0 + c < a.nq) tma_store_tile(&tmap, t, (int)pbase, (int)(q0 + c));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++ep_tile;
        }
      }
    } else if (warp >= kFwdWarp0) {
      // ---- pair forwarders (peer only): relay this CTA's completed A slots ----
      if constexpr (kFwd > 0)
      if (PAIR && rank != 0)
        for (int64_t bi = 0; bi < nblk; ++bi)
          for (int c = 0; c < nkc; ++c) {
            if (slot % (kFwd > 0 ? kFwd : 1) == warp - kFwdWarp0) {
              mbar_wait(&afull[slot], round & 1u);
              if (lane == 0) mbar_arrive_remote(afull_r + 8u * (uint32_t)slot);
              __syncwarp();
            }
            if (++slot == a.slots) {
              slot = 0;
              ++round;
            }
          }
    } else if (!PAIR || rank == 0) {
      // ---- MMA issuer: warp-uniform control flow (descriptors stay in
      // uniform registers), one elected lane issues the MMAs and commits.
      // (A single-thread loop without the per-chunk elect / warp sync was
      // measured slower: 38.2 vs 31.4 ms, cfg5 law at 10^7 points.) ----
      const uint32_t idesc = PAIR ? ((idesc_u8(NQ) & ~(31u << 24)) | ((uint32_t)(2 * kPM >> 4) << 24))
                                  : idesc_u8(NQ);
      const uint64_t bdesc0 = smem_desc(smem_u32(sB), (uint32_t)(NQL * 16), 128);
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t bt = blk_it + bi;
        const int buf = (int)(bt & 1);
        if (bt >= 2) {
          TC_T0();
          mbar_wait_mma(&dempty[buf], (uint32_t)(((bt >> 1) - 1) & 1));
          TC_ACC(tw1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t d = tmem + (uint32_t)(buf * NQ);
        for (int c = 0; c < nkc; ++c) {
          TC_T0();
          mbar_wait_mma(&afull[slot], round & 1u);
          TC_ACC(tw0);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int npair = min(KC, a.Kp - c * KC) / 2;  // Kp even
          const uint32_t ta = tmem_a + (uint32_t)(slot * SC);
          // B start address advances by NQL*16 bytes per subspace: +NQL in
          // the descriptor's (address >> 4) field
          const uint64_t bd = bdesc0 + (uint64_t)(c * KC * NQL);
          if (elect_one()) {
            if (!(a.exp & 8)) {
              if (PAIR) {
                mma_ts2(d, ta, bd, idesc, c > 0 ? 1u : 0u);
#pragma unroll
                for (int m = 1; m < KC / 2; ++m)
                  if (npair > m) mma_ts2(d, ta + 8 * m, bd + (uint64_t)(2 * m * NQL), idesc, 1u);
              } else {
                mma_ts(d, ta, bd, idesc, c > 0 ? 1u : 0u);
#pragma unroll
                for (int m = 1; m < KC / 2; ++m)
                  if (npair > m) mma_ts(d, ta + 8 * m, bd + (uint64_t)(2 * m * NQL), idesc, 1u);
              }
            }
            if (PAIR) mma_commit2(&aempty[slot]);
            else mma_commit(&aempty[slot]);
          }
          __syncwarp();
          if (++slot == a.slots) {
            slot = 0;
            ++round;
          }
        }
        if (elect_one()) {
          if (PAIR) mma_commit2(&dfull[buf]);
          else mma_commit(&dfull[buf]);
        }
        __syncwarp();
      }
    }  // (the pair peer's MMA warp idles: the leader issues)
    blk_it += nblk;
    seg += nblk;
    if (FILTER) {  // publish this CTA's segment counts of the group
      __syncthreads();
      for (int i = tid; i < NQ; i += blockDim.x)
        if (q0 + i < a.nq) a.cnt[(q0 + i) * a.nseg + seg_id] = sCnt[i];
    }
  }
  if (!FILTER && warp >= kEpiWarp0 && warp < kMmaWarp && lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef HS_TCPROF
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 1))
    printf("TCPROF cta=%d warp=%d total=%lld wait0=%lld wait1=%lld t2=%lld gen=%lld blk=%lld ldi=%lld items=%lld\n",
           (int)blockIdx.x, warp, clock64() - tstart, tw0, tw1, tw2, tw3, tw4, tw5, (long long)(it1 - it0));
#endif
  if (PAIR) cluster_sync_all();  // the peer's epilogue and the leader's MMAs are done
  else __syncthreads();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
  }
}

// pair-major packed codes (dense.py:156-170) -> blocked u32 code words:
// block b of 128 points holds [ceil(K/8)][128] words, nibble s of word (c, p)
// = code of subspace 8c+s of point p (zero past K).  A block's codes are one
// contiguous 512*ceil(K/8)-byte run (8 KB at K=128): the producers' loads of
// a block stay within one page (the row-major [word][n] layout put the rows
// n*4 bytes apart, and the per-block loads took TLB misses: ~30% of the
// kernel at 4*10^7 points, HS_TCPROF)
__global__ void k_to_hcodes(const uint8_t* __restrict__ packed, int64_t n, int npairs, int nw,
                            uint32_t* __restrict__ h) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (p >= ((n + kPM - 1) / kPM) * kPM) return;
  uint32_t w = 0;
  if (p < n) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int pair = 4 * c + t;
      if (pair < npairs) w |= (uint32_t)packed[(int64_t)pair * n + p] << (8 * t);
    }
  }
  h[((p >> 7) * nw + c) * kPM + (p & (kPM - 1))] = w;
}

int pick_nq(int Kp, int64_t nq) {
  const int64_t by_smem = (int64_t)(kSmemBudget - 1024) / ((int64_t)Kp * 16);
  // (<= 192: two accumulators of NQ columns must leave a ring of at least four
  // 32-column A slots in the 512 TMEM columns)
  int64_t v = std::min<int64_t>(192, std::min<int64_t>(kMaxNQ, by_smem)) / 32 * 32;
  const int64_t need = ceil_div(nq, 32) * 32;  // small batches: no idle columns
  if (need < v) v = need;
  return (int)std::max<int64_t>(v, 0);
}

// CTA-pair mode: each CTA holds the tables of half the group, so the group
// (MMA N) doubles — up to 192 (two double-buffered accumulators + a 128-column
// A ring fill the 512 TMEM columns); used when one CTA's shared memory holds
// fewer than 128 queries' tables (K > 96), where the single-CTA group leaves
// the producers' one-hot work amortised over too few queries.
constexpr int kPairMaxN = 192;
int pair_max_n() {
  static const int v = std::getenv("HSB200_TC_PAIRN") ? std::atoi(std::getenv("HSB200_TC_PAIRN"))
                                                      : kPairMaxN;
  return v;
}
bool pair_mode(int Kp) {
  static const char* e = std::getenv("HSB200_TC_PAIR");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return 2 * pick_nq(Kp, 1LL << 40) >= 64;
  return pick_nq(Kp, 1LL << 40) < 128 && 2 * pick_nq(Kp, 1LL << 40) >= 128;
}
int pick_group(int Kp, int64_t nq) {
  if (!pair_mode(Kp)) return pick_nq(Kp, nq);
  int64_t v = std::min<int64_t>(pair_max_n(), 2 * (int64_t)pick_nq(Kp, 1LL << 40)) / 32 * 32;
  const int64_t need = ceil_div(nq, 32) * 32;
  if (need < v) v = need;
  return (int)v;
}

}  // namespace

bool lut16_tc_supported(const DeviceIndex& ix) {
  return ix.hcodes != nullptr && ix.K > 0 && ix.K <= 257 && pick_nq(ix.Kp, 1LL << 40) >= 32;
}

int64_t lut16_tc_ld(int64_t n) { return ((n + kPM - 1) / kPM) * kPM; }

int64_t lut16_tc_group(const DeviceIndex& ix) { return pick_group(ix.Kp, 1LL << 40); }


int64_t hcodes_words(int64_t n, int K) { return ceil_div(n, kPM) * kPM * ceil_div(K, kKC); }

void launch_to_hcodes(const uint8_t* packed, int64_t n, int K, uint32_t* h, cudaStream_t st) {
  if (n <= 0 || K <= 0) return;
  const int nkc = (K + kKC - 1) / kKC;
  dim3 grid((unsigned)ceil_div(ceil_div(n, kPM) * kPM, 256), (unsigned)nkc);
  k_to_hcodes<<<grid, 256, 0, st>>>(packed, n, (K + 1) / 2, nkc, h);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

namespace {

struct TcLayout {
  int NQ;
  bool pair;
  int64_t ngroups, nblocks, items_per_cta, grid, nseg;
  double frac;  // largest share of a query's points one CTA (list segment) covers
};

TcLayout tc_layout(const DeviceIndex& ix, int64_t nq, int64_t n) {
  TcLayout L;
  L.pair = pair_mode(ix.Kp);
  L.NQ = pick_group(ix.Kp, nq);
  L.ngroups = ceil_div(nq, L.NQ);
  const int64_t pb = L.pair ? 2 * kPM : kPM;
  L.nblocks = ceil_div(n, pb);
  // one CTA per SM (it owns all of TMEM), equal contiguous shares of the
  // (group, block) items per CTA (per CTA pair in pair mode)
  const int64_t units = L.pair ? kNumSMs / 2 : kNumSMs;
  const int64_t items = L.ngroups * L.nblocks;
  const int64_t ctas = std::min<int64_t>(units, items);
  L.items_per_cta = ceil_div(items, ctas);
  const int64_t used = ceil_div(items, L.items_per_cta);
  L.grid = L.pair ? 2 * used : used;
  // CTAs covering one group: its items span at most this many CTA ranges
  const int64_t spans = std::min<int64_t>(used, ceil_div(L.nblocks, L.items_per_cta) + 1);
  L.nseg = L.pair ? 2 * spans : spans;
  L.frac = std::min(1.0, (double)L.items_per_cta * kPM / (double)std::max<int64_t>(n, 1));
  return L;
}

int launch_tc(const DeviceIndex& ix, const uint8_t* luts, int64_t nq, int64_t n_limit,
              uint16_t* tot, int64_t ld, const uint32_t* tlim, uint2* list, uint32_t* cnt,
              int64_t cap, cudaStream_t st) {
  const int64_t n = n_limit >= 0 ? std::min(n_limit, ix.n) : ix.n;
  if (nq <= 0 || n <= 0) return HS_OK;
  if (!lut16_tc_supported(ix)) HS_FAIL(HS_EUNSUPPORTED, "tensor-core LUT16 unsupported for this index");
  const bool filter = list != nullptr;
  const TcLayout L = tc_layout(ix, nq, n);
  const int NQ = L.NQ;
  TcArgs a;
  a.n = n;
  a.nq = nq;
  a.K = ix.K;
  a.Kp = ix.Kp;
  a.nq_grp = NQ;
  const int nw = (int)ceil_div(a.Kp, kKC);
  static const int kc_env = std::getenv("HSB200_TC_KC") ? std::atoi(std::getenv("HSB200_TC_KC")) : 0;
  static const int slot_cap = std::getenv("HSB200_TC_SLOTS") ? std::atoi(std::getenv("HSB200_TC_SLOTS")) : 8;
  // wide slots for K<=128 (fewer handoffs per MMA); the pair's 128-column
  // ring takes 4 narrow slots instead of 2 wide ones
  // (the pair keeps 32-column slots: with 64-column slots its ring is only
  // two deep, which hung in a dev run)
  // (8-subspace slots everywhere: the rolled producer loop with the
  // global-index chunk assignment serves them; HSB200_TC_KC=16 keeps the wide
  // slots of the single-CTA form for A/B runs)
  const int KCsel = L.pair ? 8 : kc_env == 16 ? 16 : 8;
  a.slots = std::min(slot_cap, (kTmemCols - 2 * NQ) / (4 * KCsel));
  if (a.slots < 3) HS_FAIL(HS_EUNSUPPORTED, "tensor-core LUT16: TMEM too small for the ring");
  {
    // largest distance between a producer warp's consecutive chunks under the
    // fixed residue assignment (last chunk of a block -> first of the next)
    const int nkc = (a.Kp + KCsel - 1) / KCsel;
    int maxgap = 0;
    for (int r = 0; r < kNPar && r < nkc; ++r) {
      const int last = r + ((nkc - 1 - r) / kNPar) * kNPar;
      maxgap = std::max(maxgap, (nkc - last) + r);
    }
    a.rot = (maxgap > a.slots || getenv("HSB200_TC_ROT")) ? 1 : 0;
  }
  a.hcodes = ix.hcodes;
  a.luts = luts;
  a.tot = tot;
  a.ld = ld;
  a.nwords = (int)ceil_div(ix.K, kKC);
  a.tlim = tlim;
  a.list = list;
  a.cnt = cnt;
  a.cap = cap;
  a.nseg = (int)L.nseg;
  a.exp = std::getenv("HSB200_TC_EXP") ? std::atoi(std::getenv("HSB200_TC_EXP")) : 0;
  a.tmax = 255u * (uint32_t)ix.K + 1u;
  if (filter && a.tmax > 0xFFFFu) HS_FAIL(HS_EUNSUPPORTED, "filtered tensor-core pass needs K <= 256");
  a.ngroups = L.ngroups;
  a.nblocks = L.nblocks;
  a.items_per_cta = L.items_per_cta;
  const int64_t grid = L.grid;
  const int NQL = L.pair ? NQ / 2 : NQ;
  const size_t smem =
      (size_t)a.Kp * NQL * 16 + kStageBytes + 2 * kMaxNQ * sizeof(uint32_t) +
      (2 * a.slots + 4) * sizeof(uint64_t) + 16 + 16 * (size_t)a.slots + 4 * 2 * kEpi;
  void (*kern)(TcArgs, const CUtensorMap);
  if (L.pair) {
    if (filter)
      kern = nw <= 8 ? k_lut16_tc<8, true, 8, true>
             : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, true, 16, true> : k_lut16_tc<16, true, 8, true>)
                        : k_lut16_tc<33, true, 8, true>;
    else
      kern = nw <= 8 ? k_lut16_tc<8, false, 8, true>
             : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, false, 16, true> : k_lut16_tc<16, false, 8, true>)
                        : k_lut16_tc<33, false, 8, true>;
  } else if (filter) {
    kern = nw <= 8 ? k_lut16_tc<8, true, 8, false>
           : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, true, 16, false> : k_lut16_tc<16, true, 8, false>)
                      : k_lut16_tc<33, true, 8, false>;
  } else {
    kern = nw <= 8 ? k_lut16_tc<8, false, 8, false>
           : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, false, 16, false> : k_lut16_tc<16, false, 8, false>)
                      : k_lut16_tc<33, false, 8, false>;
  }
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (!filter) {
    if (ld % kPM != 0) HS_FAIL(HS_EINVAL, "tensor-core totals stride must be a multiple of 128");
    // totals [nq][ld] u16 as a 2-D tensor; 32x32 boxes, no swizzle
    auto enc = encode_fn();
    if (!enc) HS_FAIL(HS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t gdim[2] = {(cuuint64_t)ld, (cuuint64_t)nq};
    const cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(uint16_t)};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estride[2] = {1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, tot, gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      HS_FAIL(HS_ECUDA, "cuTensorMapEncodeTiled failed for the totals buffer");
  }
  if (L.pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreadsPair);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HS_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tmap));
  } else {
    kern<<<(unsigned)grid, kThreadsTc, smem, st>>>(a, tmap);
  }
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace

int launch_lut16_tc(const DeviceIndex& ix, const uint8_t* luts, int64_t nq, uint16_t* tot,
                    int64_t ld, cudaStream_t st, int64_t n_limit) {
  return launch_tc(ix, luts, nq, n_limit, tot, ld, nullptr, nullptr, nullptr, 0, st);
}

void lut16_filter_layout(const DeviceIndex& ix, int64_t nq, int64_t* nseg, double* frac) {
  const TcLayout L = tc_layout(ix, nq, ix.n);
  *nseg = L.nseg;
  *frac = L.frac;
}

int launch_lut16_filter(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                        const uint32_t* tlim, uint2* list, uint32_t* cnt, int64_t cap,
                        cudaStream_t st) {
  HS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * nq * tc_layout(ix, nq, ix.n).nseg, st));
  return launch_tc(ix, luts, nq, -1, nullptr, 0, tlim, list, cnt, cap, st);
}

}  // namespace hs
