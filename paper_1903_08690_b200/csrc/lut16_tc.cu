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

namespace hs {

namespace {

constexpr int kPM = 128;       // points per block (MMA M, TMEM lanes)
constexpr int kKC = 8;         // subspaces per code word (8 nibbles)
constexpr int kProd = 128;     // arrivals per A chunk (one producer warp per lane quadrant)
constexpr int kNPar = 3;       // producer warps per TMEM lane quadrant (round-robin over chunks)
constexpr int kEpiPar = 2;     // epilogue warps per lane quadrant (alternate 32-column tiles)
constexpr int kProdWarps = 4 * kNPar;
constexpr int kEpiWarp0 = kProdWarps;      // a multiple of 4: warp & 3 = lane quadrant
constexpr int kMmaWarp = kEpiWarp0 + 4 * kEpiPar;
constexpr int kEpi = 128 * kEpiPar;        // epilogue threads: dempty arrivals per block
constexpr int kThreadsTc = 32 * (kMmaWarp + 1);  // 12 producer, 8 epilogue, 1 MMA warps
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
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
  int slots;               // A ring slots (32 TMEM columns each)
  const uint32_t* hcodes;  // [ceil(K/8)][n]: nibble s = code of subspace 8c+s
  const uint8_t* luts;     // [nq][Kp][16]
  uint16_t* tot;           // [nq][ld] u16 totals (totals mode)
  int64_t ld;
  int64_t stride;          // hcodes row stride (points of the whole index)
  // filter mode: emit (point, total) with total >= tlim[q] into CTA-private
  // segments list[q][cta][cap] with counts cnt[q][cta] (> cap: overflow)
  const uint32_t* tlim;    // [nq]
  uint2* list;             // [nq][nseg][cap]
  uint32_t* cnt;           // [nq][nseg]
  int64_t cap;
  int nseg;                // segment stride (>= grid size)
  int exp;                 // dev profiling knobs (HSB200_TC_EXP: 1 epilogue drain only, 2 no TMEM
                           // stores, 8 no MMAs, 16 unused; build with -DHS_TCPROF for per-warp wait cycles), results invalid when set
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
template <int MAXC, bool FILTER, int KC>
__global__ void __launch_bounds__(kThreadsTc, 1)
    k_lut16_tc(TcArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int NQ = a.nq_grp;
  unsigned char* sB = smem_raw;  // [Kp][NQ][16]
  uint16_t* sStage = reinterpret_cast<uint16_t*>(sB + (size_t)a.Kp * NQ * 16);  // epilogue staging
  uint32_t* sTlim = reinterpret_cast<uint32_t*>(sStage);  // filter mode: [NQ/2] packed thresholds
  uint32_t* sCnt = sTlim + 128;                            // filter mode: [NQ] segment counts
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sStage) + kStageBytes);
  uint64_t* afull = bars;              // [slots] producers -> MMA (count 128)
  uint64_t* aempty = afull + a.slots;  // [slots] MMA commit -> producers
  uint64_t* dfull = aempty + a.slots;  // [2]     MMA commit -> epilogue
  uint64_t* dempty = dfull + 2;        // [2]     epilogue -> MMA (count 128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t it0 = (int64_t)blockIdx.x * a.items_per_cta;
  const int64_t it1 = min(a.ngroups * a.nblocks, it0 + a.items_per_cta);
  if (it0 >= it1) return;
  constexpr int NW = KC / kKC;       // code words per chunk
  constexpr int SC = 4 * KC;         // TMEM columns per A slot
  const int nkc = (a.Kp + KC - 1) / KC;  // chunks per block
  const int nwords = (a.Kp + kKC - 1) / kKC;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < a.slots; ++s) {
      mbar_init(&afull[s], kProd);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + 2u * (uint32_t)NQ;  // A ring after the two accumulators

  // Items are (group, block) pairs in group-major order; a CTA's contiguous
  // range spans few groups.  Per group segment: load the group's tables into
  // shared memory, then stream its blocks through the pipeline.  Pipeline
  // counters run across segments so the barrier parities stay in step.
#ifdef HS_TCPROF  // per-role wait cycles, printed for two CTAs (dev builds only)
  long long tw0 = 0, tw1 = 0;
  const long long tstart = clock64();
#define TC_T0() const long long t0 = clock64()
#define TC_ACC(v) v += clock64() - t0
#else
#define TC_T0() (void)0
#define TC_ACC(v) (void)0
#endif
  int64_t blk_it = 0;
  int slot = 0;          // A ring position (producers and issuer walk it in step)
  uint32_t round = 0;    // completed passes over the ring
  int64_t ep_tile = 0;  // epilogue tiles issued by this thread (staging parity)
  for (int64_t seg = it0; seg < it1;) {
    const int64_t g = seg / a.nblocks;
    const int64_t b0 = seg % a.nblocks;
    const int64_t b1 = min(a.nblocks, b0 + (it1 - seg));
    const int64_t q0 = g * NQ;
    const int64_t nblk = b1 - b0;
    // this CTA's list segment among the CTAs covering group g
    const int64_t seg_id = (int64_t)blockIdx.x - (g * a.nblocks) / a.items_per_cta;
    // ---- B: the group's tables, [k][q][16].  Safe to overwrite: the
    // previous segment's epilogue waited for its last dfull commit, which
    // tracks every earlier MMA, before reaching this barrier.
    __syncthreads();
    {
      const int rows = a.Kp * NQ;
      for (int i = tid; i < rows; i += blockDim.x) {
        const int k = i / NQ, q = i - k * NQ;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (q0 + q < a.nq)
          v = __ldg(reinterpret_cast<const uint4*>(a.luts + ((q0 + q) * a.Kp + k) * 16));
        *reinterpret_cast<uint4*>(sB + (size_t)i * 16) = v;
      }
      if (FILTER)  // pairs of u16 thresholds (host guarantees 255*K + 1 <= 0xFFFF)
        for (int i = tid; i < NQ / 2; i += blockDim.x) {
          uint32_t w = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t q = q0 + 2 * i + h;
            const uint32_t t = q < a.nq ? min(__ldg(a.tlim + q), a.tmax) : a.tmax;
            w |= t << (16 * h);
          }
          sTlim[i] = w;
        }
      if (FILTER)
        for (int i = tid; i < NQ; i += blockDim.x) sCnt[i] = 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

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
      auto load_block = [&](int64_t bi) {
        const int64_t p = (b0 + bi) * kPM + quad * 32 + lane;
        const bool live = bi < nblk && p < a.n;
#pragma unroll
        for (int i = 0; i < OW; ++i) {
          const int w = (kNPar * (i / NW) + par) * NW + (i % NW);
          if (a.exp & 32)
            nxt[i] = (uint32_t)(p * 2654435761u + w);
          else
            nxt[i] = (live && w < nwords) ? __ldg(a.hcodes + (int64_t)w * a.stride + p) : 0u;
        }
      };
      load_block(0);
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t p = (b0 + bi) * kPM + quad * 32 + lane;
        const bool live = p < a.n;
        uint32_t cur[OW];
#pragma unroll
        for (int i = 0; i < OW; ++i) cur[i] = nxt[i];
        load_block(bi + 1);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c >= nkc) break;
          if ((c % kNPar) == par) {
            if (round > 0) {
              TC_T0();
              mbar_wait(&aempty[slot], (round - 1) & 1u);
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
            if (!(a.exp & 2)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&afull[slot]);
          }
          if (++slot == a.slots) {
            slot = 0;
            ++round;
          }
        }
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
        mbar_wait(&dfull[buf], (uint32_t)((bt >> 1) & 1));
        TC_ACC(tw0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int64_t pbase = (b0 + bi) * kPM + quad * 32;
        if (half * 32 >= NQ) {  // no tile of this block for this warp
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(&dempty[buf]);
        }
        for (int c = half * 32; c < NQ; c += 32 * kEpiPar) {
          uint32_t r[32];
          TMEM_LD32(tmem + lane_base + (uint32_t)(buf * NQ + c), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 32 * kEpiPar >= NQ) {  // this warp's part of the accumulator read: release
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&dempty[buf]);
          }
          if (a.exp & 1) continue;  // profiling knob: drain only
          if (FILTER) {
            // emit the (point, total) pairs at or above the query's threshold:
            // packed u16x2 compares against the group's packed thresholds,
            // then each lane appends its (rare) passes with one atomic each
            const int64_t p = pbase + lane;
            uint32_t pm = 0;  // bit j: column c+j passes
            uint32_t vc[16];
            uint32_t any = 0;
            {
              const uint4* tl4 = reinterpret_cast<const uint4*>(sTlim + (c >> 1));
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const uint4 t4 = tl4[g];
                const uint32_t tw[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  const int j = 8 * g + 2 * h;
                  vc[j >> 1] = __vcmpgeu2(__byte_perm(r[j], r[j + 1], 0x5410), tw[h]);
                  any |= vc[j >> 1];
                }
              }
            }
            if (any != 0u && p < a.n) {  // rare: expand the lane's pass mask
#pragma unroll
              for (int i = 0; i < 16; ++i)
                pm |= ((vc[i] & 1u) | ((vc[i] >> 15) & 2u)) << (2 * i);
            }
            while (pm) {
              const int j = __ffs(pm) - 1;
              pm &= pm - 1;
              const int64_t q = q0 + c + j;
              const uint32_t pos = atomicAdd(sCnt + c + j, 1u);  // this CTA's segment of q
              uint32_t val = 0;
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) val = jj == j ? r[jj] : val;
              if (pos < (uint32_t)a.cap)
                a.list[(q * a.nseg + seg_id) * a.cap + pos] = make_uint2((uint32_t)p, val);
            }
            continue;
          }
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
    } else {
      // ---- MMA issuer: warp-uniform control flow (descriptors stay in
      // uniform registers), one elected lane issues the MMAs and commits ----
      const uint32_t idesc = idesc_u8(NQ);
      const uint64_t bdesc0 = smem_desc(smem_u32(sB), (uint32_t)(NQ * 16), 128);
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t bt = blk_it + bi;
        const int buf = (int)(bt & 1);
        if (bt >= 2) {
          TC_T0();
          mbar_wait(&dempty[buf], (uint32_t)(((bt >> 1) - 1) & 1));
          TC_ACC(tw1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t d = tmem + (uint32_t)(buf * NQ);
        for (int c = 0; c < nkc; ++c) {
          TC_T0();
          mbar_wait(&afull[slot], round & 1u);
          TC_ACC(tw0);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int npair = min(KC, a.Kp - c * KC) / 2;  // Kp even
          const uint32_t ta = tmem_a + (uint32_t)(slot * SC);
          // B start address advances by NQ*16 bytes per subspace: +NQ in the
          // descriptor's (address >> 4) field
          const uint64_t bd = bdesc0 + (uint64_t)(c * KC * NQ);
          if (elect_one()) {
            if (!(a.exp & 8)) {
            mma_ts(d, ta, bd, idesc, c > 0 ? 1u : 0u);
#pragma unroll
            for (int m = 1; m < KC / 2; ++m)
              if (npair > m) mma_ts(d, ta + 8 * m, bd + (uint64_t)(2 * m * NQ), idesc, 1u);
            }
            mma_commit(&aempty[slot]);
          }
          __syncwarp();
          if (++slot == a.slots) {
            slot = 0;
            ++round;
          }
        }
        if (elect_one()) mma_commit(&dfull[buf]);
        __syncwarp();
      }
    }
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
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
    printf("TCPROF cta=%d warp=%d total=%lld wait0=%lld wait1=%lld items=%lld\n", (int)blockIdx.x, warp,
           clock64() - tstart, tw0, tw1, (long long)(it1 - it0));
#endif
  __syncthreads();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// pair-major packed codes (dense.py:156-170) -> [ceil(K/8)][n] u32, nibble s
// of word (c, p) = code of subspace 8c+s of point p (zero past K)
__global__ void k_to_hcodes(const uint8_t* __restrict__ packed, int64_t n, int npairs,
                            uint32_t* __restrict__ h) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (p >= n) return;
  uint32_t w = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int pair = 4 * c + t;
    if (pair < npairs) w |= (uint32_t)packed[(int64_t)pair * n + p] << (8 * t);
  }
  h[(int64_t)c * n + p] = w;
}

int pick_nq(int Kp, int64_t nq) {
  const int64_t by_smem = (int64_t)(kSmemBudget - 1024) / ((int64_t)Kp * 16);
  int64_t v = std::min<int64_t>(kMaxNQ, by_smem) / 32 * 32;
  const int64_t need = ceil_div(nq, 32) * 32;  // small batches: no idle columns
  if (need < v) v = need;
  return (int)std::max<int64_t>(v, 0);
}

}  // namespace

bool lut16_tc_supported(const DeviceIndex& ix) {
  return ix.hcodes != nullptr && ix.K > 0 && ix.K <= 257 && pick_nq(ix.Kp, 1LL << 40) >= 32;
}

int64_t lut16_tc_ld(int64_t n) { return ((n + kPM - 1) / kPM) * kPM; }

int64_t lut16_tc_group(const DeviceIndex& ix) { return pick_nq(ix.Kp, 1LL << 40); }


void launch_to_hcodes(const uint8_t* packed, int64_t n, int K, uint32_t* h, cudaStream_t st) {
  if (n <= 0 || K <= 0) return;
  const int nkc = (K + kKC - 1) / kKC;
  dim3 grid((unsigned)ceil_div(n, 256), (unsigned)nkc);
  k_to_hcodes<<<grid, 256, 0, st>>>(packed, n, (K + 1) / 2, h);
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
  int64_t ngroups, nblocks, items_per_cta, grid, nseg;
};

TcLayout tc_layout(const DeviceIndex& ix, int64_t nq, int64_t n) {
  TcLayout L;
  L.NQ = pick_nq(ix.Kp, nq);
  L.ngroups = ceil_div(nq, L.NQ);
  L.nblocks = ceil_div(n, kPM);
  // one CTA per SM (it owns all of TMEM), equal contiguous shares of the
  // (group, block) items
  const int64_t items = L.ngroups * L.nblocks;
  const int64_t ctas = std::min<int64_t>(kNumSMs, items);
  L.items_per_cta = ceil_div(items, ctas);
  L.grid = ceil_div(items, L.items_per_cta);
  // CTAs covering one group: its items span at most this many CTA ranges
  L.nseg = std::min<int64_t>(L.grid, ceil_div(L.nblocks, L.items_per_cta) + 1);
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
  const int KCsel = kc_env == 8 ? 8 : (nw > 8 && nw <= 16) ? 16 : 8;  // wide slots for K<=128
  a.slots = std::min(slot_cap, (kTmemCols - 2 * NQ) / (4 * KCsel));
  a.hcodes = ix.hcodes;
  a.luts = luts;
  a.tot = tot;
  a.ld = ld;
  a.stride = ix.n;
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
  const size_t smem =
      (size_t)a.Kp * NQ * 16 + kStageBytes + (2 * a.slots + 4) * sizeof(uint64_t) + 16;
  void (*kern)(TcArgs, const CUtensorMap);
  if (filter)
    kern = nw <= 8 ? k_lut16_tc<8, true, 8>
           : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, true, 16> : k_lut16_tc<16, true, 8>)
                      : k_lut16_tc<33, true, 8>;
  else
    kern = nw <= 8 ? k_lut16_tc<8, false, 8>
           : nw <= 16 ? (KCsel == 16 ? k_lut16_tc<16, false, 16> : k_lut16_tc<16, false, 8>)
                      : k_lut16_tc<33, false, 8>;
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
  kern<<<(unsigned)grid, kThreadsTc, smem, st>>>(a, tmap);
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
  *frac = std::min(1.0, (double)L.items_per_cta / (double)L.nblocks);
}

int launch_lut16_filter(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                        const uint32_t* tlim, uint2* list, uint32_t* cnt, int64_t cap,
                        cudaStream_t st) {
  HS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * nq * tc_layout(ix, nq, ix.n).nseg, st));
  return launch_tc(ix, luts, nq, -1, nullptr, 0, tlim, list, cnt, cap, st);
}

}  // namespace hs
