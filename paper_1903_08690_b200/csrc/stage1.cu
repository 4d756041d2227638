// stage1.cu — fused stage 1: posting-list stream (K3) + LUT16 scan (K2) +
// per-tile exact top-k (K4), for a chunk of queries.
//
// Replaces _stage1_scores (reference pipeline.py:192-203) and the first
// select_topk (pipeline.py:250-252):
//   sparse_scan   sparse.py:268-284  acc[ids] += f64(q_j) * f64(w), dims ascending
//   lut16_scan    dense.py:297-317   total = sum_k table[k][code_k] (integer, never wraps)
//   dense score   dense.py:317, pipeline.py:213   (bias_total + scale*total) + offset
//   stage-1 score pipeline.py:202   acc + dense
//
// Grid: (queries, tiles) — the query index varies fastest so the CTAs that
// are resident together stream the same tile of codes and share it in L2.
// A CTA walks its tile of layout slots in chunks of kChunk points:
//   1. dense: codes are stored "vertically" (re-tiled at upload): one u32 per
//      (subspace, 8 points), nibble j = code of point j.  A thread owns 16
//      points; per subspace it loads one uint2 and looks the 16 codes up in
//      the 16-byte u8 table held in 4 registers with PRMT (the GPU analogue
//      of the paper's in-register PSHUFB LUT16): two PRMTs
//      select among entries 0-7 / 8-15 and a third builds the byte mask from
//      the nibbles' bit 3.  Sums accumulate as 2 x u16 lanes per register
//      (K*255 < 2^16 for K <= 257; wider K is flushed every 256 subspaces).
//   2. sparse: every query dim keeps a cursor into its ascending posting list
//      and the id it points at (`dnext`) in shared memory, so a chunk only
//      touches the dims whose next posting falls inside it.  The active dims
//      are compacted in ascending order and their slices added dim by dim
//      into an f64 accumulator in shared memory (ascending dim order per
//      point, starting from +0.0 => bit-exact with the reference).
//   3. score = acc + ((bias_total + scale*total) + offset), unfused f64.
//   4. offer to a shared-memory candidate buffer guarded by the running k-th
//      best (score desc, original id asc); overflow => bitonic compaction.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;
constexpr int kPPT = 16;                   // points per thread per chunk
constexpr int kChunk = kThreads * kPPT;    // 4096 points
constexpr int kOfferPer = 4;                       // offers per thread per insertion round
constexpr int kOfferRound = kThreads * kOfferPer;  // worst-case offers per insertion round
#ifndef MINB0
#define MINB0 4
#endif
#ifndef KB0
#define KB0 3
#endif
constexpr int kSmallPostings = 512;        // below this a chunk's postings skip the barriers
constexpr int kRingBytes = 24 * 1024;  // posting ring (bulk-copy staging), default size
constexpr int kPieceMax = 1024;        // postings per staged piece
constexpr int kPieceBars = 32;         // mbarrier pairs = pieces in flight
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;  // empty bucket entry (after k_bucket_aggregate)

struct Stage1Args {
  int64_t n;
  int64_t tile_pts;
  int mode;
  int k, cap;
  int64_t out_per_tile;
  int ntiles;
  // sparse
  const uint2* post;
  const int64_t* qptr;
  const uint32_t* lbeg;
  const uint32_t* lend;
  const double* qv;
  const int32_t* lidx;
  // dense
  int has_dense;
  int K, Kp;
  const uint32_t* vcodes;  // [chunk][K][kChunk/8] u32, nibble j = point 8*word + j of the chunk
  const uint8_t* luts;
  const double* bias_total;
  const double* scale;
  const double* offset;
  // selection / output
  const uint32_t* order;
  Cand* out;
  double* dump;
  uint32_t* dump_tot;  // DUMP: integer totals (optional)
  int raw_dense;       // DUMP: bias_total + scale*total only (lut16_scan semantics)
  int max_qnnz;
  // bucketed postings (SparseBuckets); bmode == nullptr => stream every query
  const int* bmode;
  const uint32_t* boff;
  const uint32_t* bslots;
  const double* bvals;
  int64_t capq;
  int nchunks_g;
  // skip tables (long lists)
  const int32_t* skip_row;
  const uint32_t* skip;
  int nchunks_all;
  // precomputed LUT16 totals (tensor-core pass), [q][tot_ld] u16; null => PRMT scan
  const uint16_t* tot16;
  int64_t tot_ld;
  int exp_flags;       // dev experiments (HSB200_EXP): 1 no dense, 2 no sparse, 4 no offers
  const int* qmask;    // only queries with qmask[q] != 0 run (null: all)
  uint32_t ring_bytes; // WS: posting ring size (multiple of 16, >= 2 pieces)
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
// 1-D bulk copy global -> shared (TMA), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t lower_bound_ids(const uint2* __restrict__ post, uint32_t lo,
                                                    uint32_t hi, uint32_t key) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(&post[mid].x) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// number of ids < key starting at cur, given post[cur].x < key (galloping)
__device__ __forceinline__ uint32_t count_below_known(const uint2* __restrict__ post, uint32_t cur,
                                                      uint32_t end, uint32_t key) {
  uint32_t prev = cur, step = 1;
  while (prev + step < end && __ldg(&post[prev + step].x) < key) {
    prev += step;
    step <<= 1;
  }
  const uint32_t right = min(prev + step, end);
  return lower_bound_ids(post, prev + 1, right, key) - cur;
}

// Chunk accumulator layout: point 16*t + j of the chunk lives at
// j*256 + (t ^ j).  The owner threads' reads (fixed j, consecutive t) and the
// posting stream's writes (consecutive points) both spread over all banks.
static_assert(kChunk == kThreads * kPPT, "chunk = threads x points per thread");
__device__ __forceinline__ int acc_ix(uint32_t local) {
  const uint32_t j = local & (kPPT - 1), t = local / kPPT;
  return (int)(j * kThreads + (t ^ j));
}
// accumulator index of a chunk-local slot (DM == 0: plain, see pt_local)
template <int DM>
__device__ __forceinline__ int aix(uint32_t local) {
  return DM == 0 ? (int)local : acc_ix(local);
}
// owner thread of a chunk-local slot
template <int DM>
__device__ __forceinline__ uint32_t owner_of(uint32_t local) {
  return DM == 0 ? (local & (kThreads - 1)) : (local / kPPT);
}

struct Smem {
  Cand* buf;
  Cand* th;
  double* acc;
  uint4* lut;
  double* dqv;
  uint32_t* dcur;
  uint32_t* dend;
  uint32_t* dnext;
  uint32_t* alist;  // active dims of the chunk (ascending)
  uint32_t* abase;  // their slice start
  uint32_t* acnt;   // their slice length
  int32_t* dskip;   // skip-table row of the dim's list, -1 if short
  uint32_t* dbeg;   // list begin (absolute posting index)
  // warp-specialised posting stream (WS kernels)
  unsigned char* ring;  // posting ring, kRingBytes
  uint64_t* full;       // [kPieceBars] piece landed (bulk-copy transaction count)
  uint64_t* empty;      // [kPieceBars] piece consumed (one arrival per consumer warp)
  uint4* pdsc;          // [kPieceBars] piece: ring offset, ga, g0, ge
  uint64_t* pend;       // [kPieceBars] ring end (producer's byte counter) of the piece
  int* pdim;            // [kPieceBars] query dim of the piece, -1 = end of chunk
  double* scratch;      // 2 dummy accumulators
  uint32_t* bslot;  // staged bucket entries (chunk-local slot)
  double* bval;     // staged bucket entries (product)
  int* ctl;         // [0]=cnt [2]=have_th [4..12]=warp sums [16..23]=chunk posting counts
};


// Consumer-side block barrier: the whole CTA, or in warp-specialised kernels
// the kThreads consumer threads only (named barrier 1; the producer warp runs
// its own loop).
template <bool WS>
__device__ __forceinline__ void csync() {
  if constexpr (WS) {
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  } else {
    __syncthreads();
  }
}
template <bool WS>
__device__ __forceinline__ bool csync_or(bool pred) {
  if constexpr (WS) {
    int r;
    asm volatile(
        "{\n\t.reg .pred a, b;\n\tsetp.ne.s32 a, %1, 0;\n\t"
        "bar.red.or.pred b, 1, %2, a;\n\tselp.s32 %0, 1, 0, b;\n\t}"
        : "=r"(r)
        : "r"((int)pred), "n"(kThreads)
        : "memory");
    return r != 0;
  } else {
    return __syncthreads_or(pred) != 0;
  }
}

// Keep the best k of buf[0..cnt) by (score desc, original id asc) and set the
// running threshold to the k-th best.  Radix select over the score key (8-bit
// digits, early exit when a whole bin is taken) then, for exact score ties at
// the boundary, over the id; in-place order-preserving compaction.  O(cnt)
// per digit — replaces a bitonic sort of the whole buffer.  The 256-bin
// histogram lives in the bucket staging area (idle during the offer phase); the
// chunk accumulator must survive, the offer loop re-reads it for scores.
static_assert(sizeof(double) * kThreads >= 256 * sizeof(unsigned), "histogram fits the staging area");

// Smallest u16 LUT total whose dense-only score (bias_total + scale*t) + offset
// reaches the threshold score (65536: none).  The f64 ops are monotone in t
// (scale >= 0), so a point with no sparse part and total < tlim cannot pass.
__device__ int dense_tlim(double ths, double btot, double scl, double off) {
  int lo = 0, hi = 65536;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const double v = __dadd_rn(__dadd_rn(btot, __dmul_rn(scl, (double)mid)), off);
    if (v >= ths) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Offers are appended with the tie id unset (the original-id lookup is a
// dependent global load that would stall the whole block at the offer
// barrier); compaction resolves them in one parallel pass first.
constexpr uint32_t kTieUnset = 0xFFFFFFFFu;

template <bool WS>
__device__ void compact(Smem& s, int k, bool dense, double btot, double scl, double off,
                        const uint32_t* __restrict__ order) {
  const int cnt = s.ctl[0];
  csync<WS>();  // every thread has read ctl[0]
  for (int i = threadIdx.x; i < cnt; i += kThreads)
    if (s.buf[i].tie == kTieUnset) s.buf[i].tie = __ldg(order + s.buf[i].slot);
  csync<WS>();
  if (cnt <= k) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned* hist = reinterpret_cast<unsigned*>(s.bval);
  unsigned long long prefix = 0, pmask = 0;
  int need = k;
  bool whole_bin = false;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    csync<WS>();
    for (int i = tid; i < cnt; i += kThreads) {
      const unsigned long long key = score_key(s.buf[i].s);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
    }
    csync<WS>();
    if (warp == 0) find_bin(hist, need, true, s.ctl + 12);
    csync<WS>();
    const int b = s.ctl[12];
    need = s.ctl[13];
    prefix |= (unsigned long long)b << shift;
    pmask |= 0xFFull << shift;
    whole_bin = s.ctl[14] == need;
    csync<WS>();
    if (whole_bin) break;
  }
  // boundary ties in score: the `need` smallest ids among key == prefix
  uint32_t tie_lim = 0xFFFFFFFFu;
  if (!whole_bin) {
    uint32_t tpre = 0, tmask = 0;
    int tneed = need;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
      csync<WS>();
      for (int i = tid; i < cnt; i += kThreads) {
        const Cand e = s.buf[i];
        if (score_key(e.s) == prefix && (e.tie & tmask) == tpre)
          atomicAdd(&hist[(e.tie >> shift) & 255], 1u);
      }
      csync<WS>();
      if (warp == 0) find_bin(hist, tneed, false, s.ctl + 12);
      csync<WS>();
      tpre |= (uint32_t)s.ctl[12] << shift;
      tmask |= 0xFFu << shift;
      tneed = s.ctl[13];
      csync<WS>();
    }
    tie_lim = tpre;
  }
  // in-place compaction (ranks never exceed indices) + worst kept entry
  Cand worst;
  worst.s = INFINITY;
  worst.tie = 0;
  worst.slot = 0;
  int kept = 0;
  for (int base = 0; base < cnt; base += kThreads) {
    const int i = base + tid;
    Cand e;
    bool keep = false;
    if (i < cnt) {
      e = s.buf[i];
      const unsigned long long key = score_key(e.s) & pmask;
      keep = key > prefix || (key == prefix && (whole_bin || e.tie <= tie_lim));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s.ctl[4 + warp] = __popc(bal);
    csync<WS>();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const int c = s.ctl[4 + w];
      before += (w < warp) ? c : 0;
      total += c;
    }
    if (keep) {
      s.buf[kept + before + __popc(bal & ((1u << lane) - 1u))] = e;
      if (better(worst, e)) worst = e;
    }
    kept += total;
    csync<WS>();
  }
  // block min of the kept entries -> threshold
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand o_;
    o_.s = __shfl_xor_sync(0xffffffffu, worst.s, o);
    o_.tie = __shfl_xor_sync(0xffffffffu, worst.tie, o);
    o_.slot = 0;
    if (better(worst, o_)) worst = o_;
  }
  Cand* wbuf = reinterpret_cast<Cand*>(s.bval);  // histogram no longer needed
  if (lane == 0) wbuf[warp] = worst;
  csync<WS>();
  if (tid == 0) {
    Cand w = wbuf[0];
    for (int i = 1; i < kThreads / 32; ++i)
      if (better(w, wbuf[i])) w = wbuf[i];
    *s.th = w;
    s.ctl[0] = kept;
    s.ctl[2] = 1;
    s.ctl[3] = dense ? dense_tlim(w.s, btot, scl, off) : 0;
  }
  csync<WS>();
}

template <bool WS>
__device__ __forceinline__ int block_sum(int v, int* scratch) {
  // scratch: >= kThreads/32 ints; returns the block total to every thread
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) scratch[w] = v;
  csync<WS>();
  int t = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) t += scratch[i];
  csync<WS>();
  return t;
}

// two subspaces' lookups for the same 16 points, widened to u16 lanes and
// added with one IADD3 per lane pair (byte sums of two entries fit in 16 bits)
__device__ __forceinline__ void accum32(uint32_t* acc2, const uint32_t* r, const uint32_t* t) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc2[2 * i] += (r[i] & 0x00FF00FFu) + (t[i] & 0x00FF00FFu);
    acc2[2 * i + 1] += prmt(r[i], 0u, 0x4341u) + prmt(t[i], 0u, 0x4341u);  // bytes 1,3
  }
}

// Producer warp of the warp-specialised stage 1: walks the tile's chunks,
// finds each chunk's active query dims (ascending; skip tables for long lists,
// galloping cursors for short ones — lane per dim), cuts their slices into
// pieces of <= kPieceMax postings widened to 16-byte pairs from the even index
// at or below the slice start, and bulk-copies the pieces (TMA, mbarrier
// transaction counts) into the ring as far ahead as the kPieceBars slots and
// kRingBytes allow.  An end-of-chunk marker (no data) closes every chunk.
// Lane 0 issues; head/tail are ring byte counters (a piece never wraps).
__device__ __noinline__ void produce_postings(Smem& s, const Stage1Args& a, int nd, int64_t tile_lo,
                                              int64_t tile_hi, int lane) {
  const uint32_t kRing = a.ring_bytes;
  uint32_t issued = 0, released = 0;
  uint64_t head = 0, tail = 0;
  auto release = [&]() {
    const int rs = (int)(released % kPieceBars);
    mbar_wait(&s.empty[rs], (released / kPieceBars) & 1u);
    tail = s.pend[rs];
    ++released;
  };
  for (int64_t cb = tile_lo; cb < tile_hi; cb += kChunk) {
    const int64_t ce = min(tile_hi, cb + (int64_t)kChunk);
    int nact = 0;
    for (int base = 0; base < nd; base += 32) {
      const int d = base + lane;
      int32_t row = -1;
      uint32_t sk0 = 0, sk1 = 0;
      if (d < nd) {
        row = s.dskip[d];
        if (row >= 0) {
          const uint32_t* r = a.skip + (int64_t)row * (a.nchunks_all + 1) + cb / kChunk;
          sk0 = __ldg(r);
          sk1 = __ldg(r + 1);
        }
      }
      const bool f = d < nd && (row >= 0 ? sk1 > sk0 : s.dnext[d] < (uint32_t)ce) &&
                     !(a.exp_flags & 2);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) {
        const int slot = nact + __popc(bal & ((1u << lane) - 1u));
        s.alist[slot] = d;
        if (row >= 0) {
          s.abase[slot] = s.dbeg[d] + sk0;
          s.acnt[slot] = sk1 - sk0;
        } else {
          const uint32_t cur = s.dcur[d], end = s.dend[d];
          HS_DCHECK(cur < end && s.dnext[d] >= (uint32_t)cb);
          const uint32_t cnt = count_below_known(a.post, cur, end, (uint32_t)ce);
          const uint32_t nc = cur + cnt;
          s.abase[slot] = cur;
          s.acnt[slot] = cnt;
          s.dcur[d] = nc;
          s.dnext[d] = nc < end ? __ldg(&a.post[nc].x) : 0xFFFFFFFFu;
        }
      }
      nact += __popc(bal);
    }
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < nact; ++i) {
        const int d = (int)s.alist[i];
        uint32_t g = s.abase[i];
        const uint32_t end = g + s.acnt[i];
        while (g < end) {
          const uint32_t ge = min(end, g + (uint32_t)kPieceMax), ga = g & ~1u;
          const uint32_t bytes = ((ge - ga + 1) >> 1) * 16u;
          while (issued - released >= (uint32_t)kPieceBars) release();
          uint32_t phys, pad;
          for (;;) {
            if (released == issued) head = tail = 0;  // ring empty: restart at 0
            phys = (uint32_t)(head % kRing);
            pad = phys + bytes > kRing ? kRing - phys : 0u;
            if (head + pad + bytes - tail <= (uint64_t)kRing) break;
            release();
          }
          head += pad;
          if (pad) phys = 0;
          const int slot = (int)(issued % kPieceBars);
          s.pdsc[slot] = make_uint4(phys, ga, g, ge);
          s.pdim[slot] = d;
          s.pend[slot] = head + bytes;
          head += bytes;
          mbar_arrive_tx(&s.full[slot], bytes);
          bulk_g2s(s.ring + phys, a.post + ga, bytes, &s.full[slot]);
          ++issued;
          g = ge;
        }
      }
      while (issued - released >= (uint32_t)kPieceBars) release();
      const int slot = (int)(issued % kPieceBars);
      s.pdim[slot] = -1;
      s.pend[slot] = head;
      mbar_arrive(&s.full[slot]);
      ++issued;
    }
    __syncwarp();
  }
}

// DM: dense mode (0 none, 1 PRMT LUT16 scan, 2 precomputed u16 totals);
// SP: the query batch has postings to stream (else the sparse phase is elided);
// WS: warp-specialised posting stream (a 9th, producer warp; see produce_postings).
template <int DM, bool SP, bool WS>
__global__ void __launch_bounds__(WS ? kThreads + 32 : kThreads, DM == 0 ? MINB0 : 3) k_stage1(Stage1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t q = blockIdx.x;
  const int tile = blockIdx.y;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (a.qmask && a.qmask[q] == 0) return;

  // ---- carve shared memory ----
  Smem s;
  unsigned char* p = smem_raw;
  s.buf = reinterpret_cast<Cand*>(p);
  p += sizeof(Cand) * (size_t)a.cap;
  s.th = reinterpret_cast<Cand*>(p);
  p += sizeof(Cand);
  s.acc = reinterpret_cast<double*>(p);
  p += sizeof(double) * kChunk;
  s.lut = reinterpret_cast<uint4*>(p);
  p += 16 * (size_t)a.Kp;
  s.dqv = reinterpret_cast<double*>(p);
  p += sizeof(double) * a.max_qnnz;
  s.dcur = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.dend = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.dnext = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.alist = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.abase = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.acnt = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  s.dskip = reinterpret_cast<int32_t*>(p);
  p += sizeof(int32_t) * a.max_qnnz;
  s.dbeg = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * a.max_qnnz;
  if (WS) {
    p = smem_raw + ((p - smem_raw + 15) & ~(ptrdiff_t)15);
    s.ring = p;
    p += a.ring_bytes;
    s.pdsc = reinterpret_cast<uint4*>(p);
    p += sizeof(uint4) * kPieceBars;
    s.full = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * kPieceBars;
    s.empty = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * kPieceBars;
    s.pend = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * kPieceBars;
    s.scratch = reinterpret_cast<double*>(p);
    p += sizeof(double) * 2;
    s.pdim = reinterpret_cast<int*>(p);
    p += sizeof(int) * kPieceBars;
  }
  p = smem_raw + ((p - smem_raw + 7) & ~(ptrdiff_t)7);
  s.bval = reinterpret_cast<double*>(p);
  p += sizeof(double) * kThreads;
  s.bslot = reinterpret_cast<uint32_t*>(p);
  p += sizeof(uint32_t) * kThreads;
  s.ctl = reinterpret_cast<int*>(p);

  const int64_t tile_lo = (int64_t)tile * a.tile_pts;
  const int64_t tile_hi = min(a.n, tile_lo + a.tile_pts);

  // ---- per-query setup ----
  const int64_t qb = a.qptr[q], qe = a.qptr[q + 1];
  const bool bucketed = SP && a.bmode != nullptr && a.bmode[q] == 1;
  const int nd = (SP && !bucketed) ? (int)(qe - qb) : 0;  // bucketed queries skip the cursors
  const bool stream = WS && nd > 0;  // the producer warp stages this query's postings
  HS_DCHECK(nd >= 0 && nd <= a.max_qnnz);
  const uint32_t* qboff = bucketed ? a.boff + q * (int64_t)(a.nchunks_g + 1) : nullptr;
  const uint32_t* qslots = bucketed ? a.bslots + q * a.capq : nullptr;
  const double* qvals = bucketed ? a.bvals + q * a.capq : nullptr;
  for (int d = tid; d < nd; d += blockDim.x) {
    const uint32_t b = a.lbeg[qb + d], e = a.lend[qb + d];
    HS_DCHECK(b <= e);
    const int32_t li = a.lidx ? a.lidx[qb + d] : -1;
    const int32_t row = (li >= 0 && a.skip_row) ? a.skip_row[li] : -1;
    s.dqv[d] = a.qv[qb + d];
    s.dskip[d] = row;
    s.dbeg[d] = b;
    s.dend[d] = e;
    if (row < 0) {  // short list: cursor + next id
      const uint32_t c = lower_bound_ids(a.post, b, e, (uint32_t)tile_lo);
      s.dcur[d] = c;
      s.dnext[d] = c < e ? __ldg(&a.post[c].x) : 0xFFFFFFFFu;
    } else {
      s.dcur[d] = b;
      s.dnext[d] = 0xFFFFFFFFu;
    }
  }
  if (DM == 1) {
    const uint4* src = reinterpret_cast<const uint4*>(a.luts + q * (int64_t)a.Kp * 16);
    for (int i = tid; i < a.Kp; i += blockDim.x) s.lut[i] = src[i];
  }
  if (tid < 16) s.ctl[tid] = 0;
  if (WS && tid == 0) {
    for (int i = 0; i < kPieceBars; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], kThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  double btot = 0.0, scl = 0.0, off = 0.0;
  if (DM != 0) {
    btot = a.bias_total[q];
    scl = a.scale[q];
    off = a.offset ? a.offset[q] : 0.0;
  }
  const uint2* vc = reinterpret_cast<const uint2*>(a.vcodes);
  constexpr int64_t vrow = kChunk / 16;  // uint2 per subspace row of a chunk's code block
  // u16 totals are prefetched two chunks ahead (tnext: next chunk, tnext2:
  // the one after)
  uint4 tnext0 = make_uint4(0u, 0u, 0u, 0u), tnext1 = tnext0, tnext20 = tnext0, tnext21 = tnext0;
  if (DM == 2) {
    const int64_t pa = tile_lo + (int64_t)tid * kPPT;
    if (pa < tile_hi) {
      const uint4* src = reinterpret_cast<const uint4*>(a.tot16 + q * a.tot_ld + pa);
      tnext0 = __ldg(src);
      tnext1 = __ldg(src + 1);
    }
    if (pa + kChunk < tile_hi) {
      const uint4* src = reinterpret_cast<const uint4*>(a.tot16 + q * a.tot_ld + pa + kChunk);
      tnext20 = __ldg(src);
      tnext21 = __ldg(src + 1);
    }
  }
  __syncthreads();  // whole CTA (producer warp included)
  if constexpr (WS) {
    if (warp == kThreads / 32) {
      if (stream) produce_postings(s, a, nd, tile_lo, tile_hi, lane);
      return;
    }
  }
  uint32_t consumed = 0;  // pieces consumed (mbarrier slot and phase), uniform
  // skip-table entries of the next chunk (long lists, nd <= kThreads)
  uint32_t sk_lo = 0, sk_hi = 0;
  int64_t skc = -1;
  for (int64_t cb = tile_lo; cb < tile_hi; cb += kChunk) {
    const int64_t ce = min(tile_hi, cb + (int64_t)kChunk);
    const int64_t p0 = cb + (int64_t)tid * kPPT;
    // points of this thread: 16 consecutive (dense variants: the LUT16 scan's
    // layout) or, sparse-only, strided by the block (then the accumulator
    // is indexed by the plain chunk-local slot: conflict-free both for the
    // posting stream's consecutive slots and for the owners' reads)
    auto pt_local = [&](int j) -> uint32_t {
      return DM == 0 ? (uint32_t)(j * kThreads + tid) : (uint32_t)(tid * kPPT + j);
    };
    HS_DCHECK(cb >= tile_lo && ce <= a.n);
    // zero this thread's own accumulator entries (only owners read them, in
    // the previous chunk's offer phase); the streamed path's adds start after
    // the active-dim barrier below, so it needs no zeroing pass of its own
    if (SP && !WS && !bucketed) {
#pragma unroll
      for (int j = 0; j < kPPT; ++j) s.acc[aix<DM>(pt_local(j))] = 0.0;
    }

    // ---- dense: LUT16 scan of this thread's 16 points ----
    uint32_t tot[kPPT];
#pragma unroll
    for (int j = 0; j < kPPT; ++j) tot[j] = 0;
    if (DM == 2 && p0 < ce) {
      // totals of this chunk were prefetched two chunks ago
      const uint4 t0 = tnext0, t1 = tnext1;
      tnext0 = tnext20;
      tnext1 = tnext21;
      if (p0 + 2 * kChunk < tile_hi) {
        const uint4* nsrc = reinterpret_cast<const uint4*>(a.tot16 + q * a.tot_ld + p0 + 2 * kChunk);
        tnext20 = __ldg(nsrc);
        tnext21 = __ldg(nsrc + 1);
      }
      const uint32_t w8[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        tot[2 * j] = w8[j] & 0xFFFFu;
        tot[2 * j + 1] = w8[j] >> 16;
      }
    } else if (DM == 1 && p0 < ce && !(a.exp_flags & 1)) {
      // blocked vertical planes (lut16_stream.cu): chunk cb/kChunk, row k, word pair tid
      const uint2* col = vc + (cb / kChunk) * (int64_t)a.K * vrow + tid;
      uint32_t acc2[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc2[j] = 0;
      int k = 0;
      for (int kb = 0; kb < a.K; kb += 256) {
        const int kend = min(a.K, kb + 256);
        uint2 wn[8];
        if (k + 8 <= kend) {
#pragma unroll
          for (int u = 0; u < 8; ++u) wn[u] = __ldg(col + (int64_t)(k + u) * vrow);
        }
        for (; k + 8 <= kend; k += 8) {
          uint2 w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) w[u] = wn[u];
          if (k + 16 <= kend) {  // prefetch the next group while this one computes
#pragma unroll
            for (int u = 0; u < 8; ++u) wn[u] = __ldg(col + (int64_t)(k + 8 + u) * vrow);
          }
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            const uint4 T0 = s.lut[k + u], T1 = s.lut[k + u + 1];
            uint32_t r[4], t[4];
            lut8(T0, w[u].x, r[0], r[1]);
            lut8(T0, w[u].y, r[2], r[3]);
            lut8(T1, w[u + 1].x, t[0], t[1]);
            lut8(T1, w[u + 1].y, t[2], t[3]);
            accum32(acc2, r, t);
          }
        }
        for (; k < kend; ++k) {
          const uint2 w = __ldg(col + (int64_t)k * vrow);
          const uint4 T = s.lut[k];
          uint32_t r[4], t[4] = {0u, 0u, 0u, 0u};
          lut8(T, w.x, r[0], r[1]);
          lut8(T, w.y, r[2], r[3]);
          accum32(acc2, r, t);
        }
        // widen: acc2[2g] holds points (4g, 4g+2), acc2[2g+1] holds (4g+1, 4g+3)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          tot[4 * g + 0] += acc2[2 * g] & 0xFFFFu;
          tot[4 * g + 2] += acc2[2 * g] >> 16;
          tot[4 * g + 1] += acc2[2 * g + 1] & 0xFFFFu;
          tot[4 * g + 3] += acc2[2 * g + 1] >> 16;
          acc2[2 * g] = 0;
          acc2[2 * g + 1] = 0;
        }
      }
    }

    // ---- sparse: bucketed postings of this chunk (pre-pass) ----
    int nact = 0, npost = 0;
    if (SP && bucketed) {
      const int64_t cg = cb / kChunk;
      const uint32_t e0 = __ldg(qboff + cg), e1 = __ldg(qboff + cg + 1);
      if (e1 > e0) {
        // Entries are aggregated per point (k_bucket_aggregate: one sum per
        // touched point, in the reference's per-point order), then kNoSlot
        // (only in buckets that had repeated points).
        const uint32_t L = e1 - e0;
        for (int i = tid; i < kChunk; i += kThreads) s.acc[i] = 0.0;
        csync<WS>();
        for (uint32_t i = tid; i < L; i += kThreads) {
          const uint32_t sl = __ldg(qslots + e0 + i);
          if (sl == kNoSlot) break;  // the sums come first, then only kNoSlot
          HS_DCHECK(sl - (uint32_t)cb < (uint32_t)kChunk);
          s.acc[aix<DM>(sl - (uint32_t)cb)] = __ldg(qvals + e0 + i);
        }
        csync<WS>();
        nact = 1;
        npost = 0;
      }
    }
    if (stream) {
      // ---- sparse (warp-specialised): consume the producer's pieces ----
      // Pieces arrive in ascending dim order; a barrier separates dims (each
      // point's additions stay in ascending dim order), thread t adds posting
      // pairs t, t+256, ... of a piece, and every warp releases the piece's
      // ring space with one arrival on its empty barrier.
      for (int i = tid; i < kChunk; i += kThreads) s.acc[i] = 0.0;
      csync<WS>();
      int cur = -1;
      const uint32_t ring = smem_addr(s.ring);
      for (;;) {
        const int slot = (int)(consumed % kPieceBars);
        mbar_wait(&s.full[slot], (consumed / kPieceBars) & 1u);
        ++consumed;
        const int d = s.pdim[slot];
        if (d < 0) {  // end of chunk
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.empty[slot]);
          break;
        }
        const uint4 pc = s.pdsc[slot];  // ring offset, ga, g0, ge
        if (d != cur) {
          if (cur >= 0) csync<WS>();
          cur = d;
        }
        const double qv = s.dqv[d];
        const uint32_t np = (pc.w - pc.y + 1) >> 1;
        for (uint32_t j = tid; j < np; j += kThreads) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"(ring + pc.x + 16 * j));
          const uint32_t g = pc.y + 2 * j;
          // halves outside [g0, ge) go to a scratch slot; f64(q)*f64(w) is
          // exact, so the fma rounds like the reference's separate add
          double* a0 = g >= pc.z ? &s.acc[aix<DM>(v.x - (uint32_t)cb)] : s.scratch;
          double* a1 = g + 1 < pc.w ? &s.acc[aix<DM>(v.z - (uint32_t)cb)] : s.scratch + 1;
          HS_DCHECK(g < pc.z || (v.x >= cb && v.x < ce));
          HS_DCHECK(g + 1 >= pc.w || (v.z >= cb && v.z < ce));
          *a0 = fma(qv, (double)__uint_as_float(v.y), *a0);
          *a1 = fma(qv, (double)__uint_as_float(v.w), *a1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.empty[slot]);
      }
      csync<WS>();
      nact = 1;
    } else if (SP && !bucketed) {
      // ---- sparse: active dims of this chunk, in ascending dim order ----
      for (int base = 0; base < nd; base += kThreads) {
        const int d = base + tid;
        int32_t row = -1;
        uint32_t sk0 = 0, sk1 = 0;
        if (d < nd) {
          row = s.dskip[d];
          if (row >= 0) {
            const uint32_t* r = a.skip + (int64_t)row * (a.nchunks_all + 1) + cb / kChunk;
            if (nd <= kThreads && skc == cb) {  // prefetched during the previous chunk
              sk0 = sk_lo;
              sk1 = sk_hi;
            } else {
              sk0 = __ldg(r);
              sk1 = __ldg(r + 1);
            }
            if (nd <= kThreads && cb + kChunk < tile_hi) {  // next chunk: row[c+1], row[c+2]
              sk_lo = sk1;
              sk_hi = __ldg(r + 2);
              skc = cb + kChunk;
            }
          }
        }
        const bool f = d < nd && (row >= 0 ? sk1 > sk0 : s.dnext[d] < (uint32_t)ce) &&
                       !(a.exp_flags & 2);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s.ctl[4 + warp] = __popc(bal);
        csync<WS>();
        int before = 0, total = 0;
  #pragma unroll
        for (int i = 0; i < kThreads / 32; ++i) {
          const int c = s.ctl[4 + i];
          before += (i < warp) ? c : 0;
          total += c;
        }
        uint32_t mycnt = 0;  // postings of this thread's active dim in the chunk
        if (f) {
          const int slot = nact + before + __popc(bal & ((1u << lane) - 1u));
          HS_DCHECK(slot < a.max_qnnz);
          s.alist[slot] = d;
          if (row >= 0) {
            s.abase[slot] = s.dbeg[d] + sk0;
            s.acnt[slot] = sk1 - sk0;
            mycnt = sk1 - sk0;
          } else {
            const uint32_t cur = s.dcur[d], end = s.dend[d];
            HS_DCHECK(cur < end);
            HS_DCHECK(__ldg(&a.post[cur].x) == s.dnext[d]);
            HS_DCHECK(s.dnext[d] >= (uint32_t)cb);
            const uint32_t cnt = count_below_known(a.post, cur, end, (uint32_t)ce);
            HS_DCHECK(cnt >= 1 && __ldg(&a.post[cur + cnt - 1].x) < (uint32_t)ce);
            const uint32_t nc = cur + cnt;
            s.abase[slot] = cur;
            s.acnt[slot] = cnt;
            mycnt = cnt;
            s.dcur[d] = nc;
            s.dnext[d] = nc < end ? __ldg(&a.post[nc].x) : 0xFFFFFFFFu;
          }
        }
        // chunk posting count: per-warp partial sums published before the
        // barrier that ends this pass (no separate block reduction)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mycnt += __shfl_xor_sync(0xffffffffu, mycnt, o);
        if (lane == 0) s.ctl[16 + warp] = (int)mycnt;
        nact += total;
        csync<WS>();
#pragma unroll
        for (int i = 0; i < kThreads / 32; ++i) npost += s.ctl[16 + i];
        if (base + kThreads < nd) csync<WS>();  // ctl[16..] is rewritten by the next pass
      }
  #ifdef HS_DEBUG
      for (int i = tid; i < nact; i += kThreads) {
        const uint32_t id0 = __ldg(&a.post[s.abase[i]].x);
        if (!(id0 >= (uint32_t)cb && id0 < (uint32_t)ce))
          printf("STALE q=%d i=%d nact=%d d=%u base=%u cnt=%u id0=%u cb=%lld ctlw=%d,%d,%d,%d,%d,%d,%d,%d\n",
                 (int)q, i, nact, s.alist[i], s.abase[i], s.acnt[i], id0, (long long)cb, s.ctl[4],
                 s.ctl[5], s.ctl[6], s.ctl[7], s.ctl[8], s.ctl[9], s.ctl[10], s.ctl[11]);
      }
      csync<WS>();
  #endif
      if (nact > 0 && npost <= kSmallPostings) {
        // few postings: every thread walks them all in dim order (broadcast
        // loads) and adds only those landing on its own 16 points — per-point
        // order stays ascending in dim with no block barriers (own entries
        // were zeroed at the top of the chunk)
        for (int i = 0; i < nact; ++i) {
          const uint32_t b = s.abase[i], c = s.acnt[i];
          const double qv = s.dqv[s.alist[i]];
          for (uint32_t j0 = 0; j0 < c; j0 += 8) {
            uint2 pw[8];
#pragma unroll
            for (int r = 0; r < 8; ++r)  // independent loads in flight
              pw[r] = j0 + r < c ? __ldg(&a.post[b + j0 + r]) : make_uint2(0xFFFFFFFFu, 0u);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const uint32_t local = pw[r].x - (uint32_t)cb;
              if (pw[r].x != 0xFFFFFFFFu && owner_of<DM>(local) == (uint32_t)tid)
                s.acc[aix<DM>(local)] += qv * (double)__uint_as_float(pw[r].y);
            }
          }
        }
      } else if (nact > 0) {
        // many postings: block-wide per dim, one barrier between dims; the
        // next dim's first kPre*256 postings are loaded while this dim adds
        constexpr int kPre = 4;
        uint2 nxt[kPre];
        {
          const uint32_t b = s.abase[0], c = s.acnt[0];
          const uint2* p0 = a.post + b + tid;
#pragma unroll
          for (int r = 0; r < kPre; ++r) {
            if (r > 0 && (uint32_t)(r * kThreads) >= c) break;  // block-uniform
            nxt[r] = (uint32_t)(tid + r * kThreads) < c ? __ldg(p0 + r * kThreads)
                                                         : make_uint2(0xFFFFFFFFu, 0u);
          }
        }
        for (int i = 0; i < nact; ++i) {
          const uint32_t b = s.abase[i], c = s.acnt[i];
          const double qv = s.dqv[s.alist[i]];
          uint2 cur[kPre];
#pragma unroll
          for (int r = 0; r < kPre; ++r) cur[r] = nxt[r];
          if (i + 1 < nact) {
            const uint32_t b2 = s.abase[i + 1], c2 = s.acnt[i + 1];
            const uint2* p2 = a.post + b2 + tid;
#pragma unroll
            for (int r = 0; r < kPre; ++r) {
              if (r > 0 && (uint32_t)(r * kThreads) >= c2) break;  // block-uniform
              nxt[r] = (uint32_t)(tid + r * kThreads) < c2 ? __ldg(p2 + r * kThreads)
                                                            : make_uint2(0xFFFFFFFFu, 0u);
            }
          }
#pragma unroll
          for (int r = 0; r < kPre; ++r) {
            if (r > 0 && (uint32_t)(r * kThreads) >= c) break;  // block-uniform
            if (cur[r].x == 0xFFFFFFFFu) continue;
            HS_DCHECK(cur[r].x >= cb && cur[r].x < ce);
            // f64(q) * f64(w) is exact, so contraction cannot change the sum
            s.acc[aix<DM>(cur[r].x - (uint32_t)cb)] += qv * (double)__uint_as_float(cur[r].y);
          }
          // long slices: whole batches of kB x kThreads postings with plain
          // (unpredicated, immediate-offset) loads, two register sets
          // alternating so the next batch is in flight while this one adds;
          // then one predicated batch for the remainder
          constexpr int kB = DM == 0 ? KB0 : 4;  // (register budget of the dense variants)
          constexpr uint32_t kBatch = kB * kThreads;
          if (c > (uint32_t)(kPre * kThreads)) {
            const uint32_t rest = c - kPre * kThreads;
            const uint32_t nfull = rest / kBatch;
            const uint2* ptr = a.post + b + kPre * kThreads + tid;
            auto load4 = [&](uint2* v, const uint2* p) {
#pragma unroll
              for (int r = 0; r < kB; ++r) v[r] = __ldg(p + r * kThreads);
            };
            auto add4 = [&](const uint2* v) {
#pragma unroll
              for (int r = 0; r < kB; ++r)
                s.acc[aix<DM>(v[r].x - (uint32_t)cb)] += qv * (double)__uint_as_float(v[r].y);
            };
            uint2 v0[kB], v1[kB];
            if (nfull > 0) load4(v0, ptr);
            for (uint32_t k = 0; k < nfull; k += 2) {
              if (k + 1 < nfull) load4(v1, ptr + kBatch);
              add4(v0);
              if (k + 2 < nfull) load4(v0, ptr + 2 * kBatch);
              if (k + 1 < nfull) add4(v1);
              ptr += 2 * kBatch;
            }
            const uint32_t done = kPre * kThreads + nfull * kBatch;
            if (done < c) {
              const uint2* tp = a.post + b + done + tid;
#pragma unroll
              for (int r = 0; r < kB; ++r)
                v0[r] = done + tid + r * kThreads < c ? __ldg(tp + r * kThreads)
                                                      : make_uint2(0xFFFFFFFFu, 0u);
#pragma unroll
              for (int r = 0; r < kB; ++r) {
                if (v0[r].x == 0xFFFFFFFFu) continue;
                HS_DCHECK(v0[r].x >= cb && v0[r].x < ce);
                s.acc[aix<DM>(v0[r].x - (uint32_t)cb)] += qv * (double)__uint_as_float(v0[r].y);
              }
            }
          }
          csync<WS>();
        }
      }
    }

    // ---- scores (recomputed where needed instead of held in 16 f64 registers) ----
    auto acc_of = [&](int j) -> double {
      return (SP && nact > 0) ? s.acc[aix<DM>(pt_local(j))] : 0.0;
    };
    auto score_with = [&](int j, double acc) -> double {
      if (a.raw_dense) return __dadd_rn(btot, __dmul_rn(scl, (double)tot[j]));
      if (DM != 0) {
        const double dn = __dadd_rn(__dadd_rn(btot, __dmul_rn(scl, (double)tot[j])), off);
        return __dadd_rn(acc, dn);
      }
      return acc;
    };
    auto score = [&](int j) -> double { return score_with(j, acc_of(j)); };

    if (a.mode == S1_DUMP) {
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        const int64_t pt = cb + pt_local(j);
        if (pt >= ce) continue;
        a.dump[q * a.n + pt] = score(j);
        if (a.dump_tot) a.dump_tot[q * a.n + pt] = tot[j];
      }
      csync<WS>();
      continue;
    }
    if (a.mode == S1_EMIT_ALL) {
      Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        const int64_t pt = cb + pt_local(j);
        if (pt < ce) {
          Cand c;
          c.s = score(j);
          c.slot = (uint32_t)pt;
          c.tie = a.order[pt];
          o[pt - tile_lo] = c;
        }
      }
      csync<WS>();
      continue;
    }

    // ---- offer to the candidate buffer ----
    if (a.exp_flags & 4) {
      double t = 0;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) t += score(j);
      if (t == 12345.678) s.ctl[15] = 1;  // keep the scores live
      csync<WS>();
      continue;
    }
    unsigned mask = 0;
    {
      const int have = s.ctl[2];
      const int tlim = s.ctl[3];
      const Cand th = *s.th;
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        const int64_t pt = cb + pt_local(j);
        if (pt >= ce) continue;
        const double aj = acc_of(j);
        // integer pre-filter: no sparse part and a LUT total below tlim
        if (DM != 0 && aj == 0.0 && (int)tot[j] < tlim) continue;
        const double sj = score_with(j, aj);
        bool pass = !have || sj > th.s;
        if (!pass && sj == th.s) pass = a.order[pt] < th.tie;
        if (pass) mask |= 1u << j;
      }
    }
    // nothing passes anywhere in the block (the steady state once the
    // threshold has settled): one barrier, no counting
    if (!csync_or<WS>(mask != 0u)) continue;
    // snapshot the count before block_sum's barriers: threads that pass the
    // room check start appending (atomicAdd on ctl[0]) right after it
    const int cnt0 = s.ctl[0];
    const int need = block_sum<WS>(__popc(mask), s.ctl + 4);
    if (cnt0 + need <= a.cap) {
      // common case: room for every offer
      if (mask) {
        int pos = atomicAdd(&s.ctl[0], __popc(mask));
        HS_DCHECK(pos + __popc(mask) <= a.cap);
#pragma unroll
        for (int j = 0; j < kPPT; ++j) {
          if (!(mask >> j & 1)) continue;
          Cand c;
          c.s = score(j);
          c.slot = (uint32_t)(cb + pt_local(j));
          c.tie = kTieUnset;
          s.buf[pos++] = c;
        }
      }
      csync<WS>();
    } else {
      // rounds of <= kOfferPer offers per thread, compacting whenever room runs out
#pragma unroll
      for (int r = 0; r < kPPT / kOfferPer; ++r) {
        unsigned m = (mask >> (kOfferPer * r)) & ((1u << kOfferPer) - 1u);
        const int cnt_r = s.ctl[0];  // read before the barriers, see above
        const int nr = block_sum<WS>(__popc(m), s.ctl + 4);
        if (nr == 0) continue;
        if (cnt_r + nr > a.cap) {
          compact<WS>(s, a.k, DM != 0, btot, scl, off, a.order);
          const Cand th = *s.th;
          unsigned m2 = 0;
#pragma unroll
          for (int j = 0; j < kOfferPer; ++j) {
            if (!(m >> j & 1)) continue;
            const int jj = kOfferPer * r + j;
            const double sj = score(jj);
            bool pass = sj > th.s;
            if (!pass && sj == th.s) pass = a.order[cb + pt_local(jj)] < th.tie;
            if (pass) m2 |= 1u << j;
          }
          m = m2;
        }
        if (m) {
          int pos = atomicAdd(&s.ctl[0], __popc(m));
          HS_DCHECK(pos + __popc(m) <= a.cap);
#pragma unroll
          for (int j = 0; j < kOfferPer; ++j) {
            if (!(m >> j & 1)) continue;
            const int jj = kOfferPer * r + j;
            Cand c;
            c.s = score(jj);
            c.slot = (uint32_t)(cb + pt_local(jj));
            c.tie = kTieUnset;
            s.buf[pos++] = c;
          }
        }
        csync<WS>();
      }
    }
  }

  if (a.mode == S1_EMIT_ALL) {
    Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
    for (int64_t i = (tile_hi - tile_lo) + tid; i < a.out_per_tile; i += kThreads)
      o[i] = worst_cand();
    return;
  }
  if (a.mode != S1_SELECT) return;
  compact<WS>(s, a.k, false, 0.0, 0.0, 0.0, a.order);  // best k of the tile, unordered (the merge sorts)
  Cand* o = a.out + (q * a.ntiles + tile) * a.out_per_tile;
  const int keep = s.ctl[0];
  for (int i = tid; i < a.out_per_tile; i += kThreads) o[i] = i < keep ? s.buf[i] : worst_cand();
}

// Map each query nonzero to its posting list [beg, end) (binary search over
// the sorted active dims) and its effective f64 value.  `weight` != 1 scales
// the f32 value in f32 first (pipeline.py:197-198, numpy weak-scalar rule).
__global__ void k_map_dims(const uint32_t* __restrict__ dims_q, const float* __restrict__ vals,
                           int64_t nnz, const uint32_t* __restrict__ post_dims, int64_t n_active,
                           const uint32_t* __restrict__ post_ptr, float weight, int use_weight,
                           uint32_t* lbeg, uint32_t* lend, double* qv, int32_t* lidx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint32_t dim = dims_q[i];
  int64_t lo = 0, hi = n_active;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (post_dims[mid] < dim) lo = mid + 1;
    else hi = mid;
  }
  if (lo < n_active && post_dims[lo] == dim) {
    lbeg[i] = post_ptr[lo];
    lend[i] = post_ptr[lo + 1];
    lidx[i] = (int32_t)lo;
  } else {
    lbeg[i] = 0;
    lend[i] = 0;
    lidx[i] = -1;
  }
  const float v = use_weight ? __fmul_rn(vals[i], weight) : vals[i];
  qv[i] = (double)v;
}

// sparse_scan into a caller-supplied accumulator (sparse.py:277-282): the k-th
// query dim of every query is one launch, so each point receives its
// products one dim after another in the query's ascending dim order, each
// `acc = acc + q_j * w` rounded like numpy's `acc.scores[ids] += qv * w`.
// Within one dim the posting ids are distinct, so the scatter is race free.
__global__ void k_scan_dim_into(const uint2* __restrict__ post, const int64_t* __restrict__ qptr,
                                const uint32_t* __restrict__ lbeg, const uint32_t* __restrict__ lend,
                                const double* __restrict__ qv, int k, int64_t n, double* acc) {
  const int64_t q = blockIdx.y;
  const int64_t i = qptr[q] + k;
  if (i >= qptr[q + 1]) return;
  const uint32_t b = lbeg[i], e = lend[i];
  const double v = qv[i];
  double* row = acc + q * n;
  for (uint32_t p = b + blockIdx.x * blockDim.x + threadIdx.x; p < e; p += gridDim.x * blockDim.x) {
    const uint2 pw = __ldg(post + p);
    row[pw.x] = __dadd_rn(row[pw.x], __dmul_rn(v, (double)__uint_as_float(pw.y)));
  }
}

// ---------------------------------------------------------------------------
// Sparse pre-pass: bucket one query's postings by 4096-slot chunk.
// Counting sort on the chunk id; dims are scattered one after another (in the
// query's ascending dim order) and, within a dim, runs of equal chunk keep
// their ascending slots, so every bucket lists each point's postings in
// ascending dim order — the reference's summation order (sparse.py:277-282).
// ---------------------------------------------------------------------------
constexpr int kBucketThreads = 256;

__device__ __forceinline__ int block_max_scan(int v, int* scratch) {
  // inclusive max-scan over the block in thread order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, u);
  }
  if (lane == 31) scratch[warp] = v;
  __syncthreads();
  int pre = -1;
  for (int w = 0; w < warp; ++w) pre = max(pre, scratch[w]);
  __syncthreads();
  return max(v, pre);
}

__global__ void __launch_bounds__(kBucketThreads) k_sparse_bucket(
    const int64_t* __restrict__ qptr, const uint32_t* __restrict__ lbeg,
    const uint32_t* __restrict__ lend, const double* __restrict__ qv,
    const uint2* __restrict__ post, int nchunks, int64_t capq, int* __restrict__ mode,
    uint32_t* __restrict__ boff, uint32_t* __restrict__ slots, double* __restrict__ vals) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw);  // [nchunks] hist -> cursor
  int* scr = reinterpret_cast<int*>(cnt + nchunks + 1);     // [32]
  const int64_t q = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t qb = qptr[q];
  const int nd = (int)(qptr[q + 1] - qb);
  int mine = 0;
  for (int d = tid; d < nd; d += blockDim.x) mine += (int)(lend[qb + d] - lbeg[qb + d]);
  // block sum
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((tid & 31) == 0) scr[tid >> 5] = mine;
  __syncthreads();
  int64_t E = 0;
  for (int w = 0; w < kBucketThreads / 32; ++w) E += scr[w];
  __syncthreads();
  if (E == 0) {
    if (tid == 0) mode[q] = 2;  // no postings at all
    return;
  }
  if (E > capq || E > 96LL * nchunks) {
    if (tid == 0) mode[q] = 0;  // stream this query's lists in stage 1
    return;
  }
  for (int c = tid; c < nchunks; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  for (int d = 0; d < nd; ++d) {
    const uint32_t b = lbeg[qb + d], L = lend[qb + d] - b;
    for (uint32_t j = tid; j < L; j += blockDim.x) atomicAdd(&cnt[__ldg(&post[b + j].x) >> 12], 1u);
  }
  __syncthreads();
  {
    // a chunk with very many entries is summed in O(entries^2) by stage 1's
    // first-of-point pass: stream such queries instead
    uint32_t mx = 0;
    for (int c = tid; c < nchunks; c += blockDim.x) mx = max(mx, cnt[c]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) scr[tid >> 5] = (int)mx;
    __syncthreads();
    for (int w = 0; w < kBucketThreads / 32; ++w) mx = max(mx, (uint32_t)scr[w]);
    __syncthreads();
    if (mx > 1024u) {
      if (tid == 0) mode[q] = 0;
      return;
    }
  }
  // exclusive scan of the histogram (segment per thread, then across threads)
  const int per = (nchunks + kBucketThreads - 1) / kBucketThreads;
  const int c0 = min(nchunks, tid * per), c1 = min(nchunks, c0 + per);
  uint32_t run = 0;
  for (int c = c0; c < c1; ++c) run += cnt[c];
  uint32_t incl = run;
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) scr[warp] = (int)incl;
  __syncthreads();
  uint32_t base = incl - run;
  for (int w = 0; w < warp; ++w) base += (uint32_t)scr[w];
  __syncthreads();
  uint32_t* qb_off = boff + q * (int64_t)(nchunks + 1);
  for (int c = c0; c < c1; ++c) {
    const uint32_t v = cnt[c];
    cnt[c] = base;
    qb_off[c] = base;
    base += v;
  }
  if (tid == 0) {
    qb_off[nchunks] = (uint32_t)E;
    mode[q] = 1;
  }
  __syncthreads();
  uint32_t* qs = slots + q * capq;
  double* qvv = vals + q * capq;
  for (int d = 0; d < nd; ++d) {
    const uint32_t b = lbeg[qb + d], L = lend[qb + d] - b;
    const double qvd = qv[qb + d];
    for (uint32_t jb = 0; jb < L; jb += blockDim.x) {
      const uint32_t j = jb + tid;
      const bool valid = j < L;
      uint2 pw = make_uint2(0u, 0u);
      uint32_t c = 0xFFFFFFFFu;
      bool start = false, end = false;
      if (valid) {
        pw = __ldg(&post[b + j]);
        c = pw.x >> 12;
        start = (j == jb) || ((__ldg(&post[b + j - 1].x) >> 12) != c);
        end = (j + 1 == L) || (tid == kBucketThreads - 1) || ((__ldg(&post[b + j + 1].x) >> 12) != c);
      }
      const int rs = block_max_scan(start ? tid : -1, scr);
      uint32_t pos = 0;
      if (valid) {
        pos = cnt[c] + (uint32_t)(tid - rs);
        qs[pos] = pw.x;
        qvv[pos] = qvd * (double)__uint_as_float(pw.y);  // exact product of two f32
      }
      __syncthreads();  // every thread has used the old cursor
      if (valid && end) cnt[c] += (uint32_t)(tid - rs + 1);
      __syncthreads();
    }
  }
}

// Per-point aggregation of the buckets: one warp per (query, chunk) bucket.
// A slot bitmap finds the buckets with repeated points (rare with pruned
// lists; those without are left as they are).  A bucket with repeats is
// stably sorted by slot in shared memory, each point's run summed in bucket
// order — ascending dim, the reference's per-point order (sparse.py:277-282)
// — from +0.0, and rewritten: the sums compacted to its front (ascending
// slot), then kNoSlot entries.  Consumers read one entry per touched point.
// Buckets hold <= 1024 entries (k_sparse_bucket streams queries with fuller
// chunks).
constexpr int kAggWarps = 8;
constexpr int kAggMax = 1024;

__global__ void __launch_bounds__(kAggWarps * 32) k_bucket_aggregate(
    const int* __restrict__ mode, const uint32_t* __restrict__ boff, int nchunks, int64_t capq,
    uint32_t* __restrict__ slots, double* __restrict__ vals) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t q = blockIdx.x;
  if (mode[q] != 1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one sort staging area per CTA (buckets with repeats are rare), taken
  // under a shared-memory lock; a 4096-bit slot bitmap per warp
  double* val = reinterpret_cast<double*>(smem_raw);
  uint32_t* slt = reinterpret_cast<uint32_t*>(smem_raw + sizeof(double) * kAggMax);
  uint32_t* seen = slt + kAggMax + warp * (kChunk / 32);
  int* lock = reinterpret_cast<int*>(slt + kAggMax + kAggWarps * (kChunk / 32));
  if (threadIdx.x == 0) *lock = 0;
  for (int i = lane; i < kChunk / 32; i += 32) seen[i] = 0u;
  __syncthreads();
  const uint32_t* qb = boff + q * (int64_t)(nchunks + 1);
  uint32_t* qs = slots + q * capq;
  double* qv = vals + q * capq;
  for (int c = blockIdx.y * kAggWarps + warp; c < nchunks; c += gridDim.y * kAggWarps) {
    const uint32_t b0 = qb[c];
    const int L = (int)(qb[c + 1] - b0);
    if (L <= 1) continue;
    const uint32_t cbase = (uint32_t)c << 12;
    // pass 1: any repeated point?  (bitmap of the slots seen, cleared after)
    bool rep = false;
    for (int i = lane; i < L; i += 32) {
      const uint32_t ls = __ldg(qs + b0 + i) - cbase;
      const uint32_t bit = 1u << (ls & 31);
      rep |= (atomicOr(&seen[ls >> 5], bit) & bit) != 0u;
    }
    __syncwarp();
    for (int i = lane; i < L; i += 32) seen[(__ldg(qs + b0 + i) - cbase) >> 5] = 0u;
    __syncwarp();
    if (!__any_sync(0xffffffffu, rep)) continue;
    if (lane == 0)
      while (atomicCAS(lock, 0, 1) != 0) __nanosleep(64);
    __syncwarp();
    // pass 2 (buckets with repeats): stable sort by slot — key = local slot
    // << 10 | entry index — so each point's entries form a run in bucket
    // (= ascending dim) order; run heads sum their runs from +0.0
    int P = 32;
    while (P < L) P <<= 1;
    for (int i = lane; i < P; i += 32) {
      if (i < L) {
        slt[i] = ((qs[b0 + i] - cbase) << 10) | (uint32_t)i;
        val[i] = qv[b0 + i];
      } else {
        slt[i] = 0xFFFFFFFFu;
      }
    }
    __syncwarp();
    for (int kk = 2; kk <= P; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < P; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint32_t x = slt[i], y = slt[ixj];
            if ((x > y) == ((i & kk) == 0)) {
              slt[i] = y;
              slt[ixj] = x;
            }
          }
        }
        __syncwarp();
      }
    uint32_t out = 0;
    for (int r0 = 0; r0 < L; r0 += 32) {
      const int r = r0 + lane;
      bool head = false;
      uint32_t ls = 0;
      double sum = 0.0;
      if (r < L) {
        const uint32_t k = slt[r];
        ls = k >> 10;
        head = r == 0 || (slt[r - 1] >> 10) != ls;
        if (head) {
          sum += val[k & 1023u];
          for (int t = r + 1; t < L && (slt[t] >> 10) == ls; ++t) sum += val[slt[t] & 1023u];
        }
      }
      const unsigned hb = __ballot_sync(0xffffffffu, head);
      if (head) {
        const uint32_t pos = out + __popc(hb & ((1u << lane) - 1u));
        qs[b0 + pos] = cbase + ls;
        qv[b0 + pos] = sum;
      }
      out += __popc(hb);
    }
    for (uint32_t i = out + lane; i < (uint32_t)L; i += 32) qs[b0 + i] = kNoSlot;
    __syncwarp();
    if (lane == 0) atomicExch(lock, 0);
  }
}

// skip table of one long list: row[c] = #postings with id < 4096*c
__global__ void k_skip_rows(const uint2* __restrict__ post, const uint32_t* __restrict__ ptr,
                            const int32_t* __restrict__ long_lists, int nchunks,
                            uint32_t* __restrict__ skip) {
  const int r = blockIdx.x;
  const int li = long_lists[r];
  const uint32_t b = ptr[li], L = ptr[li + 1] - b;
  uint32_t* row = skip + (int64_t)r * (nchunks + 1);
  for (uint32_t j = threadIdx.x; j <= L; j += blockDim.x) {
    // chunks c in (chunk(j-1), chunk(j)] start at j
    const int64_t cprev = j == 0 ? -1 : (int64_t)(__ldg(&post[b + j - 1].x) >> 12);
    const int64_t ccur = j == L ? (int64_t)nchunks : (int64_t)(__ldg(&post[b + j].x) >> 12);
    for (int64_t c = cprev + 1; c <= ccur; ++c) row[c] = j;
  }
}

}  // namespace

int stage1_chunk_points() { return kChunk; }

int build_skip_tables(DeviceIndex& ix, const int64_t* host_ptr) {
  const int64_t nchunks = ceil_div(ix.n, kChunk);
  std::vector<int32_t> row(ix.n_active, -1);
  std::vector<int32_t> longs;
  for (int64_t i = 0; i < ix.n_active; ++i)
    if (host_ptr[i + 1] - host_ptr[i] >= 2 * nchunks && nchunks > 1) {
      row[i] = (int32_t)longs.size();
      longs.push_back((int32_t)i);
    }
  ix.n_long = (int64_t)longs.size();
  HS_CUDA(cudaMalloc(&ix.skip_row, sizeof(int32_t) * std::max<int64_t>(ix.n_active, 1)));
  if (ix.n_active)
    HS_CUDA(cudaMemcpy(ix.skip_row, row.data(), sizeof(int32_t) * ix.n_active,
                       cudaMemcpyHostToDevice));
  ix.bytes += sizeof(int32_t) * ix.n_active;
  if (ix.n_long == 0) return HS_OK;
  const size_t bytes = sizeof(uint32_t) * ix.n_long * (nchunks + 1);
  HS_CUDA(cudaMalloc(&ix.skip, bytes));
  ix.bytes += (int64_t)bytes;
  int32_t* d_long = nullptr;
  HS_CUDA(cudaMalloc(&d_long, sizeof(int32_t) * ix.n_long));
  HS_CUDA(cudaMemcpy(d_long, longs.data(), sizeof(int32_t) * ix.n_long, cudaMemcpyHostToDevice));
  k_skip_rows<<<(unsigned)ix.n_long, 256>>>(ix.post, ix.post_ptr, d_long, (int)nchunks, ix.skip);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaDeviceSynchronize());
  cudaFree(d_long);
  return HS_OK;
}

// Same tables from the device-resident post_ptr (GPU-built indices).
int build_skip_tables_dev(DeviceIndex& ix) {
  std::vector<uint32_t> p32(ix.n_active + 1);
  HS_CUDA(cudaMemcpy(p32.data(), ix.post_ptr, sizeof(uint32_t) * (ix.n_active + 1),
                     cudaMemcpyDeviceToHost));
  std::vector<int64_t> p64(p32.begin(), p32.end());
  return build_skip_tables(ix, p64.data());
}

int64_t bucket_capacity(const DeviceIndex& ix) {
  const int64_t nchunks = ceil_div(ix.n, kChunk);
  return std::min<int64_t>(96 * nchunks, 32768);
}

void launch_sparse_bucket(const DeviceIndex& ix, const QueryView& q, const uint32_t* lbeg,
                          const uint32_t* lend, const double* qv, const SparseBuckets& sb,
                          cudaStream_t st) {
  if (q.nq <= 0) return;
  const size_t smem = sizeof(uint32_t) * (sb.nchunks + 1) + sizeof(int) * 32;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_sparse_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sparse_bucket<<<(unsigned)q.nq, kBucketThreads, smem, st>>>(
      q.sp_indptr, lbeg, lend, qv, ix.post, sb.nchunks, sb.capq, sb.mode, sb.boff, sb.slots,
      sb.vals);
  const size_t asmem = (sizeof(uint32_t) + sizeof(double)) * kAggMax + kChunk / 8 * kAggWarps + 16;
  if (asmem > 48 * 1024)
    cudaFuncSetAttribute(k_bucket_aggregate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asmem);
  const int ys = (int)std::min<int64_t>(ceil_div(sb.nchunks, kAggWarps), 8);
  k_bucket_aggregate<<<dim3((unsigned)q.nq, (unsigned)ys), kAggWarps * 32, asmem, st>>>(
      sb.mode, sb.boff, sb.nchunks, sb.capq, sb.slots, sb.vals);
}

Stage1Plan plan_stage1(const DeviceIndex& ix, int64_t nq, int64_t k, int max_qnnz, int mode,
                       int64_t n_limit) {
  Stage1Plan p;
  p.mode = mode;
  p.max_qnnz = max_qnnz < 1 ? 1 : max_qnnz;
  const int64_t n = n_limit >= 0 ? std::min(n_limit, ix.n) : ix.n;
  p.n_limit = n;
  const int64_t nchunks = ceil_div(n, kChunk);
  // one wave of resident CTAs (3 per SM): more tiles per query cost more in
  // per-tile selection than they save in wave quantisation (measured)
  const int64_t target_ctas = 3LL * kNumSMs;
  if (mode == S1_SELECT) {
    // enough tiles to fill the GPU, tiles much larger than k so the per-tile
    // keep filters; the merge then sorts ntiles*k entries per query
    const int64_t nqq = nq > 0 ? nq : 1;
    const int64_t min_tile_chunks = ceil_div(8 * k, kChunk);
    int64_t max_tiles = nchunks / (min_tile_chunks > 0 ? min_tile_chunks : 1);
    if (max_tiles * k > 65536) max_tiles = 65536 / (k > 0 ? k : 1);
    if (max_tiles > nchunks) max_tiles = nchunks;
    if (max_tiles < 1) max_tiles = 1;
    // tiles per query: minimise (waves of resident CTAs) x (chunks per tile +
    // a per-tile selection overhead of ~2 chunks) — wave quantisation of
    // nq*ntiles CTAs against per-tile fill/compaction work
    int64_t ntiles = 1;
    double best = 1e300;
    const int64_t t_lo = std::min<int64_t>(max_tiles, ceil_div(target_ctas, nqq));
    for (int64_t t = t_lo; t <= std::min<int64_t>(max_tiles, 4 * t_lo + 8); ++t) {
      const double waves = (double)ceil_div(nqq * t, target_ctas);
      const double cost = waves * ((double)ceil_div(nchunks, t) + 2.0);
      if (cost < best * 0.999) {
        best = cost;
        ntiles = t;
      }
    }
    const int64_t chunks_per_tile = ceil_div(nchunks, ntiles);
    p.tile_pts = chunks_per_tile * kChunk;
    p.ntiles = (int)ceil_div(n, p.tile_pts);
    if (k >= p.tile_pts) {
      p.mode = S1_EMIT_ALL;
      p.out_per_tile = p.tile_pts;
    } else {
      p.k = (int)k;
      p.cap = (int)((k + kOfferRound + 7) / 8 * 8);  // compaction keeps k, a round adds <= kOfferRound
      p.out_per_tile = k;
    }
  } else {
    int64_t ntiles = ceil_div(target_ctas, nq > 0 ? nq : 1);
    if (ntiles > nchunks) ntiles = nchunks;
    if (ntiles < 1) ntiles = 1;
    p.tile_pts = ceil_div(nchunks, ntiles) * kChunk;
    p.ntiles = (int)ceil_div(n, p.tile_pts);
    p.out_per_tile = (mode == S1_EMIT_ALL) ? p.tile_pts : 0;
  }
  if (p.ntiles < 1) p.ntiles = 1;
  return p;
}

static uint32_t ring_bytes_env() {
  static const uint32_t v = [] {
    const char* e = getenv("HSB200_RING_KB");
    const int kb = e ? atoi(e) : 0;
    return kb >= 24 && kb <= 160 ? (uint32_t)kb * 1024u : (uint32_t)kRingBytes;
  }();
  return v;
}

size_t stage1_smem_bytes(const DeviceIndex& ix, const Stage1Plan& p, bool ws) {
  size_t b = sizeof(Cand) * (size_t)(p.mode == S1_SELECT ? p.cap : 0) + sizeof(Cand);
  b += sizeof(double) * kChunk;
  b += 16 * (size_t)ix.Kp;
  b += (sizeof(double) + 8 * sizeof(uint32_t)) * (size_t)p.max_qnnz;
  if (ws)  // posting ring + piece barriers/descriptors
    b += 16 + ring_bytes_env() + (sizeof(uint4) + 3 * sizeof(uint64_t) + sizeof(int)) * kPieceBars +
         2 * sizeof(double);
  b += 8 + (sizeof(double) + sizeof(uint32_t)) * kThreads;  // bucket staging
  b += sizeof(int) * 24;
  return b;
}

void launch_map_dims(const DeviceIndex& ix, const QueryView& q, int64_t nnz, bool use_weight,
                     uint32_t* lbeg, uint32_t* lend, double* qv, int32_t* lidx,
                     cudaStream_t st) {
  if (nnz <= 0) return;
  const int T = 256;
  k_map_dims<<<(unsigned)ceil_div(nnz, T), T, 0, st>>>(
      q.sp_dims, q.sp_vals, nnz, ix.post_dims, ix.n_active, ix.post_ptr,
      (float)ix.sparse_weight, use_weight && ix.sparse_weight != 1.0 ? 1 : 0, lbeg, lend, qv,
      lidx);
}

void launch_scan_into(const DeviceIndex& ix, const QueryView& q, int max_row_nnz,
                      const uint32_t* lbeg, const uint32_t* lend, const double* qv, double* acc,
                      cudaStream_t st) {
  if (q.nq <= 0 || ix.n <= 0 || ix.nnz_post == 0) return;
  for (int k = 0; k < max_row_nnz; ++k) {
    dim3 grid(2 * 148, (unsigned)q.nq);
    k_scan_dim_into<<<grid, 256, 0, st>>>(ix.post, q.sp_indptr, lbeg, lend, qv, k, ix.n, acc);
  }
}

int launch_stage1(const DeviceIndex& ix, const QueryView& q, const Stage1Plan& p,
                  const uint32_t* lbeg, const uint32_t* lend, const double* qv,
                  const int32_t* lidx, const uint8_t* luts, const double* bias_total, const double* scale,
                  const double* offset, Cand* out, double* dump, cudaStream_t st,
                  uint32_t* dump_tot, bool raw_dense, const SparseBuckets* sb,
                  const uint16_t* tot16, int64_t tot_ld) {
  if (q.nq <= 0 || ix.n <= 0) return HS_OK;
  Stage1Args a;
  a.n = p.n_limit >= 0 ? std::min(p.n_limit, ix.n) : ix.n;
  a.qmask = p.qmask;
  a.tile_pts = p.tile_pts;
  a.mode = p.mode;
  a.k = p.k;
  a.cap = p.mode == S1_SELECT ? p.cap : 0;
  a.out_per_tile = p.out_per_tile;
  a.ntiles = p.ntiles;
  a.post = ix.post;
  a.qptr = q.sp_indptr;
  a.lbeg = lbeg;
  a.lend = lend;
  a.qv = qv;
  a.lidx = lidx;
  a.has_dense = (ix.d_dense > 0 && ix.K > 0 && p.use_dense && !p.sparse_only_acc) ? 1 : 0;
  a.K = ix.K;
  a.Kp = ix.Kp;
  a.vcodes = ix.vcodes;
  a.luts = luts;
  a.bias_total = bias_total;
  a.scale = scale;
  a.offset = offset;
  a.order = ix.order;
  a.out = out;
  a.dump = dump;
  a.dump_tot = dump_tot;
  a.raw_dense = raw_dense ? 1 : 0;
  a.max_qnnz = p.max_qnnz;
  a.bmode = sb ? sb->mode : nullptr;
  a.boff = sb ? sb->boff : nullptr;
  a.bslots = sb ? sb->slots : nullptr;
  a.bvals = sb ? sb->vals : nullptr;
  a.capq = sb ? sb->capq : 0;
  a.nchunks_g = sb ? sb->nchunks : 0;
  a.skip_row = ix.skip_row;
  a.skip = ix.skip;
  a.nchunks_all = (int)ceil_div(ix.n, kChunk);
  a.tot16 = tot16;
  a.tot_ld = tot_ld;
  a.ring_bytes = ring_bytes_env();
  {
    static const int exp_flags = [] {
      const char* e = getenv("HSB200_EXP");
      return e ? atoi(e) : 0;
    }();
    a.exp_flags = exp_flags;
  }
  const int dm = !a.has_dense ? 0 : (tot16 != nullptr ? 2 : 1);
  const bool sp = p.sparse && ix.nnz_post > 0 && lbeg != nullptr;
  // warp-specialised posting stream (kernels without the PRMT scan): opt-in
  // with HSB200_WS=1 — measured slower than the single-role kernel on cfg4
  // (1.59 s vs 1.18 s per 10K queries), kept for the experiment
  static const bool ws_env = [] {
    const char* e = getenv("HSB200_WS");
    return e && e[0] == '1';
  }();
  const bool ws = sp && dm != 1 && ws_env;
  const size_t smem = stage1_smem_bytes(ix, p, ws);
  if (smem > 227 * 1024) HS_FAIL(HS_EUNSUPPORTED, "stage-1 shared memory exceeds 227 KB "
                                                  "(too many query nonzeros or candidates)");
  void (*kern)(Stage1Args) = nullptr;
  switch (dm * 2 + (sp ? 1 : 0)) {
    case 0: kern = k_stage1<0, false, false>; break;
    case 1: kern = ws ? k_stage1<0, true, true> : k_stage1<0, true, false>; break;
    case 2: kern = k_stage1<1, false, false>; break;
    case 3: kern = k_stage1<1, true, false>; break;
    case 4: kern = k_stage1<2, false, false>; break;
    default: kern = ws ? k_stage1<2, true, true> : k_stage1<2, true, false>; break;
  }
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)q.nq, (unsigned)p.ntiles);
  kern<<<grid, ws ? kThreads + 32 : kThreads, smem, st>>>(a);
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

}  // namespace hs
