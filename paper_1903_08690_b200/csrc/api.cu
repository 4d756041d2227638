// api.cu — the C ABI (include/hsb200.h): index upload, the batched
// three-stage search driver and the unit entry points.
//
// Search driver (replaces search_topk / search_batch, reference
// pipeline.py:226-300): queries are processed in chunks; per chunk
//   map_dims -> lut_build -> stage1 (fused scan + per-tile top-k) ->
//   select (merge tiles to the top k1) -> stage2 -> stage3 -> outputs,
// all enqueued on the index's stream with no host round trip between stages.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "kernels.cuh"

namespace hs {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

namespace {

bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] && e[0] != '0';
}

template <typename T>
int dalloc(DeviceIndex& ix, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return HS_OK;
  HS_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count));
  ix.bytes += (int64_t)(sizeof(T) * count);
  return HS_OK;
}

template <typename T>
int dupload(DeviceIndex& ix, T** p, const T* src, size_t count) {
  HS_CHECK(dalloc(ix, p, count));
  if (count) HS_CUDA(cudaMemcpy(*p, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HS_OK;
}

__global__ void k_interleave(const uint32_t* ids, const float* w, int64_t n, uint2* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_uint2(ids[i], __float_as_uint(w[i]));
}

__global__ void k_order_u32(const int64_t* in, int64_t n, uint32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)in[i];
}

void free_device_arrays(DeviceIndex* ix) {
  if (!ix) return;
  cudaSetDevice(ix->device);
  void* ptrs[] = {ix->order,    ix->post_dims,  ix->post_ptr, ix->post,       ix->res_indptr,
                  ix->res_indices, ix->res_data, ix->subdims,  ix->dim_off,    ix->cen_off,
                  ix->centers,  ix->vcodes,     ix->sq_lo,    ix->sq_step,    ix->sq_codes,
                  ix->wh_mean,  ix->wh_inv_t,   ix->ds_dense, ix->ds_indptr,  ix->ds_indices,
                  ix->ds_data,  ix->scratch,    ix->skip_row, ix->skip,     ix->io_dev,
                  ix->hcodes,   ix->pcodes,     ix->ds_dense_h, ix->ds_dmask};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ix->io_host) cudaFreeHost(ix->io_host);
  if (ix->stream) cudaStreamDestroy(ix->stream);
  if (ix->aux) cudaStreamDestroy(ix->aux);
  if (ix->ev_fork) cudaEventDestroy(ix->ev_fork);
  if (ix->ev_join) cudaEventDestroy(ix->ev_join);
  if (ix->ev_done) cudaEventDestroy(ix->ev_done);
  for (cudaEvent_t e : ix->evpool) cudaEventDestroy(e);
  ix->evpool.clear();
}

int ensure_scratch(DeviceIndex& ix, size_t bytes) {
  if (bytes <= ix.scratch_bytes) return HS_OK;
  if (ix.scratch) {
    HS_CUDA(cudaStreamSynchronize(ix.stream));
    if (ix.ev_done) HS_CUDA(cudaEventSynchronize(ix.ev_done));
    cudaFree(ix.scratch);
    ix.scratch = nullptr;
    ix.scratch_bytes = 0;
  }
  const size_t want = bytes + bytes / 4;
  HS_CUDA(cudaMalloc(&ix.scratch, want));
  ix.scratch_bytes = want;
  return HS_OK;
}

struct Arena {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * count;
    return p;
  }
};

struct Sizes {
  int64_t k1 = 0, k2 = 0, kh = 0;
};

int resolve_sizes(const DeviceIndex& ix, const hs_search_params* p, Sizes* s) {
  if (!p) HS_FAIL(HS_EINVAL, "null search params");
  if (p->h < 1) HS_FAIL(HS_EINVAL, "h must be >= 1");
  if (!(p->overfetch >= p->retain && p->retain >= 1.0))
    HS_FAIL(HS_EINVAL, "need overfetch >= retain >= 1");
  // k1 = min(n, ceil(alpha*h)); k2 = min(k1, ceil(beta*h)) (pipeline.py:251, 261)
  const double a = std::ceil(p->overfetch * (double)p->h);
  const double b = std::ceil(p->retain * (double)p->h);
  s->k1 = (int64_t)std::min<double>((double)ix.n, a);
  s->k2 = (int64_t)std::min<double>((double)s->k1, b);
  s->kh = std::min<int64_t>(p->h, s->k2);
  return HS_OK;
}

constexpr int64_t kMaxRerank = 8192;  // k1/k2 held in shared memory for stages 2-3
// batches at least this large use the tensor cores; smaller ones stream the
// codes once per query (one tensor-core pass costs about as much as ten
// streamed queries).  HSB200_TC_MIN: dev / test knob.
int64_t tc_min_queries() {
  const char* e = std::getenv("HSB200_TC_MIN");
  return e ? std::max<int64_t>(1, std::atoll(e)) : 16;
}

// time accumulation helpers.  Two modes: FULL records an event after every
// kernel (the bench's per-kernel breakdown; it serialises the aux-stream
// overlap), STAGE records only the stage boundaries StageStats needs (three
// events per chunk, overlap kept).  Events come from a per-index pool.
enum TimerMode { TM_OFF = 0, TM_STAGE = 1, TM_FULL = 2 };
struct Timer {
  DeviceIndex* ix;
  cudaStream_t st;
  int mode;
  size_t used = 0;
  std::vector<std::string> names;
  Timer(DeviceIndex* ix_, cudaStream_t st_, int mode_) : ix(ix_), st(st_), mode(mode_) {}
  bool full() const { return mode == TM_FULL; }
  void record(const char* name) {
    if (used == ix->evpool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      ix->evpool.push_back(e);
    }
    cudaEventRecord(ix->evpool[used++], st);
    names.push_back(name ? name : "");
  }
  // per-kernel mark (FULL only)
  void mark(const char* name) {
    if (mode == TM_FULL) record(name);
  }
  // stage boundary: "begin", "stage1" (end of stage 1), "stage2", "stage3"
  void boundary(const char* name) {
    if (mode == TM_STAGE || (mode == TM_FULL && std::strcmp(name, "stage1") != 0)) record(name);
  }
  // names[i] labels the interval (evs[i-1], evs[i])
  void finish(double* stage_seconds) {
    if (mode == TM_OFF || used == 0) return;
    cudaEventSynchronize(ix->evpool[used - 1]);
    if (mode == TM_FULL) {
      ix->tnames.clear();
      ix->tms.clear();
    }
    double st3[3] = {0, 0, 0};
    for (size_t i = 1; i < used; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ix->evpool[i - 1], ix->evpool[i]);
      const std::string& nm = names[i];
      if (mode == TM_FULL) {
        auto it = std::find(ix->tnames.begin(), ix->tnames.end(), nm);
        if (it == ix->tnames.end()) {
          ix->tnames.push_back(nm);
          ix->tms.push_back(ms);
        } else {
          ix->tms[it - ix->tnames.begin()] += ms;
        }
      }
      if (nm == "stage2") st3[1] += ms;
      else if (nm == "stage3") st3[2] += ms;
      else if (nm != "begin") st3[0] += ms;
    }
    if (stage_seconds)
      for (int i = 0; i < 3; ++i) stage_seconds[i] = st3[i] * 1e-3;
    used = 0;
    names.clear();
  }
};

// Full search for a device-resident query batch.  `max_qnnz`/`nnz` known.
int run_search(DeviceIndex& ix, const hs_query_batch& qb, int64_t nnz, int max_qnnz,
               const hs_search_params* params, int64_t* d_ids, double* d_scores, cudaStream_t st,
               Timer* tm, bool check_lut = false) {
  Sizes sz;
  HS_CHECK(resolve_sizes(ix, params, &sz));
  const int64_t nq = qb.nq;
  if (nq <= 0 || sz.kh <= 0) return HS_OK;
  // every search carves the same scratch arena: a call on another stream
  // must not start before the previous call's kernels are done with it
  if (ix.ev_done) HS_CUDA(cudaStreamWaitEvent(st, ix.ev_done, 0));
  if (ix.d_dense > 0 && ix.K == 0) HS_FAIL(HS_EINVAL, "index has no dense PQ codes");
  if (ix.d_dense > 0 && ix.l != 16) HS_FAIL(HS_EUNSUPPORTED, "lut16_scan requires 16-center codes");
  if (params->exact_final_rerank && !ix.has_ds)
    HS_FAIL(HS_EINVAL, "exact_final_rerank requires the original dataset");
  if (sz.k1 > kMaxRerank)
    HS_FAIL(HS_EUNSUPPORTED, "overfetch*h above 8192 candidates is not supported");
  if (max_qnnz > 8192) HS_FAIL(HS_EUNSUPPORTED, "queries with more than 8192 sparse nonzeros");

  // tensor-core LUT16 for large batches (>= tc_min_queries() queries): either
  // threshold-filtered (fuse.cu: sample -> threshold -> filtered tensor-core
  // pass -> candidate scoring) or, when that does not apply, u16 totals for
  // every point followed by the full stage-1 scan
  const int64_t d = ix.d_dense;
  const int64_t tc_ld = lut16_tc_ld(ix.n);
  const bool use_tc = d > 0 && lut16_tc_supported(ix) && nq >= tc_min_queries() &&
                      !getenv_flag("HSB200_NO_TC");
  // smaller batches: the same threshold-filtered stage 1 with the HBM-bound
  // CUDA-core scan (lut16_stream.cu) in place of the tensor-core pass — every
  // query streams the codes once
  const bool use_stream = d > 0 && !use_tc && lut16_stream_supported(ix) &&
                          !getenv_flag("HSB200_NO_STREAM");
  const bool use_buckets = nnz > 0 && ix.nnz_post > 0 && !getenv_flag("HSB200_NO_BUCKETS");
  const bool sparse_part = nnz > 0 && ix.nnz_post > 0;
  // bucketing overlapped with the dense chain on the aux stream (not while
  // timing: the per-kernel breakdown needs the serial order)
  const bool overlap = use_buckets && ix.aux != nullptr && !(tm && tm->full()) &&
                       !getenv_flag("HSB200_NO_OVERLAP");
  // sample size of the threshold pass and capacity of the filtered lists
  // (HSB200_FUSE_SAMPLE / HSB200_FUSE_CAP: test knobs that shrink the sample
  // and the list capacity so small indices exercise the filter and fallback)
  const char* ev_s = std::getenv("HSB200_FUSE_SAMPLE");
  const char* ev_c = std::getenv("HSB200_FUSE_CAP");
  const int64_t m_min = ev_s ? std::max<int64_t>(128, std::atoll(ev_s)) : 65536;
  // sample ~ k1*n/E points (=> ~E expected dense candidates per query); E
  // grows with k1 so that the sample stays a few percent of a large index
  // (10^8 points, k1 = 1000: a 2M-point sample instead of 17M)
  // ... scaled by sqrt(n / 10^8): the sample pass costs ~ n/E and the candidate
  // scoring + selection ~ E per query, so the best E grows like sqrt(n) (at
  // 10^8 points E = 50 k1 balances the two; an id-range shard of 1/8 of them
  // wants ~18 k1)
  // (HSB200_FUSE_ECAND: candidates per k1 at 10^8 points, a tuning knob)
  static const double e_mult = std::getenv("HSB200_FUSE_ECAND")
                                   ? std::max(1.0, std::atof(std::getenv("HSB200_FUSE_ECAND")))
                                   : 50.0;
  const double e_cand = std::max(
      6000.0, e_mult * (double)sz.k1 * std::min(1.0, std::sqrt((double)ix.n / 1.0e8)));
  const int64_t m_auto = std::max<int64_t>(
      65536, (int64_t)((double)sz.k1 * (double)ix.n / e_cand));
  // (a whole number of stage-1 chunks, so the sample ends on a chunk boundary)
  const int64_t cpts = stage1_chunk_points();
  const int64_t m_s = std::min<int64_t>(
      ix.n, ceil_div(std::max<int64_t>(ev_s ? m_min : m_auto, 4 * sz.k1), cpts) * cpts);
  // threshold from the exact sample top-k1 (full stage-1 kernels) instead of
  // the sample's totals (dev / A-B knob)
  const bool exact_sample = getenv_flag("HSB200_EXACT_SAMPLE");
  const bool use_fuse = (use_tc || use_stream) && ix.K <= 256 && sz.k1 <= 4096 && ix.n >= 8 * m_s &&
                        (!sparse_part || (use_buckets && ix.pcodes != nullptr)) &&
                        !getenv_flag("HSB200_NO_FUSE");
  const int64_t expect = (int64_t)((double)sz.k1 * (double)ix.n / (double)m_s);
  // per-(query, tensor-core CTA) list segments: ~4x the expected passes of
  // the largest share of a query's points one CTA covers, + 64
  int64_t QB = std::min<int64_t>(nq, 2048);
  int64_t nseg = 0, Cf = 0;
  auto seg_cap = [&](int64_t qb) {
    double frac = 1.0;
    if (use_tc) lut16_filter_layout(ix, qb, &nseg, &frac);
    else lut16_stream_layout(ix, &nseg, &frac);
    Cf = ((int64_t)(4.0 * (double)expect * frac) + 64 + 31) / 32 * 32;
    if (ev_c) Cf = std::max<int64_t>(1, std::atoll(ev_c));
  };
  if (use_fuse) seg_cap(QB);
  const int64_t capq_all = use_buckets ? bucket_capacity(ix) : 0;
  // scored candidates: every dense pass (<= the segments) + touched points
  auto cand_rows = [&]() { return std::min<int64_t>(Cf * nseg, ix.n) + capq_all; };
  int64_t Mf = use_fuse ? cand_rows() : 0;
  const int64_t ld_s = lut16_tc_ld(m_s);
  const int64_t words = ceil_div(ix.n, 32);
  // query-chunk size bounded by scratch for the stage-1 per-tile outputs
  if (use_tc || (use_stream && use_fuse)) {
    const int64_t grp = use_tc ? lut16_tc_group(ix) : 1;
    const double per_q = use_fuse
        ? (double)Cf * nseg * 8 + (double)Mf * 16 + (double)ld_s * 2 +
              (sparse_part ? words * 4.0 : 0.0)
        : 2.0 * (double)tc_ld;  // u16 totals [QB][tc_ld]
    // arena budget for the per-chunk stage-1 buffers: half of what the device
    // has free (counting the arena already held), between 2 and 16 GB — larger
    // chunks give the per-query kernels (one CTA per query) more CTAs per
    // launch: cfg5 1236 -> 1197 ms per step from 8 to 16 GB, flat beyond
    // (HSB200_SCRATCH_GB overrides)
    // (decided once per index handle: cudaMemGetInfo is not free on a latency path)
    if (ix.scratch_budget <= 0.0) {
      double bud = 8.0e9;
      if (const char* eb = std::getenv("HSB200_SCRATCH_GB")) {
        bud = std::max(0.5, std::atof(eb)) * 1e9;
      } else {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
          bud = std::min(16.0e9,
                         std::max(2.0e9, 0.5 * ((double)free_b + (double)ix.scratch_bytes)));
      }
      ix.scratch_budget = bud;
    }
    const double budget = ix.scratch_budget;
    const int64_t cap = std::max<int64_t>(grp, (int64_t)(budget / per_q) / grp * grp);
    if (QB > cap) QB = cap;
  }
  if (use_fuse) {  // layout of the final chunk size (segments depend on it)
    int64_t worst_seg = 0, worst_cf = 0;
    for (int64_t qb : {QB, nq % QB}) {
      if (qb <= 0) continue;
      seg_cap(qb);
      worst_seg = std::max(worst_seg, nseg);
      worst_cf = std::max(worst_cf, Cf);
    }
    nseg = worst_seg;
    Cf = worst_cf;
    Mf = cand_rows();
  }
  int64_t s1_entries = 0;
  for (;;) {
    const Stage1Plan p0 = plan_stage1(ix, QB, sz.k1, max_qnnz, S1_SELECT);
    s1_entries = QB * p0.ntiles * p0.out_per_tile;
    const int64_t last = nq % QB;
    if (last) {
      const Stage1Plan p1 = plan_stage1(ix, last, sz.k1, max_qnnz, S1_SELECT);
      s1_entries = std::max<int64_t>(s1_entries, last * p1.ntiles * p1.out_per_tile);
    }
    if (use_fuse) {
      const Stage1Plan ps = plan_stage1(ix, QB, sz.k1, max_qnnz, S1_SELECT, m_s);
      s1_entries = std::max<int64_t>(s1_entries, QB * ps.ntiles * ps.out_per_tile);
      if (last) {
        const Stage1Plan ps1 = plan_stage1(ix, last, sz.k1, max_qnnz, S1_SELECT, m_s);
        s1_entries = std::max<int64_t>(s1_entries, last * ps1.ntiles * ps1.out_per_tile);
      }
    }
    if ((double)s1_entries * sizeof(Cand) <= 1.0e9 || QB == 1) break;
    QB = (QB + 1) / 2;
  }
  const int Kp16 = ix.Kp * 16;
  const int64_t nchunks = ceil_div(ix.n, stage1_chunk_points());
  const int64_t capq = bucket_capacity(ix);
  size_t need = 0;
  auto carve = [&](auto& a) {
    struct Ptrs {
      uint32_t *lbeg, *lend;
      double* qv;
      int32_t* lidx;
      double *qd, *qw;
      uint8_t* luts;
      double *btot, *scl, *off;
      int* bad;
      Cand *s1out, *cand1, *cand2;
      SparseBuckets sb;
      uint16_t* tot16;
      // fused path
      uint16_t* tot_s;
      Cand* cand_s;
      double* T;
      uint32_t* tlim;
      uint2* list;
      uint32_t* lcnt;
      Cand* fout;
      uint32_t* fcnt;
      int* fallback;
      uint32_t* bitmap;
    } p{};
    p.lbeg = a.template take<uint32_t>(nnz + 1);
    p.lend = a.template take<uint32_t>(nnz + 1);
    p.qv = a.template take<double>(nnz + 1);
    p.lidx = a.template take<int32_t>(nnz + 1);
    p.qd = a.template take<double>(QB * d + 1);
    p.qw = a.template take<double>(QB * d + 1);
    p.luts = a.template take<uint8_t>(QB * Kp16 + 16);
    p.btot = a.template take<double>(QB);
    p.scl = a.template take<double>(QB);
    p.off = a.template take<double>(QB);
    p.bad = a.template take<int>(QB);
    p.s1out = a.template take<Cand>((size_t)s1_entries + 1);
    p.cand1 = a.template take<Cand>(QB * sz.k1 + 1);
    p.cand2 = a.template take<Cand>(QB * sz.k2 + 1);
    if (use_buckets) {
      p.sb.mode = a.template take<int>(QB);
      p.sb.boff = a.template take<uint32_t>(QB * (nchunks + 1));
      p.sb.slots = a.template take<uint32_t>(QB * capq);
      p.sb.vals = a.template take<double>(QB * capq);
      p.sb.capq = capq;
      p.sb.nchunks = (int)nchunks;
    }
    if (use_tc && !use_fuse) p.tot16 = a.template take<uint16_t>(QB * tc_ld);
    if (use_fuse) {
      p.tot_s = a.template take<uint16_t>(QB * ld_s);
      p.cand_s = exact_sample ? a.template take<Cand>(QB * sz.k1 + 1) : nullptr;
      p.T = a.template take<double>(QB);
      p.tlim = a.template take<uint32_t>(QB);
      p.list = a.template take<uint2>(QB * nseg * Cf);
      p.lcnt = a.template take<uint32_t>(QB * nseg);
      p.fout = a.template take<Cand>(QB * Mf);
      p.fcnt = a.template take<uint32_t>(QB);
      p.fallback = a.template take<int>(QB);
      if (sparse_part) p.bitmap = a.template take<uint32_t>(QB * words);
    }
    return p;
  };
  {
    Arena a{nullptr};
    carve(a);
    need = a.off + 1024;
  }
  HS_CHECK(ensure_scratch(ix, need));
  Arena arena{static_cast<char*>(ix.scratch)};
  auto P = carve(arena);
  uint32_t* lbeg = P.lbeg;
  uint32_t* lend = P.lend;
  double* qv = P.qv;
  int32_t* lidx = P.lidx;
  double* qd = P.qd;
  double* qw = P.qw;
  uint8_t* luts = P.luts;
  double* btot = P.btot;
  double* scl = P.scl;
  double* off = P.off;
  int* bad = P.bad;
  Cand* s1out = P.s1out;
  Cand* cand1 = P.cand1;
  Cand* cand2 = P.cand2;
  SparseBuckets sb = P.sb;
  uint16_t* tot16 = P.tot16;

  if (tm) tm->boundary("begin");
  QueryView all;
  all.nq = nq;
  all.sp_indptr = qb.sp_indptr;
  all.sp_dims = qb.sp_dims;
  all.sp_vals = qb.sp_vals;
  all.dense = qb.dense;
  launch_map_dims(ix, all, nnz, true, lbeg, lend, qv, lidx, st);
  ix.launches += nnz > 0 ? 1 : 0;
  if (tm) tm->mark("map_dims");
  if (d > 0) HS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int) * QB, st));
  if (use_fuse && sparse_part)
    HS_CUDA(cudaMemsetAsync(P.bitmap, 0, sizeof(uint32_t) * QB * words, st));

  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nqc = std::min(QB, nq - q0);
    QueryView qc;
    qc.nq = nqc;
    qc.sp_indptr = qb.sp_indptr + q0;
    qc.sp_dims = qb.sp_dims;
    qc.sp_vals = qb.sp_vals;
    qc.dense = qb.dense ? qb.dense + q0 * d : nullptr;
    Stage1Plan pc = plan_stage1(ix, nqc, sz.k1, max_qnnz, S1_SELECT);
    pc.sparse = nnz > 0;
    if (d > 0) {
      launch_lut_build(ix, qc.dense, nqc, qd, qw, luts, btot, scl, off, bad, st);
      HS_CUDA(cudaGetLastError());
      ix.launches += 1;
      if (tm) tm->mark("lut_build");
    }
    bool sb_pending = false;  // bucketing in flight on the aux stream
    if (use_buckets) {
      if (overlap) {  // fork: aux waits for everything issued so far on st
        HS_CUDA(cudaEventRecord(ix.ev_fork, st));
        HS_CUDA(cudaStreamWaitEvent(ix.aux, ix.ev_fork, 0));
        launch_sparse_bucket(ix, qc, lbeg, lend, qv, sb, ix.aux);
        HS_CUDA(cudaEventRecord(ix.ev_join, ix.aux));
        sb_pending = true;
      } else {
        launch_sparse_bucket(ix, qc, lbeg, lend, qv, sb, st);
      }
      HS_CUDA(cudaGetLastError());
      ix.launches += 1;
      if (tm) tm->mark("sparse_bucket");
    }
    auto join_sb = [&]() -> int {  // before the first consumer of the buckets
      if (sb_pending) {
        HS_CUDA(cudaStreamWaitEvent(st, ix.ev_join, 0));
        sb_pending = false;
      }
      return HS_OK;
    };
    // every chunk of a tensor-core batch stays on the tensor cores: a short
    // last chunk gets a narrower query group (the MMA N shrinks with it)
    const bool tc_chunk = use_tc;
    if (use_fuse) {
      // 1. u16 totals of the first m_s points -> threshold
      if (tc_chunk) HS_CHECK(launch_lut16_tc(ix, luts, nqc, P.tot_s, ld_s, st, m_s));
      else HS_CHECK(launch_lut16_stream_totals(ix, luts, nqc, P.tot_s, ld_s, st, m_s));
      ix.launches += 1;
      if (exact_sample) {
      HS_CHECK(join_sb());
      Stage1Plan ps = plan_stage1(ix, nqc, sz.k1, max_qnnz, S1_SELECT, m_s);
      ps.sparse = nnz > 0;
      HS_CHECK(launch_stage1(ix, qc, ps, lbeg, lend, qv, lidx, luts, btot, scl, off, s1out,
                             nullptr, st, nullptr, false, use_buckets ? &sb : nullptr, P.tot_s,
                             ld_s));
      HS_CHECK(launch_select_topk(s1out, nqc, (int64_t)ps.ntiles * ps.out_per_tile, sz.k1,
                                  P.cand_s, st));
      launch_tlim(P.cand_s, nqc, (int)sz.k1, btot, scl, off, P.tlim, P.T, st);
      ix.launches += 3;
      } else {
        launch_sample_tlim(P.tot_s, ld_s, m_s, nqc, (int)sz.k1, nnz > 0 ? qc.sp_indptr : nullptr, qv,
                           ix.post_wmin, ix.post_wmax, btot, scl, off, P.tlim, P.T, st);
        ix.launches += 1;
      }
      if (tm) tm->mark("sample");
      // 2. filtered pass over every point (tensor cores, or the streamed scan)
      if (tc_chunk) HS_CHECK(launch_lut16_filter(ix, luts, nqc, P.tlim, P.list, P.lcnt, Cf, st));
      else HS_CHECK(launch_lut16_stream_filter(ix, luts, nqc, P.tlim, P.list, P.lcnt, Cf, st));
      ix.launches += 1;
      if (tm) tm->mark(tc_chunk ? "lut16_tc" : "lut16_stream");
      // 3. candidate scoring (+ touched points) and exact top-k1
      int64_t nseg_c = 0;
      double frac_c = 1.0;
      if (tc_chunk) lut16_filter_layout(ix, nqc, &nseg_c, &frac_c);
      else lut16_stream_layout(ix, &nseg_c, &frac_c);
      HS_CHECK(join_sb());
      HS_CHECK(launch_fuse_cands(ix, nqc, luts, btot, scl, off, P.list, P.lcnt, Cf, (int)nseg_c,
                                 sparse_part ? &sb : nullptr, P.bitmap, P.fout, Mf, P.fcnt,
                                 P.fallback, P.T, st));
      if (tm) tm->mark("fuse");
      HS_CHECK(launch_select_topk(P.fout, nqc, Mf, sz.k1, cand1, st, P.fcnt));
      ix.launches += 2;
      if (tm) tm->mark("fuse_select");
      // 4. flagged queries (overflow / streamed postings): unfiltered stage 1
      Stage1Plan pf = pc;
      pf.qmask = P.fallback;
      HS_CHECK(launch_stage1(ix, qc, pf, lbeg, lend, qv, lidx, luts, btot, scl, off, s1out,
                             nullptr, st, nullptr, false, use_buckets ? &sb : nullptr));
      HS_CHECK(launch_select_topk(s1out, nqc, (int64_t)pf.ntiles * pf.out_per_tile, sz.k1,
                                  cand1, st, nullptr, P.fallback));
      ix.launches += 2;
      if (tm) tm->mark("fallback");
    } else {
      if (tc_chunk) {
        HS_CHECK(launch_lut16_tc(ix, luts, nqc, tot16, tc_ld, st));
        ix.launches += 1;
        if (tm) tm->mark("lut16_tc");
      }
      ix.launches += 2;  // stage1, merge
      HS_CHECK(join_sb());
      HS_CHECK(launch_stage1(ix, qc, pc, lbeg, lend, qv, lidx, luts, btot, scl, off, s1out,
                             nullptr, st, nullptr, false, use_buckets ? &sb : nullptr,
                             tc_chunk ? tot16 : nullptr, tc_ld));
      if (tm) tm->mark("stage1");
      HS_CHECK(launch_select_topk(s1out, nqc, (int64_t)pc.ntiles * pc.out_per_tile, sz.k1,
                                  cand1, st));
      if (tm) tm->mark("merge");
    }
    HS_CHECK(join_sb());
    if (tm) tm->boundary("stage1");
    ix.launches += 2;  // stage2, stage3
    launch_stage2(ix, cand1, nqc, (int)sz.k1, (int)sz.k2, qw, cand2, st);
    HS_CUDA(cudaGetLastError());
    if (tm) tm->boundary("stage2");
    launch_stage3(ix, qc, cand2, nqc, (int)sz.k2, (int)sz.kh, params->exact_final_rerank ? 1 : 0,
                  max_qnnz, qd, d_ids + q0 * sz.kh, d_scores + q0 * sz.kh, st);
    HS_CUDA(cudaGetLastError());
    if (tm) tm->boundary("stage3");
  }
  if (ix.ev_done) HS_CUDA(cudaEventRecord(ix.ev_done, st));
  if (check_lut && d > 0) {
    std::vector<int> hb(QB);
    HS_CUDA(cudaMemcpyAsync(hb.data(), bad, sizeof(int) * QB, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    for (int v : hb)
      if (v) HS_FAIL(HS_EINVAL, "lookup table contains non-finite values");
  }
  return HS_OK;
}

// host query batch -> device copies through the handle's pinned staging
// buffer; `result_bytes` more device bytes are reserved after the queries for
// the caller's outputs (DevQueries::out)
struct DevQueries {
  hs_query_batch b{};
  int64_t nnz = 0;
  int max_row = 0;
  char* out = nullptr;       // device result area
  char* out_host = nullptr;  // pinned host mirror of it
};

int grow(void** p, size_t* have, size_t want, bool host, cudaStream_t st,
         cudaEvent_t done = nullptr) {
  if (want <= *have) return HS_OK;
  HS_CUDA(cudaStreamSynchronize(st));
  if (done) HS_CUDA(cudaEventSynchronize(done));
  if (*p) host ? cudaFreeHost(*p) : cudaFree(*p);
  *p = nullptr;
  *have = 0;
  const size_t bytes = want + want / 4 + 4096;
  if (host) HS_CUDA(cudaMallocHost(p, bytes));
  else HS_CUDA(cudaMalloc(p, bytes));
  *have = bytes;
  return HS_OK;
}

int upload_queries(DeviceIndex& ix, const hs_query_batch* q, DevQueries* out, bool check,
                   size_t result_bytes = 0) {
  if (!q || q->nq < 0) HS_FAIL(HS_EINVAL, "bad query batch");
  const int64_t nq = q->nq;
  const int64_t base = nq ? q->sp_indptr[0] : 0;
  const int64_t nnz = nq ? q->sp_indptr[nq] - base : 0;
  int max_row = 0;
  for (int64_t i = 0; i < nq; ++i) {
    const int64_t len = q->sp_indptr[i + 1] - q->sp_indptr[i];
    if (len < 0) HS_FAIL(HS_EINVAL, "query indptr not monotone");
    max_row = std::max<int64_t>(max_row, len);
  }
  if (check)
    for (int64_t i = 0; i < nnz; ++i)
      if ((int64_t)q->sp_dims[base + i] >= ix.d_sparse)
        HS_FAIL(HS_EINVAL, "query sparse dimension out of range");
  if (ix.d_dense > 0 && nq > 0 && !q->dense) HS_FAIL(HS_EINVAL, "query dense dimension mismatch");
  Arena lay{nullptr};
  const size_t o_ptr = (size_t)lay.take<int64_t>(nq + 1);
  const size_t o_dims = (size_t)lay.take<uint32_t>(nnz + 1);
  const size_t o_vals = (size_t)lay.take<float>(nnz + 1);
  const size_t o_dense = (size_t)lay.take<float>(nq * ix.d_dense + 1);
  const size_t in_bytes = lay.off;
  const size_t o_out = (size_t)lay.take<char>(result_bytes + 1);
  HS_CHECK(grow(&ix.io_dev, &ix.io_dev_bytes, lay.off, false, ix.stream, ix.ev_done));
  HS_CHECK(grow(&ix.io_host, &ix.io_host_bytes, lay.off, true, ix.stream, ix.ev_done));
  char* hb = static_cast<char*>(ix.io_host);
  char* db = static_cast<char*>(ix.io_dev);
  int64_t* hp = reinterpret_cast<int64_t*>(hb + o_ptr);
  for (int64_t i = 0; i <= nq; ++i) hp[i] = q->sp_indptr[i] - base;
  if (nnz) {
    std::memcpy(hb + o_dims, q->sp_dims + base, sizeof(uint32_t) * nnz);
    std::memcpy(hb + o_vals, q->sp_vals + base, sizeof(float) * nnz);
  }
  if (ix.d_dense > 0 && nq > 0)
    std::memcpy(hb + o_dense, q->dense, sizeof(float) * nq * ix.d_dense);
  HS_CUDA(cudaMemcpyAsync(db, hb, in_bytes, cudaMemcpyHostToDevice, ix.stream));
  out->b.nq = nq;
  out->b.sp_indptr = reinterpret_cast<int64_t*>(db + o_ptr);
  out->b.sp_dims = reinterpret_cast<uint32_t*>(db + o_dims);
  out->b.sp_vals = reinterpret_cast<float*>(db + o_vals);
  out->b.dense = ix.d_dense > 0 ? reinterpret_cast<float*>(db + o_dense) : nullptr;
  out->b.nnz = nnz;
  out->b.max_row_nnz = max_row;
  out->nnz = nnz;
  out->max_row = max_row;
  out->out = db + o_out;
  out->out_host = hb + o_out;
  return HS_OK;
}

int derive_hints(DeviceIndex& ix, const hs_query_batch* q, int64_t* nnz, int* max_row,
                 cudaStream_t st) {
  if (q->nnz > 0 && q->max_row_nnz > 0) {
    *nnz = q->nnz;
    *max_row = q->max_row_nnz;
    return HS_OK;
  }
  std::vector<int64_t> ptr(q->nq + 1);
  HS_CUDA(cudaMemcpyAsync(ptr.data(), q->sp_indptr, sizeof(int64_t) * (q->nq + 1),
                          cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  *nnz = ptr[q->nq] - ptr[0];
  int m = 0;
  for (int64_t i = 0; i < q->nq; ++i) m = std::max<int64_t>(m, ptr[i + 1] - ptr[i]);
  *max_row = m;
  (void)ix;
  return HS_OK;
}

}  // namespace
}  // namespace hs

using namespace hs;

struct hs_index : public hs::DeviceIndex {};
struct hs_builder : public hs::Builder {};

namespace hs {
static void free_index(hs_index* ix) {
  if (!ix) return;
  free_device_arrays(ix);
  delete ix;
}
}  // namespace hs

namespace {
// device buffers of a unit entry point, freed on every return path
struct TmpBufs {
  DeviceIndex ix;
  std::vector<void*> ptrs;
  template <typename T>
  int alloc(T** p, size_t count) {
    HS_CHECK(dalloc(ix, p, count));
    ptrs.push_back(*p);
    return HS_OK;
  }
  template <typename T>
  int upload(T** p, const T* src, size_t count) {
    HS_CHECK(dupload(ix, p, src, count));
    ptrs.push_back(*p);
    return HS_OK;
  }
  ~TmpBufs() {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};
}  // namespace

extern "C" {

const char* hs_last_error(void) { return hs::last_error(); }
const char* hs_version(void) { return "hsb200 0.1.0 (sm_100a)"; }

int hs_index_create(const hs_index_desc* ds, int device, hs_index_t* out) {
  if (!ds || !out) HS_FAIL(HS_EINVAL, "null argument");
  *out = nullptr;
  if (ds->n < 0 || ds->n >= (int64_t)0xFFFFFFFFLL) HS_FAIL(HS_EINVAL, "n out of range (< 2^32)");
  if (ds->d_sparse < 0 || ds->d_sparse > (int64_t)0xFFFFFFFFLL)
    HS_FAIL(HS_EINVAL, "d_sparse must be < 2^32");
  const int64_t nnz_post = ds->n_active ? ds->post_ptr[ds->n_active] : 0;
  if (nnz_post >= (int64_t)0xFFFFFFFFLL) HS_FAIL(HS_EINVAL, "more than 2^32 postings");
  // indices the kernels dereference: reject a corrupt (e.g. hand-edited file)
  // index here rather than read out of bounds on the device
  for (int64_t i = 0; i < ds->n; ++i)
    if (ds->order[i] < 0 || ds->order[i] >= ds->n) HS_FAIL(HS_EINVAL, "layout order out of range");
  for (int64_t a = 0; a < ds->n_active; ++a) {
    if ((int64_t)ds->post_dims[a] >= ds->d_sparse) HS_FAIL(HS_EINVAL, "posting dimension out of range");
    if (ds->post_ptr[a + 1] < ds->post_ptr[a]) HS_FAIL(HS_EINVAL, "posting offsets not ascending");
  }
  if (ds->n_active > 0 && ds->post_ptr[0] != 0) HS_FAIL(HS_EINVAL, "posting offsets must start at 0");
  for (int64_t e = 0; e < nnz_post; ++e)
    if ((int64_t)ds->post_ids[e] >= ds->n) HS_FAIL(HS_EINVAL, "posting id out of range");
  // CSR row pointers the rerank kernels dereference (scipy's csr_matrix only
  // checks the first and last entry): start at 0, monotone, columns in range
  auto check_csr = [&](const int64_t* indptr, const uint32_t* indices, const char* what) -> int {
    if (!indptr || ds->n == 0) return HS_OK;
    if (indptr[0] != 0) HS_FAIL(HS_EINVAL, std::string(what) + " row pointers must start at 0");
    for (int64_t i = 0; i < ds->n; ++i)
      if (indptr[i + 1] < indptr[i]) HS_FAIL(HS_EINVAL, std::string(what) + " row pointers not monotone");
    const int64_t nnz = indptr[ds->n];
    if (nnz > 0 && !indices) HS_FAIL(HS_EINVAL, std::string(what) + " column indices missing");
    for (int64_t e = 0; e < nnz; ++e)
      if ((int64_t)indices[e] >= ds->d_sparse)
        HS_FAIL(HS_EINVAL, std::string(what) + " column index out of range");
    return HS_OK;
  };
  HS_CHECK(check_csr(ds->res_indptr, ds->res_indices, "sparse residual"));
  if (ds->has_dataset) {
    if (!ds->ds_indptr) HS_FAIL(HS_EINVAL, "dataset row pointers missing");
    HS_CHECK(check_csr(ds->ds_indptr, ds->ds_indices, "dataset"));
    if (ds->d_dense > 0 && !ds->ds_dense) HS_FAIL(HS_EINVAL, "dataset dense part missing");
  }
  HS_CUDA(cudaSetDevice(device));
  std::unique_ptr<hs_index, void (*)(hs_index*)> ix(new hs_index(), [](hs_index* p) {
    hs::free_index(p);
  });
  ix->device = device;
  ix->n = ds->n;
  ix->d_sparse = ds->d_sparse;
  ix->d_dense = ds->d_dense;
  ix->id_offset = ds->id_offset;
  ix->sparse_weight = ds->sparse_weight;
  ix->dense_weight = ds->dense_weight;
  HS_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
  HS_CUDA(cudaStreamCreateWithFlags(&ix->aux, cudaStreamNonBlocking));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_fork, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_join, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_done, cudaEventDisableTiming));
  const int64_t n = ds->n;
  const int T = 256;

  // order (u32 on device)
  {
    int64_t* tmp = nullptr;
    HS_CUDA(cudaMalloc(&tmp, sizeof(int64_t) * std::max<int64_t>(n, 1)));
    if (n) HS_CUDA(cudaMemcpy(tmp, ds->order, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    HS_CHECK(dalloc(*ix, &ix->order, std::max<int64_t>(n, 1)));
    if (n) k_order_u32<<<(unsigned)ceil_div(n, T), T>>>(tmp, n, ix->order);
    HS_CUDA(cudaDeviceSynchronize());
    cudaFree(tmp);
  }
  // postings
  ix->n_active = ds->n_active;
  ix->nnz_post = nnz_post;
  {
    std::vector<uint32_t> ptr32(ds->n_active + 1);
    for (int64_t i = 0; i <= ds->n_active; ++i) ptr32[i] = (uint32_t)(ds->n_active ? ds->post_ptr[i] : 0);
    HS_CHECK(dupload(*ix, &ix->post_dims, ds->post_dims, ds->n_active));
    HS_CHECK(dupload(*ix, &ix->post_ptr, ptr32.data(), ds->n_active + 1));
    if (nnz_post) {
      uint32_t* tid = nullptr;
      float* tw = nullptr;
      HS_CUDA(cudaMalloc(&tid, sizeof(uint32_t) * nnz_post));
      HS_CUDA(cudaMalloc(&tw, sizeof(float) * nnz_post));
      HS_CUDA(cudaMemcpy(tid, ds->post_ids, sizeof(uint32_t) * nnz_post, cudaMemcpyHostToDevice));
      HS_CUDA(cudaMemcpy(tw, ds->post_w, sizeof(float) * nnz_post, cudaMemcpyHostToDevice));
      if (ix->d_dense > 0) {  // weight range: the filtered stage 1's sparse lower bound
        float lo = ds->post_w[0], hi = ds->post_w[0];
        for (int64_t i = 1; i < nnz_post; ++i) {
          lo = std::min(lo, ds->post_w[i]);
          hi = std::max(hi, ds->post_w[i]);
        }
        ix->post_wmin = lo;
        ix->post_wmax = hi;
      }
      // one pad posting: the stream copies 16-byte pairs and may read past the end
      HS_CHECK(dalloc(*ix, &ix->post, nnz_post + 1));
      HS_CUDA(cudaMemset(ix->post + nnz_post, 0xFF, sizeof(uint2)));
      k_interleave<<<(unsigned)ceil_div(nnz_post, T), T>>>(tid, tw, nnz_post, ix->post);
      HS_CUDA(cudaDeviceSynchronize());
      cudaFree(tid);
      cudaFree(tw);
    } else {
      HS_CHECK(dalloc(*ix, &ix->post, 1));
    }
  }
  if (nnz_post) HS_CHECK(build_skip_tables(*ix, ds->post_ptr));
  // sparse residual
  if (ds->res_indptr && n) {
    ix->res_nnz = ds->res_indptr[n] - ds->res_indptr[0];
    HS_CHECK(dupload(*ix, &ix->res_indptr, ds->res_indptr, n + 1));
    HS_CHECK(dupload(*ix, &ix->res_indices, ds->res_indices, ix->res_nnz));
    HS_CHECK(dupload(*ix, &ix->res_data, ds->res_data, ix->res_nnz));
  }
  // dense
  if (ds->d_dense > 0 && ds->n_subspaces > 0) {
    const int K = ds->n_subspaces;
    ix->K = K;
    ix->l = ds->n_centers;
    ix->Kp = (K + 1) & ~1;
    ix->npairs = (K + 1) / 2;
    std::vector<int32_t> doff(K), coff(K);
    int64_t dsum = 0, csum = 0;
    for (int k = 0; k < K; ++k) {
      doff[k] = (int32_t)dsum;
      coff[k] = (int32_t)csum;
      dsum += ds->subdims[k];
      csum += (int64_t)ds->subdims[k] * ds->n_centers;
      ix->max_width = std::max(ix->max_width, ds->subdims[k]);
    }
    if (dsum != ds->d_dense) HS_FAIL(HS_EINVAL, "subspace widths do not sum to d_dense");
    HS_CHECK(dupload(*ix, &ix->subdims, ds->subdims, K));
    HS_CHECK(dupload(*ix, &ix->dim_off, doff.data(), K));
    HS_CHECK(dupload(*ix, &ix->cen_off, coff.data(), K));
    HS_CHECK(dupload(*ix, &ix->centers, ds->centers, csum));
    if (ds->n_centers == 16 && ds->packed) {
      // upload the reference pair-major layout, re-tile into vertical planes
      HS_CHECK(dalloc(*ix, &ix->vcodes, (size_t)vertical_words(n, K)));
      uint8_t* tmp = nullptr;
      HS_CUDA(cudaMalloc(&tmp, std::max<size_t>((size_t)ix->npairs * n, 1)));
      if (n) HS_CUDA(cudaMemcpy(tmp, ds->packed, (size_t)ix->npairs * n, cudaMemcpyHostToDevice));
      launch_to_vertical(tmp, n, K, ix->vcodes, 0);
      HS_CHECK(dalloc(*ix, &ix->hcodes, (size_t)hcodes_words(n, K)));
      launch_to_hcodes(tmp, n, K, ix->hcodes, 0);
      if (ds->n_active > 0) {  // point-major rows for the filtered stage 1's sparse part
        HS_CHECK(dalloc(*ix, &ix->pcodes, (size_t)pcodes_row(ix->npairs) * n));
        launch_to_pcodes(tmp, n, ix->npairs, ix->pcodes, 0);
      }
      HS_CUDA(cudaDeviceSynchronize());
      cudaFree(tmp);
    }
    ix->has_sq = ds->has_sq;
    if (ds->has_sq) {
      HS_CHECK(dupload(*ix, &ix->sq_lo, ds->sq_lo, ds->d_dense));
      HS_CHECK(dupload(*ix, &ix->sq_step, ds->sq_step, ds->d_dense));
      HS_CHECK(dupload(*ix, &ix->sq_codes, ds->sq_codes, (size_t)n * ds->d_dense));
    }
    ix->has_wh = ds->has_whitening;
    if (ds->has_whitening) {
      HS_CHECK(dupload(*ix, &ix->wh_mean, ds->wh_mean, ds->d_dense));
      // stored transposed: thread r of the whitening GEMV reads column r, so a
      // warp's loads of one k are consecutive (the row-major copy made every
      // load instruction touch 32 rows)
      const int64_t dd = ds->d_dense;
      std::vector<double> tr((size_t)dd * dd);
      for (int64_t r = 0; r < dd; ++r)
        for (int64_t c = 0; c < dd; ++c) tr[(size_t)c * dd + r] = ds->wh_inverse_t[(size_t)r * dd + c];
      HS_CHECK(dupload(*ix, &ix->wh_inv_t, tr.data(), (size_t)dd * dd));
    }
  }
  // raw dataset
  ix->has_ds = ds->has_dataset;
  if (ds->has_dataset) {
    if (ds->d_dense > 0) HS_CHECK(dupload(*ix, &ix->ds_dense, ds->ds_dense, (size_t)n * ds->d_dense));
    ix->ds_nnz = n ? ds->ds_indptr[n] - ds->ds_indptr[0] : 0;
    HS_CHECK(dupload(*ix, &ix->ds_indptr, ds->ds_indptr, n + 1));
    HS_CHECK(dupload(*ix, &ix->ds_indices, ds->ds_indices, ix->ds_nnz));
    HS_CHECK(dupload(*ix, &ix->ds_data, ds->ds_data, ix->ds_nnz));
  }
  HS_CUDA(cudaDeviceSynchronize());
  *out = ix.release();
  return HS_OK;
}

void hs_index_destroy(hs_index_t index) { hs::free_index(index); }

int hs_index_memory_bytes(hs_index_t index, int64_t* bytes) {
  if (!index || !bytes) HS_FAIL(HS_EINVAL, "null argument");
  *bytes = index->bytes;
  return HS_OK;
}

int hs_result_sizes(hs_index_t index, const hs_search_params* p, int64_t counts[3]) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  Sizes s;
  HS_CHECK(resolve_sizes(*index, p, &s));
  counts[0] = s.k1;
  counts[1] = s.k2;
  counts[2] = s.kh;
  return HS_OK;
}

int hs_search_batch(hs_index_t index, const hs_query_batch* queries,
                    const hs_search_params* params, int64_t* out_ids, double* out_scores,
                    double* stage_seconds) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  std::lock_guard<std::mutex> lock(index->mu);
  HS_CUDA(cudaSetDevice(index->device));
  Sizes sz;
  HS_CHECK(resolve_sizes(*index, params, &sz));
  if (!queries) HS_FAIL(HS_EINVAL, "null query batch");
  const int64_t nq = queries->nq;
  const int64_t total = nq * sz.kh;
  const size_t ids_bytes = ((sizeof(int64_t) * total + 255) & ~size_t(255));
  DevQueries dq;
  HS_CHECK(upload_queries(*index, queries, &dq, true, ids_bytes + sizeof(double) * total));
  int64_t* d_ids = reinterpret_cast<int64_t*>(dq.out);
  double* d_sc = reinterpret_cast<double*>(dq.out + ids_bytes);
  Timer tm(index, index->stream, index->timing ? TM_FULL : TM_STAGE);
  int rc = run_search(*index, dq.b, dq.nnz, dq.max_row, params, d_ids, d_sc, index->stream, &tm,
                      true);
  cudaError_t e = cudaSuccess;
  if (rc == HS_OK && total)
    e = cudaMemcpyAsync(dq.out_host, dq.out, ids_bytes + sizeof(double) * total,
                        cudaMemcpyDeviceToHost, index->stream);
  const cudaError_t es = cudaStreamSynchronize(index->stream);
  if (e == cudaSuccess) e = es;
  tm.finish(stage_seconds);
  if (rc != HS_OK) return rc;
  if (e != cudaSuccess) HS_FAIL(HS_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
  if (total) {
    std::memcpy(out_ids, dq.out_host, sizeof(int64_t) * total);
    std::memcpy(out_scores, dq.out_host + ids_bytes, sizeof(double) * total);
  }
  return HS_OK;
}

int hs_search_batch_dev(hs_index_t index, const hs_query_batch* queries,
                        const hs_search_params* params, int64_t* d_out_ids,
                        double* d_out_scores, void* stream) {
  if (!index || !queries) HS_FAIL(HS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(index->mu);
  HS_CUDA(cudaSetDevice(index->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
  int64_t nnz = 0;
  int max_row = 0;
  HS_CHECK(derive_hints(*index, queries, &nnz, &max_row, st));
  if (!index->timing_dev)
    return run_search(*index, *queries, nnz, max_row, params, d_out_ids, d_out_scores, st,
                      nullptr);
  Timer tm(index, st, TM_FULL);
  const int rc =
      run_search(*index, *queries, nnz, max_row, params, d_out_ids, d_out_scores, st, &tm);
  tm.finish(nullptr);
  return rc;
}

int hs_set_timing(hs_index_t index, int on) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  index->timing_dev = on != 0;
  index->timing = on != 0;
  return HS_OK;
}

int hs_index_launches(hs_index_t index, int64_t* launches) {
  if (!index || !launches) HS_FAIL(HS_EINVAL, "null argument");
  *launches = index->launches;
  return HS_OK;
}

int hs_adc_table(const float* centers, const int32_t* subdims, int32_t K, int32_t l,
                 const double* qw, int64_t nq, int64_t d, double* T) {
  if (K <= 0 || l <= 0 || nq < 0) HS_FAIL(HS_EINVAL, "bad shape");
  std::vector<int32_t> doff(K), coff(K);
  int64_t ds = 0, cs = 0;
  for (int k = 0; k < K; ++k) {
    doff[k] = (int32_t)ds;
    coff[k] = (int32_t)cs;
    ds += subdims[k];
    cs += (int64_t)subdims[k] * l;
  }
  if (ds != d) HS_FAIL(HS_EINVAL, "query dense dimension mismatch");
  DeviceIndex tmp;
  float* dc;
  int32_t *dsd, *ddo, *dco;
  double *dq, *dT;
  HS_CHECK(dupload(tmp, &dc, centers, cs));
  HS_CHECK(dupload(tmp, &dsd, subdims, K));
  HS_CHECK(dupload(tmp, &ddo, doff.data(), K));
  HS_CHECK(dupload(tmp, &dco, coff.data(), K));
  HS_CHECK(dupload(tmp, &dq, qw, nq * d));
  HS_CHECK(dalloc(tmp, &dT, nq * K * l));
  launch_adc_table(dc, dsd, ddo, dco, K, l, dq, nq, d, dT, 0);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaMemcpy(T, dT, sizeof(double) * nq * K * l, cudaMemcpyDeviceToHost));
  cudaFree(dc); cudaFree(dsd); cudaFree(ddo); cudaFree(dco); cudaFree(dq); cudaFree(dT);
  return HS_OK;
}

int hs_quantize_lut(const double* T, int64_t nq, int32_t K, int32_t l, uint8_t* table,
                    double* bias, double* scale, double* bias_total) {
  if (K < 0 || l <= 0 || nq < 0) HS_FAIL(HS_EINVAL, "bad shape");
  if (nq == 0) return HS_OK;
  DeviceIndex tmp;
  double *dT, *db, *ds, *dbt;
  uint8_t* dt;
  int* dbad;
  HS_CHECK(dupload(tmp, &dT, T, nq * K * l));
  HS_CHECK(dalloc(tmp, &dt, nq * K * l + 1));
  HS_CHECK(dalloc(tmp, &db, nq * K + 1));
  HS_CHECK(dalloc(tmp, &ds, nq));
  HS_CHECK(dalloc(tmp, &dbt, nq));
  HS_CHECK(dalloc(tmp, &dbad, nq));
  HS_CUDA(cudaMemset(dbad, 0, sizeof(int) * nq));
  launch_quantize(dT, nq, K, l, K, dt, db, ds, dbt, dbad, 0);
  HS_CUDA(cudaGetLastError());
  std::vector<int> hbad(nq);
  HS_CUDA(cudaMemcpy(hbad.data(), dbad, sizeof(int) * nq, cudaMemcpyDeviceToHost));
  if (K > 0 && l > 0) HS_CUDA(cudaMemcpy(table, dt, nq * K * l, cudaMemcpyDeviceToHost));
  if (K) HS_CUDA(cudaMemcpy(bias, db, sizeof(double) * nq * K, cudaMemcpyDeviceToHost));
  HS_CUDA(cudaMemcpy(scale, ds, sizeof(double) * nq, cudaMemcpyDeviceToHost));
  HS_CUDA(cudaMemcpy(bias_total, dbt, sizeof(double) * nq, cudaMemcpyDeviceToHost));
  cudaFree(dT); cudaFree(dt); cudaFree(db); cudaFree(ds); cudaFree(dbt); cudaFree(dbad);
  for (int64_t i = 0; i < nq; ++i)
    if (hbad[i]) HS_FAIL(HS_EINVAL, "lookup table contains non-finite values");
  return HS_OK;
}

int hs_lut16_scan(const uint8_t* packed, int64_t n, int32_t K, const uint8_t* qtable,
                  const double* bias_total, const double* scale, int64_t nq, int32_t* totals,
                  double* scores) {
  if (K <= 0 || n < 0 || nq < 0) HS_FAIL(HS_EINVAL, "bad shape");
  if (n == 0 || nq == 0) return HS_OK;
  // a dense-only temporary index view over the caller's codes
  hs_index_desc dsc;
  std::memset(&dsc, 0, sizeof(dsc));
  std::vector<int64_t> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::vector<int32_t> sub(K, 1);
  std::vector<float> cen((size_t)K * 16, 0.f);
  int64_t zero_ptr = 0;
  dsc.n = n;
  dsc.d_sparse = 0;
  dsc.d_dense = K;
  dsc.order = order.data();
  dsc.n_active = 0;
  dsc.post_ptr = &zero_ptr;
  dsc.n_subspaces = K;
  dsc.n_centers = 16;
  dsc.subdims = sub.data();
  dsc.centers = cen.data();
  dsc.packed = packed;
  dsc.sparse_weight = 1.0;
  dsc.dense_weight = 1.0;
  int dev = 0;
  HS_CUDA(cudaGetDevice(&dev));
  hs_index_t ix = nullptr;
  HS_CHECK(hs_index_create(&dsc, dev, &ix));
  std::unique_ptr<hs_index, void (*)(hs_index*)> guard(ix, [](hs_index* p) { hs::free_index(p); });
  const int Kp = ix->Kp;
  // padded LUTs [nq][Kp][16]
  std::vector<uint8_t> lp((size_t)nq * Kp * 16, 0);
  for (int64_t q = 0; q < nq; ++q)
    std::memcpy(&lp[(size_t)q * Kp * 16], qtable + (size_t)q * K * 16, (size_t)K * 16);
  DeviceIndex tmp;
  uint8_t* dl;
  double *dbt, *dsc2, *dout;
  uint32_t* dtot;
  int64_t* dptr;
  HS_CHECK(dupload(tmp, &dl, lp.data(), lp.size()));
  HS_CHECK(dupload(tmp, &dbt, bias_total, nq));
  HS_CHECK(dupload(tmp, &dsc2, scale, nq));
  HS_CHECK(dalloc(tmp, &dout, nq * n));
  HS_CHECK(dalloc(tmp, &dtot, nq * n));
  std::vector<int64_t> qp(nq + 1, 0);
  HS_CHECK(dupload(tmp, &dptr, qp.data(), nq + 1));
  QueryView qv;
  qv.nq = nq;
  qv.sp_indptr = dptr;
  Stage1Plan p = plan_stage1(*ix, nq, 1, 1, S1_DUMP);
  HS_CHECK(launch_stage1(*ix, qv, p, nullptr, nullptr, nullptr, nullptr, dl, dbt, dsc2, nullptr, nullptr,
                         dout, ix->stream, dtot, true));
  HS_CUDA(cudaStreamSynchronize(ix->stream));
  HS_CUDA(cudaMemcpy(scores, dout, sizeof(double) * nq * n, cudaMemcpyDeviceToHost));
  HS_CUDA(cudaMemcpy(totals, dtot, sizeof(uint32_t) * nq * n, cudaMemcpyDeviceToHost));
  cudaFree(dl); cudaFree(dbt); cudaFree(dsc2); cudaFree(dout); cudaFree(dtot); cudaFree(dptr);
  return HS_OK;
}

static int stage1_dump(hs_index_t index, const hs_query_batch* queries, double* out, bool raw_acc) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  std::lock_guard<std::mutex> lock(index->mu);
  HS_CUDA(cudaSetDevice(index->device));
  DevQueries dq;
  HS_CHECK(upload_queries(*index, queries, &dq, true));
  const int64_t nq = queries->nq, n = index->n, d = index->d_dense;
  if (nq == 0 || n == 0) return HS_OK;
  if (!raw_acc && d > 0 && index->K == 0) HS_FAIL(HS_EINVAL, "index has no dense PQ codes");
  if (!raw_acc && d > 0 && index->l != 16)
    HS_FAIL(HS_EUNSUPPORTED, "lut16_scan requires 16-center codes");
  DeviceIndex tmp;
  uint32_t *lb, *le;
  double *qv, *qd, *qw, *bt, *sc, *of, *dump;
  uint8_t* luts;
  int* bad;
  int32_t* lidx;
  HS_CHECK(dalloc(tmp, &lb, dq.nnz + 1));
  HS_CHECK(dalloc(tmp, &le, dq.nnz + 1));
  HS_CHECK(dalloc(tmp, &qv, dq.nnz + 1));
  HS_CHECK(dalloc(tmp, &lidx, dq.nnz + 1));
  HS_CHECK(dalloc(tmp, &qd, nq * d + 1));
  HS_CHECK(dalloc(tmp, &qw, nq * d + 1));
  HS_CHECK(dalloc(tmp, &luts, nq * index->Kp * 16 + 16));
  HS_CHECK(dalloc(tmp, &bt, nq));
  HS_CHECK(dalloc(tmp, &sc, nq));
  HS_CHECK(dalloc(tmp, &of, nq));
  HS_CHECK(dalloc(tmp, &bad, nq));
  HS_CHECK(dalloc(tmp, &dump, nq * n));
  HS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int) * nq, index->stream));
  QueryView qvw;
  qvw.nq = nq;
  qvw.sp_indptr = dq.b.sp_indptr;
  qvw.sp_dims = dq.b.sp_dims;
  qvw.sp_vals = dq.b.sp_vals;
  qvw.dense = dq.b.dense;
  launch_map_dims(*index, qvw, dq.nnz, !raw_acc, lb, le, qv, lidx, index->stream);
  if (!raw_acc && d > 0)
    launch_lut_build(*index, qvw.dense, nq, qd, qw, luts, bt, sc, of, bad, index->stream);
  Stage1Plan p = plan_stage1(*index, nq, 1, dq.max_row, S1_DUMP);
  p.sparse_only_acc = raw_acc;
  p.sparse = dq.nnz > 0;
  SparseBuckets sb;
  const bool use_buckets = dq.nnz > 0 && index->nnz_post > 0 && !getenv_flag("HSB200_NO_BUCKETS");
  if (use_buckets) {
    sb.nchunks = (int)ceil_div(n, stage1_chunk_points());
    sb.capq = bucket_capacity(*index);
    HS_CHECK(dalloc(tmp, &sb.mode, nq));
    HS_CHECK(dalloc(tmp, &sb.boff, nq * (sb.nchunks + 1)));
    HS_CHECK(dalloc(tmp, &sb.slots, nq * sb.capq));
    HS_CHECK(dalloc(tmp, &sb.vals, nq * sb.capq));
    launch_sparse_bucket(*index, qvw, lb, le, qv, sb, index->stream);
  }
  HS_CHECK(launch_stage1(*index, qvw, p, lb, le, qv, lidx, luts, bt, sc, of, nullptr, dump,
                         index->stream, nullptr, false, use_buckets ? &sb : nullptr));
  HS_CUDA(cudaStreamSynchronize(index->stream));
  std::vector<int> hbad(nq);
  HS_CUDA(cudaMemcpy(hbad.data(), bad, sizeof(int) * nq, cudaMemcpyDeviceToHost));
  HS_CUDA(cudaMemcpy(out, dump, sizeof(double) * nq * n, cudaMemcpyDeviceToHost));
  cudaFree(lb); cudaFree(le); cudaFree(qv); cudaFree(lidx); cudaFree(qd); cudaFree(qw); cudaFree(luts);
  cudaFree(bt); cudaFree(sc); cudaFree(of); cudaFree(bad); cudaFree(dump);
  if (use_buckets) {
    cudaFree(sb.mode); cudaFree(sb.boff); cudaFree(sb.slots); cudaFree(sb.vals);
  }
  for (int64_t i = 0; i < nq; ++i)
    if (hbad[i]) HS_FAIL(HS_EINVAL, "lookup table contains non-finite values");
  return HS_OK;
}

int hs_sparse_scan(hs_index_t index, const hs_query_batch* queries, double* acc) {
  return stage1_dump(index, queries, acc, true);
}


int hs_sparse_scan_into(hs_index_t index, const hs_query_batch* queries, double* acc) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  std::lock_guard<std::mutex> lock(index->mu);
  HS_CUDA(cudaSetDevice(index->device));
  DevQueries dq;
  HS_CHECK(upload_queries(*index, queries, &dq, true));
  const int64_t nq = queries->nq, n = index->n;
  if (nq == 0 || n == 0) return HS_OK;
  TmpBufs t;
  uint32_t *lb, *le;
  double *qv, *dacc;
  int32_t* lidx;
  HS_CHECK(t.alloc(&lb, dq.nnz + 1));
  HS_CHECK(t.alloc(&le, dq.nnz + 1));
  HS_CHECK(t.alloc(&qv, dq.nnz + 1));
  HS_CHECK(t.alloc(&lidx, dq.nnz + 1));
  HS_CHECK(t.upload(&dacc, acc, (size_t)(nq * n)));
  QueryView qvw;
  qvw.nq = nq;
  qvw.sp_indptr = dq.b.sp_indptr;
  qvw.sp_dims = dq.b.sp_dims;
  qvw.sp_vals = dq.b.sp_vals;
  qvw.dense = dq.b.dense;
  launch_map_dims(*index, qvw, dq.nnz, false, lb, le, qv, lidx, index->stream);
  launch_scan_into(*index, qvw, dq.max_row, lb, le, qv, dacc, index->stream);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaStreamSynchronize(index->stream));
  HS_CUDA(cudaMemcpy(acc, dacc, sizeof(double) * nq * n, cudaMemcpyDeviceToHost));
  return HS_OK;
}

static int sq_args(const uint8_t* codes, int64_t n, int32_t d, const float* lo, const float* step,
                   const int64_t* rows, int64_t m) {
  if (n < 0 || d < 0 || m < 0) HS_FAIL(HS_EINVAL, "bad shape");
  if (!lo || !step || (n * d > 0 && !codes)) HS_FAIL(HS_EINVAL, "null residual array");
  if (rows) {
    for (int64_t i = 0; i < m; ++i)
      if (rows[i] < 0 || rows[i] >= n) HS_FAIL(HS_EINVAL, "row index out of range");
  } else if (m != n) {
    HS_FAIL(HS_EINVAL, "rows == NULL requires m == n");
  }
  return HS_OK;
}

int hs_sq_decode(const uint8_t* codes, int64_t n, int32_t d, const float* lo, const float* step,
                 const int64_t* rows, int64_t m, double* out) {
  HS_CHECK(sq_args(codes, n, d, lo, step, rows, m));
  if (m == 0 || d == 0) return HS_OK;
  TmpBufs t;
  uint8_t* dc;
  float *dlo, *dst;
  int64_t* dr = nullptr;
  double* dout;
  HS_CHECK(t.upload(&dc, codes, (size_t)(n * d)));
  HS_CHECK(t.upload(&dlo, lo, (size_t)d));
  HS_CHECK(t.upload(&dst, step, (size_t)d));
  if (rows) HS_CHECK(t.upload(&dr, rows, (size_t)m));
  HS_CHECK(t.alloc(&dout, (size_t)(m * d)));
  launch_sq_decode(dc, d, dlo, dst, dr, m, dout, 0);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaMemcpy(out, dout, sizeof(double) * m * d, cudaMemcpyDeviceToHost));
  return HS_OK;
}

int hs_sq_residual_dot(const uint8_t* codes, int64_t n, int32_t d, const float* lo,
                       const float* step, const int64_t* rows, int64_t m, const double* q,
                       double* out) {
  HS_CHECK(sq_args(codes, n, d, lo, step, rows, m));
  if (m == 0) return HS_OK;
  if (d == 0) {
    for (int64_t i = 0; i < m; ++i) out[i] = 0.0;
    return HS_OK;
  }
  if (!q) HS_FAIL(HS_EINVAL, "null query");
  TmpBufs t;
  uint8_t* dc;
  float *dlo, *dst;
  int64_t* dr = nullptr;
  double *dq, *dout;
  HS_CHECK(t.upload(&dc, codes, (size_t)(n * d)));
  HS_CHECK(t.upload(&dlo, lo, (size_t)d));
  HS_CHECK(t.upload(&dst, step, (size_t)d));
  HS_CHECK(t.upload(&dq, q, (size_t)d));
  if (rows) HS_CHECK(t.upload(&dr, rows, (size_t)m));
  HS_CHECK(t.alloc(&dout, (size_t)m));
  launch_sq_dot(dc, d, dlo, dst, dr, m, dq, dout, 0);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaMemcpy(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return HS_OK;
}

int hs_stage1_scores(hs_index_t index, const hs_query_batch* queries, double* scores) {
  return stage1_dump(index, queries, scores, false);
}

int hs_select_topk(const double* scores, int64_t nq, int64_t n, int64_t k,
                   const int64_t* tie_ids, int64_t* out) {
  if (nq < 0 || n < 0) HS_FAIL(HS_EINVAL, "bad shape");
  k = std::min(k, n);
  if (k <= 0 || nq == 0) return HS_OK;
  if (tie_ids)
    for (int64_t i = 0; i < n; ++i)
      if (tie_ids[i] < 0 || tie_ids[i] >= (int64_t)0xFFFFFFFFLL)
        HS_FAIL(HS_EUNSUPPORTED, "tie ids must lie in [0, 2^32-1)");
  DeviceIndex tmp;
  double* ds;
  int64_t *dt = nullptr, *dout;
  Cand *c, *co;
  HS_CHECK(dupload(tmp, &ds, scores, nq * n));
  if (tie_ids) HS_CHECK(dupload(tmp, &dt, tie_ids, n));
  HS_CHECK(dalloc(tmp, &c, nq * n));
  HS_CHECK(dalloc(tmp, &co, nq * k));
  HS_CHECK(dalloc(tmp, &dout, nq * k));
  launch_scores_to_cands(ds, dt, nq, n, c, 0);
  HS_CHECK(launch_select_topk(c, nq, n, k, co, 0));
  launch_cands_to_positions(co, nq, k, dout, 0);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaMemcpy(out, dout, sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost));
  cudaFree(ds); if (dt) cudaFree(dt); cudaFree(c); cudaFree(co); cudaFree(dout);
  return HS_OK;
}

int hs_exact_topk(hs_index_t index, const hs_query_batch* queries, int32_t h, int64_t* out_ids,
                  double* out_scores) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  if (!index->has_ds) HS_FAIL(HS_EINVAL, "exact scoring requires the original dataset");
  if (h < 1) HS_FAIL(HS_EINVAL, "h must be >= 1");
  std::lock_guard<std::mutex> lock(index->mu);
  HS_CUDA(cudaSetDevice(index->device));
  DevQueries dq;
  HS_CHECK(upload_queries(*index, queries, &dq, true));
  const int64_t nq = queries->nq, n = index->n, d = index->d_dense;
  const int64_t kh = std::min<int64_t>(h, n);
  if (nq == 0 || kh == 0) return HS_OK;
  // chunk queries so the per-point candidate array stays below ~2 GB
  int64_t QB = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)(2.0e9 / (16.0 * n))));
  DeviceIndex tmp;
  Cand *all, *top;
  double* qd;
  int64_t* dids;
  double* dsc;
  HS_CHECK(dalloc(tmp, &all, QB * n));
  HS_CHECK(dalloc(tmp, &top, QB * kh));
  HS_CHECK(dalloc(tmp, &qd, nq * d + 1));
  HS_CHECK(dalloc(tmp, &dids, nq * kh));
  HS_CHECK(dalloc(tmp, &dsc, nq * kh));
  cudaStream_t st = index->stream;
  if (d > 0) launch_query_qd(dq.b.dense, nq, d, index->dense_weight, qd, st);
  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nqc = std::min(QB, nq - q0);
    QueryView qc;
    qc.nq = nqc;
    qc.sp_indptr = dq.b.sp_indptr + q0;
    qc.sp_dims = dq.b.sp_dims;
    qc.sp_vals = dq.b.sp_vals;
    launch_exact_scores(*index, qc, dq.max_row, qd + q0 * d, all, st);
    HS_CHECK(launch_select_topk(all, nqc, n, kh, top, st));
    launch_cands_to_ids(top, nqc * kh, index->id_offset, dids + q0 * kh, dsc + q0 * kh, st);
  }
  HS_CUDA(cudaStreamSynchronize(st));
  HS_CUDA(cudaMemcpy(out_ids, dids, sizeof(int64_t) * nq * kh, cudaMemcpyDeviceToHost));
  HS_CUDA(cudaMemcpy(out_scores, dsc, sizeof(double) * nq * kh, cudaMemcpyDeviceToHost));
  cudaFree(all); cudaFree(top); cudaFree(qd); cudaFree(dids); cudaFree(dsc);
  return HS_OK;
}

int hs_shard_merge_dev(const int64_t* d_ids, const double* d_scores, int64_t G, int64_t nq,
                       int64_t kh, int32_t h, int64_t* d_out_ids, double* d_out_scores,
                       void* stream) {
  if (G <= 0 || nq < 0 || kh < 0 || h < 1) HS_FAIL(HS_EINVAL, "bad shape");
  if (G * kh > 8192) HS_FAIL(HS_EUNSUPPORTED, "G*kh above 8192");
  launch_shard_merge(d_ids, d_scores, G, nq, kh, h, d_out_ids, d_out_scores,
                     static_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

// Raw dataset rows of local original ids (sampled checks of indices whose
// dataset lives only on the GPU).  indptr [m+1] relative offsets; pass
// indices/data NULL first to size them.  dense [m][d] as f32.
int hs_index_gather_rows(hs_index_t ix, const int64_t* ids, int64_t m, int64_t* indptr,
                         uint32_t* indices, float* data, float* dense) {
  if (!ix || (m > 0 && (!ids || !indptr))) HS_FAIL(HS_EINVAL, "null argument");
  if (!ix->has_ds) HS_FAIL(HS_EINVAL, "index holds no dataset");
  HS_CUDA(cudaSetDevice(ix->device));
  const int64_t d = ix->d_dense;
  indptr[0] = 0;
  std::vector<__half> hrow(d > 0 ? d : 1);
  for (int64_t i = 0; i < m; ++i) {
    if (ids[i] < 0 || ids[i] >= ix->n) HS_FAIL(HS_EINVAL, "row id out of range");
    int64_t be[2];
    HS_CUDA(cudaMemcpy(be, ix->ds_indptr + ids[i], sizeof(int64_t) * 2, cudaMemcpyDeviceToHost));
    const int64_t len = be[1] - be[0];
    indptr[i + 1] = indptr[i] + len;
    if (indices && len)
      HS_CUDA(cudaMemcpy(indices + indptr[i], ix->ds_indices + be[0], sizeof(uint32_t) * len,
                         cudaMemcpyDeviceToHost));
    if (data && len)
      HS_CUDA(cudaMemcpy(data + indptr[i], ix->ds_data + be[0], sizeof(float) * len,
                         cudaMemcpyDeviceToHost));
    if (dense && d > 0) {
      if (ix->ds_dense_h) {
        HS_CUDA(cudaMemcpy(hrow.data(), ix->ds_dense_h + ids[i] * d, sizeof(__half) * d,
                           cudaMemcpyDeviceToHost));
        for (int64_t j = 0; j < d; ++j) dense[i * d + j] = __half2float(hrow[j]);
      } else {
        HS_CUDA(cudaMemcpy(dense + i * d, ix->ds_dense + ids[i] * d, sizeof(float) * d,
                           cudaMemcpyDeviceToHost));
      }
    }
  }
  return HS_OK;
}

// Move a GPU build's products into a search index (the builder is consumed).
int hs_builder_finish(hs_builder_t bp, double sparse_weight, double dense_weight,
                      int64_t id_offset, hs_index_t* out) {
  std::unique_ptr<hs_builder, void (*)(hs_builder*)> b(bp, [](hs_builder* p) {
    if (!p) return;
    hs::builder_free(p);
    delete p;
  });
  if (!b || !out) HS_FAIL(HS_EINVAL, "null argument");
  *out = nullptr;
  if (!b->sparse_done) HS_FAIL(HS_EINVAL, "sparse part not built");
  if (b->d_dense > 0 && !b->dense_done) HS_FAIL(HS_EINVAL, "dense part not built");
  HS_CUDA(cudaSetDevice(b->device));
  HS_CUDA(cudaStreamSynchronize(b->st));
  std::unique_ptr<hs_index, void (*)(hs_index*)> ix(new hs_index(), [](hs_index* p) {
    hs::free_index(p);
  });
  const int64_t n = b->n;
  ix->device = b->device;
  ix->n = n;
  ix->d_sparse = b->d_sparse;
  ix->d_dense = b->d_dense;
  ix->id_offset = id_offset;
  ix->sparse_weight = sparse_weight;
  ix->dense_weight = dense_weight;
  HS_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
  HS_CUDA(cudaStreamCreateWithFlags(&ix->aux, cudaStreamNonBlocking));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_fork, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_join, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&ix->ev_done, cudaEventDisableTiming));
  auto take = [&](auto*& dst, auto*& src, int64_t bytes) {
    dst = src;
    src = nullptr;
    ix->bytes += bytes;
  };
  take(ix->order, b->order, 4 * n);
  ix->n_active = b->n_active;
  ix->nnz_post = b->nnz_post;
  take(ix->post_dims, b->post_dims, 4 * b->n_active);
  take(ix->post_ptr, b->post_ptr, 4 * (b->n_active + 1));
  take(ix->post, b->post, 8 * (b->nnz_post + 1));
  ix->post_wmin = b->wmin;
  ix->post_wmax = b->wmax;
  if (ix->nnz_post) HS_CHECK(build_skip_tables_dev(*ix));
  // residual = the raw rows' non-data entries (no separate CSR)
  ix->res_raw = 1;
  ix->res_eps = b->res_eps;
  ix->res_nnz = b->nnz - b->nnz_post;
  take(ix->ds_dmask, b->dmask, 4 * ceil_div(b->nnz, 32));
  if (b->d_dense > 0) {
    const int K = b->K;
    ix->K = K;
    ix->l = b->l;
    ix->Kp = (K + 1) & ~1;
    ix->npairs = (K + 1) / 2;
    std::vector<int32_t> doff(K), coff(K);
    int64_t dsum = 0, csum = 0;
    for (int k = 0; k < K; ++k) {
      doff[k] = (int32_t)dsum;
      coff[k] = (int32_t)csum;
      dsum += b->subdims[k];
      csum += (int64_t)b->subdims[k] * b->l;
      ix->max_width = std::max(ix->max_width, b->subdims[k]);
    }
    HS_CHECK(dupload(*ix, &ix->subdims, b->subdims.data(), K));
    HS_CHECK(dupload(*ix, &ix->dim_off, doff.data(), K));
    HS_CHECK(dupload(*ix, &ix->cen_off, coff.data(), K));
    HS_CHECK(dupload(*ix, &ix->centers, b->centers.data(), csum));
    HS_CHECK(dalloc(*ix, &ix->vcodes, (size_t)vertical_words(n, K)));
    launch_to_vertical(b->packed, n, K, ix->vcodes, b->st);
    HS_CHECK(dalloc(*ix, &ix->hcodes, (size_t)hcodes_words(n, K)));
    launch_to_hcodes(b->packed, n, K, ix->hcodes, b->st);
    HS_CUDA(cudaGetLastError());
    HS_CUDA(cudaStreamSynchronize(b->st));
    take(ix->pcodes, b->pcodes, pcodes_row(ix->npairs) * n);
    ix->has_sq = 1;
    HS_CHECK(dupload(*ix, &ix->sq_lo, b->sq_lo.data(), b->d_dense));
    HS_CHECK(dupload(*ix, &ix->sq_step, b->sq_step.data(), b->d_dense));
    take(ix->sq_codes, b->sq, n * b->d_dense);
    ix->has_wh = b->has_wh;
    if (b->has_wh) {
      const int64_t dd = b->d_dense;
      HS_CHECK(dupload(*ix, &ix->wh_mean, b->wh_mean.data(), dd));
      std::vector<double> tr((size_t)dd * dd);
      for (int64_t r = 0; r < dd; ++r)
        for (int64_t c = 0; c < dd; ++c) tr[(size_t)c * dd + r] = b->wh_inv_t[(size_t)r * dd + c];
      HS_CHECK(dupload(*ix, &ix->wh_inv_t, tr.data(), (size_t)dd * dd));
    }
  }
  ix->has_ds = 1;
  ix->ds_nnz = b->nnz;
  take(ix->ds_indptr, b->indptr, 8 * (n + 1));
  take(ix->ds_indices, b->indices, 4 * b->nnz);
  take(ix->ds_data, b->data, 4 * b->nnz);
  if (b->d_dense > 0) {
    if (b->dense_fp16) take(ix->ds_dense_h, b->dense_h, 2 * n * b->d_dense);
    else take(ix->ds_dense, b->dense, 4 * n * b->d_dense);
  }
  HS_CUDA(cudaDeviceSynchronize());
  *out = ix.release();
  return HS_OK;
}

int hs_last_kernel_times(hs_index_t index, double* ms, int32_t max_entries, int32_t* n_entries,
                         char* names, int32_t names_cap) {
  if (!index) HS_FAIL(HS_EINVAL, "null index");
  const int32_t n = (int32_t)std::min<size_t>(index->tms.size(), (size_t)max_entries);
  std::string joined;
  for (int32_t i = 0; i < n; ++i) {
    ms[i] = index->tms[i];
    if (i) joined += ";";
    joined += index->tnames[i];
  }
  *n_entries = n;
  if (names && names_cap > 0) {
    std::strncpy(names, joined.c_str(), names_cap - 1);
    names[names_cap - 1] = 0;
  }
  return HS_OK;
}

}  // extern "C"
