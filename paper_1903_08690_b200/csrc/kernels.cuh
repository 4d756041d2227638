// kernels.cuh — device index layout and the kernel launchers shared by the
// translation units of libhsb200.so.
#pragma once

#include <mutex>
#include <string>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"

namespace hs {

// Immutable device copy of one hybrid index (the C-ABI handle).
struct DeviceIndex {
  int device = 0;
  int64_t n = 0, d_sparse = 0, d_dense = 0, id_offset = 0;
  double sparse_weight = 1.0, dense_weight = 1.0;

  uint32_t* order = nullptr;  // [n] slot -> original id (u32)

  // pruned scan index: interleaved (id, w-bits) postings, CSR over active dims
  int64_t n_active = 0, nnz_post = 0;
  uint32_t* post_dims = nullptr;  // [n_active]
  uint32_t* post_ptr = nullptr;   // [n_active+1] (nnz_post < 2^32)
  uint2* post = nullptr;          // [nnz_post] {id, __float_as_uint(w)}
  double post_wmin = 0.0, post_wmax = 0.0;  // range of the posting weights
  // chunk skip tables of long lists: skip_row[list] = row index or -1;
  // row r holds, for every 4096-slot chunk c, the list-relative position of
  // the first posting with id >= 4096*c (nchunks+1 entries)
  int32_t* skip_row = nullptr;    // [n_active]
  uint32_t* skip = nullptr;       // [n_long][nchunks+1]
  int64_t n_long = 0;

  // forward sparse residual (layout order)
  int64_t res_nnz = 0;
  int64_t* res_indptr = nullptr;
  uint32_t* res_indices = nullptr;
  float* res_data = nullptr;

  // dense PQ part
  int K = 0, l = 0, Kp = 0, npairs = 0, max_width = 0;
  int32_t* subdims = nullptr;  // [K]
  int32_t* dim_off = nullptr;  // [K] first dense dim of subspace k
  int32_t* cen_off = nullptr;  // [K] offset of centers[k] in `centers`
  float* centers = nullptr;
  uint32_t* vcodes = nullptr;  // blocked [n/4096][K][512] vertical nibble planes (lut16_stream.cu, stage1.cu)
  uint32_t* hcodes = nullptr;  // blocked [n/128][ceil(K/8)][128] 8-code words (lut16_tc.cu)
  uint8_t* pcodes = nullptr;   // [n][pcodes_row] point-major packed codes (fuse.cu)
  int has_sq = 0;
  float *sq_lo = nullptr, *sq_step = nullptr;
  uint8_t* sq_codes = nullptr;  // [n][d_dense]
  int has_wh = 0;
  double *wh_mean = nullptr, *wh_inv_t = nullptr;  // wh_inv_t stored transposed ([col][row])

  // raw dataset (original order) for exact rerank / ground truth
  int has_ds = 0;
  float* ds_dense = nullptr;
  __half* ds_dense_h = nullptr;  // fp16-stored dense part (cfg 5), instead of ds_dense
  // GPU-built indices keep no separate residual CSR: the residual of a raw
  // row is its entries whose data-part flag (bit e of ds_dmask) is clear and
  // whose magnitude is >= res_eps (prune_split, sparse.py:83-103), read in
  // the row's column order like the residual CSR (pipeline.py:137-138)
  int res_raw = 0;
  uint32_t* ds_dmask = nullptr;  // [ceil(ds_nnz / 32)]
  double res_eps = 0.0;
  int64_t* ds_indptr = nullptr;
  uint32_t* ds_indices = nullptr;
  float* ds_data = nullptr;
  int64_t ds_nnz = 0;

  int64_t bytes = 0;
  cudaStream_t stream = nullptr;
  // second stream + fork/join events: the sparse bucketing of a query chunk
  // runs concurrently with its LUT build and sample pass
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // recorded at the end of every search: the next search (any stream) waits
  // on it before reusing the scratch arena
  cudaEvent_t ev_done = nullptr;
  std::mutex mu;

  // scratch arena (grown on demand, owned by the handle)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  double scratch_budget = 0.0;  // bytes the per-chunk stage-1 buffers may take (set on first search)
  // host entry point I/O staging (grown on demand): device query/result
  // buffers and a pinned host mirror, so a call does no cudaMalloc/cudaFree
  void* io_dev = nullptr;
  size_t io_dev_bytes = 0;
  void* io_host = nullptr;
  size_t io_host_bytes = 0;

  // per-kernel timing of the last batch (CUDA events; bench roofline)
  bool timing = false;      // host entry point: per-kernel events (else stage events only)
  bool timing_dev = false;  // _dev entry point (adds a sync)
  std::vector<cudaEvent_t> evpool;  // reused timing events
  int64_t launches = 0;
  std::vector<std::string> tnames;
  std::vector<double> tms;
};

// ---- GPU index build (devbuild.cu sparse part, build.cu dense part) ----
// A dataset resident on one GPU (generated there or uploaded) and the index
// products built from it; hs_builder_finish moves them into a DeviceIndex.
struct Builder {
  int device = 0;
  cudaStream_t st = nullptr;
  int64_t n = 0, d_sparse = 0, d_dense = 0, nnz = 0;
  int dense_fp16 = 0;
  // dataset, original row order (CSR columns ascending per row)
  int64_t* indptr = nullptr;  // [n+1]
  uint32_t* indices = nullptr;
  float* data = nullptr;
  float* dense = nullptr;     // [n][d] f32, or
  __half* dense_h = nullptr;  // [n][d] fp16
  // sparse products (hs_builder_sparse)
  int sparse_done = 0;
  uint32_t* dmask = nullptr;  // [ceil(nnz/32)] data-part flag per entry
  double res_eps = 0.0;
  uint32_t* order = nullptr;  // [n] layout slot -> row
  int64_t n_active = 0, nnz_post = 0, n_head = 0;
  uint32_t* post_dims = nullptr;  // [n_active]
  uint32_t* post_ptr = nullptr;   // [n_active+1]
  uint2* post = nullptr;          // [nnz_post] {slot, w bits}
  float wmin = 0.f, wmax = 0.f;
  uint32_t* head_dims = nullptr;  // [n_head] dims whose count exceeds top_t
  uint32_t* head_thr = nullptr;   // [n_head] |v| bit pattern of the top_t-th largest
  // dense products (hs_builder_dense_encode)
  int dense_done = 0;
  int K = 0, l = 0;
  std::vector<int32_t> subdims;
  std::vector<float> centers;
  uint8_t* packed = nullptr;  // [npairs][n] pair-major (reference layout)
  uint8_t* pcodes = nullptr;  // [n][pcodes_row] point-major
  uint8_t* sq = nullptr;      // [n][d]
  std::vector<float> sq_lo, sq_step;
  int has_wh = 0;
  std::vector<double> wh_mean, wh_inv_t;
  // phase timings (seconds)
  std::vector<std::string> tnames;
  std::vector<double> tsec;
  void* tmp = nullptr;  // cub temp storage, grown on demand
  size_t tmp_bytes = 0;
  int64_t bytes = 0;
};
int builder_tmp(Builder& b, size_t bytes);
void builder_phase(Builder& b, const char* name, double sec);
void builder_free(Builder* b);
// f64 rows of the dense part (gathered by `rows`, or order[slot0 + i] when
// rows == nullptr), optionally whitened: out[i] = (x - mean) @ fwd^T
int launch_dense_rows(const Builder& b, const uint32_t* rows_u32, const int64_t* rows_i64,
                      int64_t slot0, int64_t m, const double* mean, const double* fwd,
                      double* out, cudaStream_t st);
int build_skip_tables_dev(DeviceIndex& ix);

// ---- per-batch device views of a query chunk ----
struct QueryView {
  int64_t nq = 0;
  const int64_t* sp_indptr = nullptr;  // device [nq+1], absolute offsets
  const uint32_t* sp_dims = nullptr;
  const float* sp_vals = nullptr;
  const float* dense = nullptr;  // [nq][d]
};

// lut.cu
void launch_lut_build(const DeviceIndex& ix, const float* qdense, int64_t nq, double* qd_out,
                      double* qw_out, uint8_t* luts, double* bias_total, double* scale,
                      double* offset, int* bad, cudaStream_t st);
void launch_adc_table(const float* centers, const int32_t* subdims, const int32_t* dim_off,
                      const int32_t* cen_off, int K, int l, const double* qw, int64_t nq,
                      int64_t d, double* T, cudaStream_t st);
void launch_quantize(const double* T, int64_t nq, int K, int l, int Kp, uint8_t* table,
                     double* bias, double* scale, double* bias_total, int* bad,
                     cudaStream_t st);

// stage1.cu
enum Stage1Mode { S1_SELECT = 0, S1_EMIT_ALL = 1, S1_DUMP = 2 };
struct Stage1Plan {
  int mode = S1_SELECT;
  int ntiles = 1;
  int64_t tile_pts = 0;   // multiple of the chunk size
  int k = 0;              // per-tile keep (SELECT)
  int cap = 0;            // candidate buffer entries (pow2, >= k + chunk)
  int64_t out_per_tile = 0;
  int max_qnnz = 0;
  bool use_dense = true;  // DUMP: include the dense part
  bool sparse_only_acc = false;  // DUMP: raw accumulator (no weights, no dense)
  bool sparse = true;     // the batch has sparse nonzeros to stream
  int64_t n_limit = -1;   // scan points [0, n_limit) only (< 0: all)
  const int* qmask = nullptr;  // if set, only queries with qmask[q] != 0 run
};
// per-query postings bucketed by 4096-slot chunk (stable: ascending dim then
// slot inside a bucket) with exact f64 products; mode[q] = 1 when query q
// uses the buckets, 0 when it streams its lists in stage 1
struct SparseBuckets {
  int* mode = nullptr;       // [nq]
  uint32_t* boff = nullptr;  // [nq][nchunks+1]
  uint32_t* slots = nullptr; // [nq][capq]
  double* vals = nullptr;    // [nq][capq]
  int64_t capq = 0;
  int nchunks = 0;
};
int64_t bucket_capacity(const DeviceIndex& ix);
int build_skip_tables(DeviceIndex& ix, const int64_t* host_ptr);
void launch_sparse_bucket(const DeviceIndex& ix, const QueryView& q, const uint32_t* lbeg,
                          const uint32_t* lend, const double* qv, const SparseBuckets& sb,
                          cudaStream_t st);
int stage1_chunk_points();
Stage1Plan plan_stage1(const DeviceIndex& ix, int64_t nq, int64_t k, int max_qnnz, int mode,
                       int64_t n_limit = -1);
size_t stage1_smem_bytes(const DeviceIndex& ix, const Stage1Plan& p, bool ws);
void launch_map_dims(const DeviceIndex& ix, const QueryView& q, int64_t nnz, bool use_weight,
                     uint32_t* lbeg, uint32_t* lend, double* qv, int32_t* lidx,
                     cudaStream_t st);
void launch_scan_into(const DeviceIndex& ix, const QueryView& q, int max_row_nnz,
                      const uint32_t* lbeg, const uint32_t* lend, const double* qv, double* acc,
                      cudaStream_t st);
int launch_stage1(const DeviceIndex& ix, const QueryView& q, const Stage1Plan& p,
                  const uint32_t* lbeg, const uint32_t* lend, const double* qv,
                  const int32_t* lidx, const uint8_t* luts, const double* bias_total, const double* scale,
                  const double* offset, Cand* out, double* dump, cudaStream_t st,
                  uint32_t* dump_tot = nullptr, bool raw_dense = false,
                  const SparseBuckets* sb = nullptr, const uint16_t* tot16 = nullptr,
                  int64_t tot_ld = 0);

// lut16_stream.cu (HBM-bound LUT16 scan for small batches; owns the vertical code layout)
int64_t vertical_words(int64_t n, int K);
void launch_to_vertical(const uint8_t* packed, int64_t n, int K, uint32_t* v, cudaStream_t st);
bool lut16_stream_supported(const DeviceIndex& ix);
// filter-mode list layout: one segment per CTA, each a contiguous range of
// 4096-point code blocks; frac = the largest share of the points in one
void lut16_stream_layout(const DeviceIndex& ix, int64_t* nseg, double* frac);
// u16 totals [nq][ld] of points [0, n_limit) (n_limit < 0: all)
int launch_lut16_stream_totals(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                               uint16_t* tot, int64_t ld, cudaStream_t st, int64_t n_limit = -1);
// same contract as launch_lut16_filter, segments of lut16_stream_layout
int launch_lut16_stream_filter(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                               const uint32_t* tlim, uint2* list, uint32_t* cnt, int64_t cap,
                               cudaStream_t st);

// lut16_tc.cu (tensor-core batched LUT16 totals)
bool lut16_tc_supported(const DeviceIndex& ix);
int64_t lut16_tc_ld(int64_t n);
int64_t lut16_tc_group(const DeviceIndex& ix);  // queries per tensor-core group
// filter-mode list layout for a batch of nq queries: segments per query and
// the largest fraction of a query's points one segment (CTA) covers
void lut16_filter_layout(const DeviceIndex& ix, int64_t nq, int64_t* nseg, double* frac);
void launch_to_hcodes(const uint8_t* packed, int64_t n, int K, uint32_t* h, cudaStream_t st);
int64_t hcodes_words(int64_t n, int K);
// totals mode: u16 totals [nq][ld] of points [0, n_limit) (n_limit < 0: all)
int launch_lut16_tc(const DeviceIndex& ix, const uint8_t* luts, int64_t nq, uint16_t* tot,
                    int64_t ld, cudaStream_t st, int64_t n_limit = -1);
// filter mode: (point, total) pairs with total >= tlim[q], appended to CTA-
// private segments list[q][s][0..cap) (s < kNumSMs) in no particular order;
// cnt[q][s] = passes of segment s (> cap: overflow, the segment holds an
// arbitrary subset); s < nseg of lut16_filter_layout
int launch_lut16_filter(const DeviceIndex& ix, const uint8_t* luts, int64_t nq,
                        const uint32_t* tlim, uint2* list, uint32_t* cnt, int64_t cap,
                        cudaStream_t st);

// fuse.cu (threshold-filtered stage 1 on the tensor-core path)
int64_t pcodes_row(int npairs);
void launch_to_pcodes(const uint8_t* packed, int64_t n, int npairs, uint8_t* pc, cudaStream_t st);
void launch_tlim(const Cand* cand_s, int64_t nq, int k, const double* btot, const double* scl,
                 const double* off, uint32_t* tlim, double* T, cudaStream_t st);
void launch_sample_tlim(const uint16_t* tot_s, int64_t ld, int64_t m, int64_t nq, int k,
                        const int64_t* qptr, const double* qv, double wmin, double wmax,
                        const double* btot, const double* scl, const double* off,
                        uint32_t* tlim, double* T, cudaStream_t st);
int launch_fuse_cands(const DeviceIndex& ix, int64_t nq, const uint8_t* luts, const double* btot,
                      const double* scl, const double* off, const uint2* list,
                      const uint32_t* cnt, int64_t cap, int nseg, const SparseBuckets* sb,
                      uint32_t* bitmap, Cand* out, int64_t M, uint32_t* out_cnt, int* fallback,
                      const double* T, cudaStream_t st);

// select.cu
// best k of each query's row in[q][0..m) (or [0..counts[q]) when counts is
// given), sorted by (score desc, tie asc); rows with qmask[q] == 0 are skipped
int launch_select_topk(const Cand* in, int64_t nq, int64_t m, int64_t k, Cand* out,
                       cudaStream_t st, const uint32_t* counts = nullptr,
                       const int* qmask = nullptr);
void launch_scores_to_cands(const double* scores, const int64_t* tie_ids, int64_t nq,
                            int64_t n, Cand* out, cudaStream_t st);
void launch_cands_to_positions(const Cand* c, int64_t nq, int64_t k, int64_t* out,
                               cudaStream_t st);
void launch_shard_merge(const int64_t* ids, const double* scores, int64_t G, int64_t nq,
                        int64_t kh, int h, int64_t* out_ids, double* out_scores,
                        cudaStream_t st);

// rerank.cu
void launch_stage2(const DeviceIndex& ix, const Cand* cand1, int64_t nq, int k1, int k2,
                   const double* qw, Cand* cand2, cudaStream_t st);
void launch_stage3(const DeviceIndex& ix, const QueryView& q, const Cand* cand2, int64_t nq,
                   int k2, int kh, int exact, int max_qnnz, const double* qd, int64_t* out_ids,
                   double* out_scores, cudaStream_t st);
void launch_query_qd(const float* qdense, int64_t nq, int64_t d, double w, double* qd,
                     cudaStream_t st);
void launch_exact_scores(const DeviceIndex& ix, const QueryView& q, int max_qnnz,
                         const double* qd, Cand* out, cudaStream_t st);
void launch_cands_to_ids(const Cand* c, int64_t total, int64_t id_offset, int64_t* ids,
                         double* scores, cudaStream_t st);
void launch_sq_decode(const uint8_t* codes, int64_t d, const float* lo, const float* step,
                      const int64_t* rows, int64_t m, double* out, cudaStream_t st);
void launch_sq_dot(const uint8_t* codes, int64_t d, const float* lo, const float* step,
                   const int64_t* rows, int64_t m, const double* q, double* out, cudaStream_t st);

}  // namespace hs
