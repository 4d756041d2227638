/*
 * hsb200.h — C ABI of the B200-native hybrid sparse+dense inner-product search
 * (the hot path of arXiv 1903.08690's `hybridsearch` reference package).
 *
 * Plain pointers and sizes only: no torch / Python types cross this boundary.
 * Every entry point returns an hs_status; hs_last_error() gives the message of
 * the calling thread's last failure.  Host-pointer entry points copy inputs to
 * the device inside the call (borrowed for the duration of the call) and copy
 * results back into caller-allocated host buffers.  `_dev` entry points take
 * device pointers and a cudaStream_t (as void*), and enqueue without syncing.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/hybridsearch):
 *   hs_index_create      <- the HybridIndex a search consumes      pipeline.py:92-116
 *                           (InvertedIndex sparse.py:172-200, PQCodes dense.py:183-209,
 *                            Codebooks dense.py:25-54, ScalarQuantResidual dense.py:361-378,
 *                            WhiteningTransform dense.py:320-330, HybridDataset data.py:118-162)
 *   hs_search_batch      <- search_batch / search_topk             pipeline.py:282-300, 226-279
 *   hs_search_batch_dev  <- same, device-resident queries/results  (no reference counterpart)
 *   hs_adc_table         <- adc_table                              dense.py:212-220
 *   hs_quantize_lut      <- quantize_lut + QuantizedLUT.bias_total dense.py:248-260, 243-245
 *   hs_lut16_scan        <- lut16_scan / lut16_scan_reference      dense.py:297-317, 263-281
 *   hs_sparse_scan       <- sparse_scan (Accumulator scores)       sparse.py:268-284
 *   hs_sparse_scan_into  <- sparse_scan into a non-zero Accumulator sparse.py:277-282
 *   hs_sq_decode         <- ScalarQuantResidual.decode, sq_decode dense.py:369-371, 393-394
 *   hs_sq_residual_dot   <- ScalarQuantResidual.dot                dense.py:373-375
 *   hs_stage1_scores     <- _stage1_scores                         pipeline.py:192-203
 *   hs_select_topk       <- select_topk                            pipeline.py:165-189
 *   hs_exact_topk        <- brute_force_topk (_exact_scores)       harness.py:25-35, pipeline.py:313-322
 *   hs_shard_merge_dev   <- (new) top-h merge of per-shard results; no reference counterpart
 *   hs_dense_encode      <- build_index's dense part: pq_encode(...)[order] + pack_codes +
 *                           sq_encode(residual)   pipeline.py:142-157, dense.py:138-170, 381-390
 *   hs_builder_*         <- build_index on the GPU (+ the BASELINE data generator),
 *                           see the section at the end of this header
 */
#ifndef HSB200_H
#define HSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HS_OK = 0,
  HS_EINVAL = 1,       /* -> ValueError   (pipeline.py:235-245, dense.py:251-252, dense.py:304-305) */
  HS_ENOMEM = 2,       /* -> MemoryError */
  HS_ECUDA = 3,        /* -> RuntimeError */
  HS_ENCCL = 4,        /* -> RuntimeError */
  HS_EUNSUPPORTED = 5  /* -> ValueError (e.g. 256-center codes in lut16_scan, dense.py:304-305) */
} hs_status;

typedef struct hs_index* hs_index_t;

/* Borrowed host arrays describing one immutable hybrid index.  All sparse
 * dimension ids are uint32 (d_sparse < 2^32); row pointers are int64. */
typedef struct {
  int64_t n;             /* points */
  int64_t d_sparse;      /* sparse dimensionality */
  int64_t d_dense;       /* dense dimensionality (0 = no dense part) */
  const int64_t* order;  /* [n] layout slot -> original id (pipeline.py:102) */

  /* pruned scan index: posting lists of the active dims, ascending dims,
   * ids strictly ascending within a list (sparse.py:219-235) */
  int64_t n_active;
  const uint32_t* post_dims;  /* [n_active] */
  const int64_t* post_ptr;    /* [n_active+1] */
  const uint32_t* post_ids;   /* [nnz] layout slots */
  const float* post_w;        /* [nnz] */

  /* forward sparse residual, rows in layout order (pipeline.py:137-138) */
  const int64_t* res_indptr;  /* [n+1] or NULL when empty */
  const uint32_t* res_indices;
  const float* res_data;

  /* dense PQ part (present iff d_dense > 0) */
  int32_t n_subspaces;        /* K */
  int32_t n_centers;          /* l: 16 for the LUT16 scan, 256 is rejected at search */
  const int32_t* subdims;     /* [K] widths, contiguous subspaces (dense.py:57-62) */
  const float* centers;       /* concatenation over k of centers[k] (l x subdims[k]) row-major */
  const uint8_t* packed;      /* [(K+1)/2][n] pair-major 4-bit codes (dense.py:156-170) */
  int32_t has_sq;             /* scalar-quant residual present (dense.py:361-378) */
  const float* sq_lo;         /* [d_dense] */
  const float* sq_step;       /* [d_dense] */
  const uint8_t* sq_codes;    /* [n][d_dense] layout order */
  int32_t has_whitening;      /* query-side whitening (dense.py:351-357) */
  const double* wh_mean;      /* [d_dense] */
  const double* wh_inverse_t; /* [d_dense][d_dense] */

  /* raw dataset for exact rerank / ground truth (optional; original id order) */
  int32_t has_dataset;
  const float* ds_dense;      /* [n][d_dense] */
  const int64_t* ds_indptr;   /* [n+1] */
  const uint32_t* ds_indices;
  const float* ds_data;

  /* query-time weights from HybridIndexConfig (pipeline.py:51-52) */
  double sparse_weight;
  double dense_weight;
  /* added to every returned original id (multi-GPU id-range shards) */
  int64_t id_offset;
} hs_index_desc;

/* A batch of queries: CSR sparse parts (ascending dims per row) + dense rows. */
typedef struct {
  int64_t nq;
  const int64_t* sp_indptr;   /* [nq+1] */
  const uint32_t* sp_dims;    /* [nnz] */
  const float* sp_vals;       /* [nnz] */
  const float* dense;         /* [nq][d_dense] (may be NULL when d_dense == 0) */
  /* optional hints for the _dev entry points (<= 0: derived with a D2H copy) */
  int64_t nnz;                /* sp_indptr[nq] - sp_indptr[0] */
  int32_t max_row_nnz;        /* max over rows of the row length */
} hs_query_batch;

/* Per-call search knobs; resolved by the caller from HybridIndexConfig and
 * the call overrides (pipeline.py:233-245). */
typedef struct {
  int32_t h;
  double overfetch;           /* alpha: k1 = min(n, ceil(alpha*h)) */
  double retain;              /* beta:  k2 = min(k1, ceil(beta*h)) */
  int32_t exact_final_rerank;
} hs_search_params;

const char* hs_last_error(void);
const char* hs_version(void);

/* ---- index lifetime ---- */
int hs_index_create(const hs_index_desc* desc, int device, hs_index_t* out);
void hs_index_destroy(hs_index_t index);
int hs_index_memory_bytes(hs_index_t index, int64_t* bytes);

/* Result slots per query = kh = min(h, k2); counts[3] = {k1, k2, kh}.
 * stage_seconds[3] receives device time per stage summed over the batch. */
int hs_result_sizes(hs_index_t index, const hs_search_params* p, int64_t counts[3]);

/* ---- the hot path ---- */
int hs_search_batch(hs_index_t index, const hs_query_batch* queries,
                    const hs_search_params* params, int64_t* out_ids,
                    double* out_scores, double* stage_seconds);

/* Device-resident variant: every pointer in `queries` and the outputs are
 * device pointers; enqueued on `stream` (cudaStream_t; NULL = the legacy
 * default stream), no host sync.  sp_indptr[0] must be 0. */
int hs_search_batch_dev(hs_index_t index, const hs_query_batch* queries,
                        const hs_search_params* params, int64_t* d_out_ids,
                        double* d_out_scores, void* stream);

/* ---- unit entry points (parity tests; each mirrors one reference function) ---- */
/* T[q][k][c] = <centers[k][c], qw[q][slice k]> in f64. */
int hs_adc_table(const float* centers, const int32_t* subdims, int32_t K, int32_t l,
                 const double* qw, int64_t nq, int64_t d, double* T);
/* u8 table, per-row bias, shared scale, numpy-pairwise bias_total. */
int hs_quantize_lut(const double* T, int64_t nq, int32_t K, int32_t l, uint8_t* table,
                    double* bias, double* scale, double* bias_total);
/* integer totals and bias_total + scale*total for nq LUTs over n points. */
int hs_lut16_scan(const uint8_t* packed, int64_t n, int32_t K, const uint8_t* qtable,
                  const double* bias_total, const double* scale, int64_t nq,
                  int32_t* totals, double* scores);
/* f64 accumulator in layout order, weights NOT applied (sparse.py:268-284). */
int hs_sparse_scan(hs_index_t index, const hs_query_batch* queries, double* acc);
/* sparse_scan into a non-zero accumulator: acc [nq][n] holds the initial
 * scores and receives acc + q_j*w added one query dim at a time in ascending
 * dim order, each addition rounded (sparse.py:277-282, Accumulator sparse.py:239-258). */
int hs_sparse_scan_into(hs_index_t index, const hs_query_batch* queries, double* acc);
/* ScalarQuantResidual.decode(rows) / sq_decode (dense.py:369-371, 393-394):
 * out [m][d] = lo + step*(codes[rows] + 0.5) in f64; rows NULL = all n (m == n). */
int hs_sq_decode(const uint8_t* codes, int64_t n, int32_t d, const float* lo,
                 const float* step, const int64_t* rows, int64_t m, double* out);
/* ScalarQuantResidual.dot(rows, q) (dense.py:373-375): out [m] = decode(rows) @ q. */
int hs_sq_residual_dot(const uint8_t* codes, int64_t n, int32_t d, const float* lo,
                       const float* step, const int64_t* rows, int64_t m, const double* q,
                       double* out);
/* stage-1 scores in layout order with the index's weights (pipeline.py:192-203). */
int hs_stage1_scores(hs_index_t index, const hs_query_batch* queries, double* scores);
/* top-k positions per row by (score desc, tie asc); tie_ids NULL = positions. */
int hs_select_topk(const double* scores, int64_t nq, int64_t n, int64_t k,
                   const int64_t* tie_ids, int64_t* out);
/* exact top-h (brute force over the raw dataset), ids original. */
int hs_exact_topk(hs_index_t index, const hs_query_batch* queries, int32_t h,
                  int64_t* out_ids, double* out_scores);

/* Merge G gathered per-shard results (ids/scores [G][nq][kh], device) into
 * the top-h per query by (score desc, id asc). */
int hs_shard_merge_dev(const int64_t* d_ids, const double* d_scores, int64_t G,
                       int64_t nq, int64_t kh, int32_t h, int64_t* d_out_ids,
                       double* d_out_scores, void* stream);

/* Per-kernel CUDA-event timing of search calls (on by default for the host
 * entry point; enables it for the _dev entry point too, which then syncs). */
int hs_set_timing(hs_index_t index, int on);
/* Cumulative number of kernels this index's search calls have launched. */
int hs_index_launches(hs_index_t index, int64_t* launches);

/* Timing of the last search on this index: per-kernel CUDA-event averages
 * (used by bench.py for the roofline). names joined by ';'. */
int hs_last_kernel_times(hs_index_t index, double* ms, int32_t max_entries,
                         int32_t* n_entries, char* names, int32_t names_cap);

/* ---- index build (dense slice) ---- */
/* Host pointers.  vec [n][d] f64 in original id order (whitened when the
 * config whitens), order [n] layout slot -> id, K subspaces of width 1 or 2,
 * centers = concatenation over k of 16 x subdims[k] f32.  Outputs in layout
 * order: packed [(K+1)/2][n] pair-major 4-bit codes; optional (NULL = skip)
 * sq_lo/sq_step [d] and sq_codes [n][d].  Bit-identical to the host build.
 * seconds (optional) receives the device time of the two kernels. */
int hs_dense_encode(const double* vec, int64_t n, int64_t d, const int64_t* order,
                    int32_t K, const int64_t* subdims, const float* centers, int32_t l,
                    uint8_t* packed, float* sq_lo, float* sq_step, uint8_t* sq_codes,
                    int device, double* seconds);

/* ---- GPU index build and the on-device data generator ----
 * A builder holds one dataset resident on a GPU — generated there
 * (hs_builder_generate) or uploaded (hs_builder_upload) — and builds the
 * index products in place, following build_index (pipeline.py:119-162):
 *   hs_builder_sparse        <- prune_split + cache_sort + build_inverted
 *                               (sparse.py:66-163, 219-235): thresholds, data-part
 *                               flags, layout order, postings — integer products
 *                               identical to the reference's
 *   hs_builder_dense_moments <- whiten_fit's mean and covariance (dense.py:333-348;
 *                               the d x d eigendecomposition stays on the host)
 *   hs_builder_gather_dense  <- the k-means training sample (dense.py:126-129),
 *                               whitened (dense.py:351-357)
 *   hs_builder_dense_encode  <- pq_encode(...)[order] + pack_codes + sq_encode of the
 *                               residual (pipeline.py:152-157, dense.py:138-170, 381-390)
 *   hs_builder_finish        -> an hs_index_t (the builder's arrays move into it)
 * Rows of a generated dataset are keyed by their global id (row0 + i), so the
 * id-range shards of a multi-GPU job generate exactly the rows of the full set. */
typedef struct hs_builder* hs_builder_t;

typedef struct {
  int64_t n;            /* rows generated: global ids [row0, row0 + n) */
  int64_t d_sparse;
  int64_t d_dense;
  double mean_nnz;      /* Poisson mean of the distinct sparse nonzeros per row */
  double zipf_s;        /* Zipf exponent of the dimension ranks (> 1) */
  int32_t value_law;    /* 0: |N(0,1)|, 1: lognormal(0,1) */
  int32_t dense_fp16;   /* store the normalised dense part as fp16 */
  uint64_t seed;        /* data seed */
  uint64_t perm_seed;   /* seed of the rank -> dim bijection (shared with queries) */
  int64_t row0;
} hs_gen_params;

int hs_builder_generate(const hs_gen_params* p, int device, hs_builder_t* out);
int hs_builder_upload(int64_t n, int64_t d_sparse, int64_t d_dense, const int64_t* indptr,
                      const uint32_t* indices, const float* data, const float* dense,
                      int32_t dense_fp16, int device, hs_builder_t* out);
void hs_builder_destroy(hs_builder_t b);
/* info[8] = {n, d_sparse, d_dense, nnz, n_active, nnz_post, n_head, dense_fp16} */
int hs_builder_info(hs_builder_t b, int64_t* info);
int hs_builder_phase_times(hs_builder_t b, double* sec, int32_t max_entries,
                           int32_t* n_entries, char* names, int32_t names_cap);
int hs_builder_download_rows(hs_builder_t b, int64_t lo, int64_t hi, int64_t* indptr,
                             uint32_t* indices, float* data, float* dense);
/* top_t < 0: top_t=None with the constant data_min; residual_min constant */
int hs_builder_sparse(hs_builder_t b, int64_t top_t, double data_min, double residual_min);
int hs_builder_download_sparse(hs_builder_t b, int64_t* order, uint32_t* post_dims,
                               int64_t* post_ptr, uint32_t* post_ids, float* post_w,
                               uint32_t* dmask, uint32_t* head_dims, float* head_thr);
/* column means [d] and the biased covariance [d][d] of the dense part (f64) */
int hs_builder_dense_moments(hs_builder_t b, double* mean, double* cov);
/* rows [m] (original ids) -> out [m][d] f64, whitened when fwd != NULL:
 * (x - mean) @ fwd^T (whiten_apply "data", dense.py:354) */
int hs_builder_gather_dense(hs_builder_t b, const int64_t* rows, int64_t m, const double* mean,
                            const double* fwd, double* out);
/* PQ codes + SQ residual in layout order; whitening (mean, fwd, inverse_t)
 * optional (NULL = off); centers as in hs_dense_encode */
int hs_builder_dense_encode(hs_builder_t b, int32_t K, const int32_t* subdims,
                            const float* centers, int32_t l, const double* wh_mean,
                            const double* wh_fwd, const double* wh_inverse_t);
int hs_builder_download_dense(hs_builder_t b, uint8_t* packed, float* sq_lo, float* sq_step,
                              uint8_t* sq_codes);
/* Raw dataset rows of original ids (local to the index) — sampled checks of a
 * GPU-built index whose dataset lives only on the device.  indptr [m+1]
 * (relative); call with indices/data NULL first to size them; dense [m][d] f32. */
int hs_index_gather_rows(hs_index_t index, const int64_t* ids, int64_t m, int64_t* indptr,
                         uint32_t* indices, float* data, float* dense);
/* move the products into a search index; the builder is consumed (destroyed,
 * also on failure) */
int hs_builder_finish(hs_builder_t b, double sparse_weight, double dense_weight,
                      int64_t id_offset, hs_index_t* out);

#ifdef __cplusplus
}
#endif
#endif /* HSB200_H */
