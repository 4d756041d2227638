/* hsformats.h — native readers of the reference's on-disk index / dataset
 * formats, exported by libhsbuild.so (host C++).
 *
 * A file is mapped once (mmap) and decoded straight into caller-allocated
 * arrays in the layout `hs_index_desc` (hsb200.h) consumes, so a cached
 * reference index reaches the device without the per-dimension dict of
 * posting lists the reference's loader builds.  Reference interfaces:
 *
 *   kind HS_FILE_HIDX  <- load_index            pipeline.py:362-453 (magic "HIDX")
 *   kind HS_FILE_HSIX  <- load_inverted_index   sparse.py:365-410   (magic "HSIX")
 *   kind HS_FILE_HDPQ  <- load_dense_index      dense.py:423-516    (magic "HDPQ")
 *   kind HS_FILE_HYBX  <- load_dataset          data.py:250-296     (magic "HYBX")
 *
 * Two phases: hs_file_open validates the whole file (magic, version, every
 * length against the file size) and reports the array sizes; the caller
 * allocates and calls the hs_file_read_* functions it needs; hs_file_close
 * unmaps.  Errors carry the reference's exception class in the status and its
 * message ("truncated file while reading <what>", ...) in hs_file_last_error().
 */
#ifndef HSFORMATS_H
#define HSFORMATS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HS_FILE_HIDX = 1,
  HS_FILE_HSIX = 2,
  HS_FILE_HDPQ = 3,
  HS_FILE_HYBX = 4
};

enum {
  HS_FMT_OK = 0,
  HS_FMT_EIO = 1,          /* -> OSError (open/mmap failed) */
  HS_FMT_EBADMAGIC = 2,    /* -> BadMagicError   (data.py:288, sparse.py:397, dense.py:482, pipeline.py:421) */
  HS_FMT_EBADVERSION = 3,  /* -> BadVersionError (data.py:291, sparse.py:400, dense.py:485, pipeline.py:424) */
  HS_FMT_ETRUNCATED = 4,   /* -> TruncatedFileError (data.py:258-262) */
  HS_FMT_EINVAL = 5        /* -> ValueError (missing section, wrong kind, bad argument) */
};

typedef struct hs_file* hs_file_t;

typedef struct {
  int32_t kind;            /* HS_FILE_* */
  int64_t n, d_sparse, d_dense;
  /* sparse scan index (HIDX SPIX section, HSIX) */
  int32_t has_sparse;
  int64_t n_active;        /* dims with a non-empty posting list */
  int64_t post_nnz;        /* postings */
  /* sparse residual (HIDX SRES section) */
  int32_t has_residual;
  int64_t res_rows, res_nnz;
  /* dense PQ index (HIDX DPQX section, HDPQ) */
  int32_t has_dense;
  int32_t n_subspaces, n_centers;
  int64_t centers_len;     /* floats over all subspaces */
  int64_t codes_bytes;     /* (K+1)/2 * n packed (l == 16) or n * K wide */
  int32_t has_sq, has_whitening;
  /* dataset (HYBX) */
  int64_t ds_nnz;
  /* HIDX META JSON length in bytes (no terminator) */
  int64_t meta_len;
} hs_file_info;

const char* hs_file_last_error(void);

/* expect_kind = 0 accepts any of the four magics. */
int hs_file_open(const char* path, int32_t expect_kind, hs_file_t* out, hs_file_info* info);
void hs_file_close(hs_file_t f);

/* META JSON bytes (HIDX only), meta_len bytes. */
int hs_file_read_meta(hs_file_t f, char* buf);

/* order[n] (i64), dims[n_active] (i64, ascending), ptr[n_active+1] (i64),
 * ids[post_nnz] (u32 layout slots), w[post_nnz] (f32). */
int hs_file_read_sparse(hs_file_t f, int64_t* order, int64_t* dims, int64_t* ptr,
                        uint32_t* ids, float* w);

/* CSR of the residual (HIDX) or of the dataset's sparse part (HYBX):
 * indptr[rows+1] (i64), indices[nnz] (i32), data[nnz] (f32). */
int hs_file_read_csr(hs_file_t f, int64_t* indptr, int32_t* indices, float* data);

/* Dense PQ index: subdims[K] (i64), centers[centers_len] (concatenation of the
 * l x subdims[k] row-major blocks), codes[codes_bytes]; sq_* and wh_* may be
 * NULL when the flag is 0. */
int hs_file_read_dense(hs_file_t f, int64_t* subdims, float* centers, uint8_t* codes,
                       float* sq_lo, float* sq_step, uint8_t* sq_codes,
                       double* wh_mean, double* wh_forward, double* wh_inverse_t);

/* HYBX dense block [n][d_dense] f32. */
int hs_file_read_dataset_dense(hs_file_t f, float* dense);

#ifdef __cplusplus
}
#endif

#endif /* HSFORMATS_H */
