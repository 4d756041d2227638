// formats.cpp — mmap readers of the reference's index / dataset files
// (include/hsformats.h).  Host C++, part of
// libhsbuild.so.  Formats (all little-endian):
//   HYBX data.py:250-296       magic, u32 version, u64 N, u64 d_sparse, u32 d_dense,
//                              dense f32 [N][d_dense], CSR u64 offsets, u32 dims, f32 values
//   HSIX sparse.py:365-410     magic, u32 version, u64 N, u64 d_sparse, u32 order[N],
//                              u32 counts[d_sparse], then (u32 id, f32 w) per posting,
//                              dims ascending
//   HDPQ dense.py:423-516      magic, u32 version, u64 N, u32 d, u32 K, u32 l, u32 subdims[K],
//                              f32 centers per subspace, codes, u8 sq flag [+ lo, step, codes],
//                              u8 whitening flag [+ f64 mean, forward, inverse_t]
//   HIDX pipeline.py:362-453   magic, u32 version, u32 count, (tag, u64 off, u64 len)[count];
//                              sections META (JSON), SPIX (HSIX blob), SRES (u64 rows,
//                              u64 nnz, u64 indptr, u32 indices, f32 data), DPQX (HDPQ blob)
// The whole file is validated at open (every read the reference's loader
// would make is bounds-checked against the mapping); the read calls then
// decode with no further checks.
#include "../../include/hsformats.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct FmtError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw FmtError{code, std::move(msg)}; }

// Bounded cursor over a byte range; need() mirrors data.py:258-262.
struct Cursor {
  const uint8_t* base;
  size_t pos, end;
  const uint8_t* take(size_t nbytes, const std::string& what) {
    if (nbytes > end - pos) fail(HS_FMT_ETRUNCATED, "truncated file while reading " + what);
    const uint8_t* p = base + pos;
    pos += nbytes;
    return p;
  }
  template <class T>
  T get(const std::string& what) {
    T v;
    std::memcpy(&v, take(sizeof(T), what), sizeof(T));
    return v;
  }
};

// Checked byte count a*b (SIZE_MAX on overflow, which no cursor can satisfy,
// so a hostile length reads as a truncated file instead of wrapping).
inline size_t nb(size_t a, size_t b) {
  size_t r;
  return __builtin_mul_overflow(a, b, &r) ? SIZE_MAX : r;
}

template <class T>
T ld(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

std::string bytes_repr(const uint8_t* m, size_t n) {
  std::string s = "b'";
  for (size_t i = 0; i < n; ++i) {
    unsigned c = m[i];
    if (c == '\\' || c == '\'') {
      s += '\\';
      s += char(c);
    } else if (c >= 32 && c < 127) {
      s += char(c);
    } else {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\x%02x", c);
      s += buf;
    }
  }
  return s + "'";
}

struct SparseView {  // a validated HSIX blob
  int64_t n = 0, d = 0, n_active = 0, nnz = 0;
  const uint8_t* order = nullptr;   // u32[n]
  const uint8_t* counts = nullptr;  // u32[d]
  const uint8_t* recs = nullptr;    // (u32, f32)[nnz]
};

struct DenseView {  // a validated HDPQ blob
  int64_t n = 0;
  int32_t d = 0, K = 0, l = 0;
  const uint8_t* subdims = nullptr;
  const uint8_t* centers = nullptr;
  int64_t centers_len = 0, codes_bytes = 0;
  const uint8_t* codes = nullptr;
  int32_t has_sq = 0, has_wh = 0;
  const uint8_t *sq_lo = nullptr, *sq_step = nullptr, *sq_codes = nullptr;
  const uint8_t *wh_mean = nullptr, *wh_fwd = nullptr, *wh_inv = nullptr;
};

struct CsrView {
  int64_t rows = 0, nnz = 0;
  const uint8_t* indptr = nullptr;  // u64[rows+1]
  const uint8_t* indices = nullptr; // u32[nnz]
  const uint8_t* data = nullptr;    // f32[nnz]
};

void check_magic(Cursor& c, const char* magic, const std::string& bad_msg, bool repr) {
  const uint8_t* m = c.take(4, "magic");
  if (std::memcmp(m, magic, 4) != 0)
    fail(HS_FMT_EBADMAGIC, repr ? bad_msg + " (magic " + bytes_repr(m, 4) + ")" : bad_msg);
}

// sparse.py:393-410
SparseView parse_hsix(Cursor c) {
  SparseView v;
  check_magic(c, "HSIX", "not a sparse index file", false);
  const uint8_t* h = c.take(20, "header");
  uint32_t version = ld<uint32_t>(h);
  v.n = int64_t(ld<uint64_t>(h + 4));
  v.d = int64_t(ld<uint64_t>(h + 12));
  if (version != 1) fail(HS_FMT_EBADVERSION, "unsupported sparse index version " + std::to_string(version));
  if (v.n < 0 || v.d < 0) fail(HS_FMT_ETRUNCATED, "truncated file while reading permutation");
  v.order = c.take(nb(size_t(v.n), 4), "permutation");
  v.counts = c.take(nb(size_t(v.d), 4), "posting counts");
  v.recs = c.base + c.pos;
  size_t off = 0;
  for (int64_t j = 0; j < v.d; ++j) {
    uint32_t cnt = ld<uint32_t>(v.counts + 4 * j);
    if (!cnt) continue;
    ++v.n_active;
    off += size_t(cnt) * 8;
    if (off > c.end - c.pos) fail(HS_FMT_ETRUNCATED, "truncated file while reading postings dim " + std::to_string(j));
    v.nnz += cnt;
  }
  return v;
}

// dense.py:478-516
DenseView parse_hdpq(Cursor c) {
  DenseView v;
  check_magic(c, "HDPQ", "not a dense index file", false);
  const uint8_t* h = c.take(24, "header");
  uint32_t version = ld<uint32_t>(h);
  v.n = int64_t(ld<uint64_t>(h + 4));
  v.d = int32_t(ld<uint32_t>(h + 12));
  v.K = int32_t(ld<uint32_t>(h + 16));
  v.l = int32_t(ld<uint32_t>(h + 20));
  if (version != 1) fail(HS_FMT_EBADVERSION, "unsupported dense index version " + std::to_string(version));
  if (v.n < 0 || v.d < 0 || v.K < 0 || v.l < 0) fail(HS_FMT_EINVAL, "dense header out of range");
  v.subdims = c.take(nb(size_t(v.K), 4), "subdims");
  v.centers = c.base + c.pos;
  for (int32_t k = 0; k < v.K; ++k) {
    int64_t len = int64_t(v.l) * ld<uint32_t>(v.subdims + 4 * k);
    c.take(nb(size_t(len), 4), "centers " + std::to_string(k));
    v.centers_len += len;
  }
  const size_t cb = v.l == 16 ? nb(size_t((v.K + 1) / 2), size_t(v.n)) : nb(size_t(v.n), size_t(v.K));
  v.codes = c.take(cb, "codes");
  v.codes_bytes = int64_t(cb);
  v.has_sq = *c.take(1, "residual flag") ? 1 : 0;
  if (v.has_sq) {
    v.sq_lo = c.take(nb(size_t(v.d), 4), "sq lo");
    v.sq_step = c.take(nb(size_t(v.d), 4), "sq step");
    v.sq_codes = c.take(nb(size_t(v.n), size_t(v.d)), "sq codes");
  }
  v.has_wh = *c.take(1, "whitening flag") ? 1 : 0;
  if (v.has_wh) {
    v.wh_mean = c.take(nb(size_t(v.d), 8), "whitening mean");
    v.wh_fwd = c.take(nb(nb(size_t(v.d), size_t(v.d)), 8), "whitening forward");
    v.wh_inv = c.take(nb(nb(size_t(v.d), size_t(v.d)), 8), "whitening inverse");
  }
  return v;
}

// pipeline.py:440-445 (the SRES section)
CsrView parse_sres(Cursor c) {
  CsrView v;
  const uint8_t* h = c.take(16, "residual header");
  v.rows = int64_t(ld<uint64_t>(h));
  v.nnz = int64_t(ld<uint64_t>(h + 8));
  if (v.rows < 0 || v.nnz < 0) fail(HS_FMT_EINVAL, "residual header out of range");
  v.indptr = c.take(nb(size_t(v.rows) + 1, 8), "residual indptr");
  v.indices = c.take(nb(size_t(v.nnz), 4), "residual indices");
  v.data = c.take(nb(size_t(v.nnz), 4), "residual data");
  return v;
}

}  // namespace

struct hs_file {
  void* map = nullptr;
  size_t size = 0;
  int32_t kind = 0;
  int64_t n = 0, d_sparse = 0, d_dense = 0;
  bool has_sparse = false, has_residual = false, has_dense = false;
  SparseView sp;
  DenseView dn;
  CsrView csr;                       // SRES (HIDX) or dataset CSR (HYBX)
  const uint8_t* ds_dense = nullptr;  // HYBX
  const uint8_t* meta = nullptr;
  int64_t meta_len = 0;
};

namespace {

void parse_hybx(hs_file* f, Cursor c) {
  check_magic(c, "HYBX", "not a dataset file", true);
  const uint8_t* h = c.take(24, "header");
  uint32_t version = ld<uint32_t>(h);
  f->n = int64_t(ld<uint64_t>(h + 4));
  f->d_sparse = int64_t(ld<uint64_t>(h + 12));
  f->d_dense = int64_t(ld<uint32_t>(h + 20));
  if (version != 1) fail(HS_FMT_EBADVERSION, "unsupported dataset version " + std::to_string(version));
  if (f->n < 0) fail(HS_FMT_ETRUNCATED, "truncated file while reading dense block");
  f->ds_dense = c.take(nb(nb(size_t(f->n), size_t(f->d_dense)), 4), "dense block");
  f->csr.rows = f->n;
  f->csr.indptr = c.take(nb(size_t(f->n) + 1, 8), "csr offsets");
  f->csr.nnz = int64_t(ld<uint64_t>(f->csr.indptr + 8 * f->n));
  if (f->csr.nnz < 0) fail(HS_FMT_ETRUNCATED, "truncated file while reading csr indices");
  f->csr.indices = c.take(nb(size_t(f->csr.nnz), 4), "csr indices");
  f->csr.data = c.take(nb(size_t(f->csr.nnz), 4), "csr values");
  f->has_residual = true;
}

void parse_hidx(hs_file* f, Cursor c) {
  check_magic(c, "HIDX", "not a hybrid index file", false);
  const uint8_t* h = c.take(8, "header");
  uint32_t version = ld<uint32_t>(h), count = ld<uint32_t>(h + 4);
  if (version != 1) fail(HS_FMT_EBADVERSION, "unsupported index version " + std::to_string(version));
  struct Sec { const uint8_t* tag; uint64_t off, len; };
  std::vector<Sec> table;
  for (uint32_t i = 0; i < count; ++i) {
    const uint8_t* tag = c.take(4, "section tag");
    const uint8_t* e = c.take(16, "section entry");
    table.push_back({tag, ld<uint64_t>(e), ld<uint64_t>(e + 8)});
  }
  const Sec* meta = nullptr; const Sec* spix = nullptr; const Sec* sres = nullptr; const Sec* dpqx = nullptr;
  for (const Sec& s : table) {  // later duplicates win, as in the reference's dict
    if (s.off > c.end || s.len > c.end - s.off)
      fail(HS_FMT_ETRUNCATED, "truncated file while reading section " + bytes_repr(s.tag, 4));
    if (!std::memcmp(s.tag, "META", 4)) meta = &s;
    else if (!std::memcmp(s.tag, "SPIX", 4)) spix = &s;
    else if (!std::memcmp(s.tag, "SRES", 4)) sres = &s;
    else if (!std::memcmp(s.tag, "DPQX", 4)) dpqx = &s;
  }
  if (!meta || !spix || !sres) fail(HS_FMT_EINVAL, std::string("index file lacks section ") +
                                    (!meta ? "b'META'" : !spix ? "b'SPIX'" : "b'SRES'"));
  f->meta = c.base + meta->off;
  f->meta_len = int64_t(meta->len);
  f->sp = parse_hsix(Cursor{c.base + spix->off, 0, size_t(spix->len)});
  f->has_sparse = true;
  f->csr = parse_sres(Cursor{c.base + sres->off, 0, size_t(sres->len)});
  f->has_residual = true;
  if (dpqx) {
    f->dn = parse_hdpq(Cursor{c.base + dpqx->off, 0, size_t(dpqx->len)});
    f->has_dense = true;
  }
  // n / d_sparse / d_dense come from META in the reference; the blobs agree
  // for files it wrote, and the Python layer cross-checks META against them.
  // The blobs must agree with each other: every array the device index
  // uploads is sized by the sparse index's n.
  if (f->csr.rows != f->sp.n)
    fail(HS_FMT_EINVAL, "residual rows (" + std::to_string(f->csr.rows) +
                            ") do not match the sparse index (" + std::to_string(f->sp.n) + ")");
  if (f->has_dense && f->dn.n != f->sp.n)
    fail(HS_FMT_EINVAL, "dense index rows (" + std::to_string(f->dn.n) +
                            ") do not match the sparse index (" + std::to_string(f->sp.n) + ")");
  f->n = f->sp.n;
  f->d_sparse = f->sp.d;
  f->d_dense = f->has_dense ? f->dn.d : 0;
}

int guard(int (*fn)(void*), void* arg) {
  try {
    return fn(arg);
  } catch (const FmtError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HS_FMT_EINVAL;
  }
}

}  // namespace

extern "C" {

const char* hs_file_last_error(void) { return g_err.c_str(); }

int hs_file_open(const char* path, int32_t expect_kind, hs_file_t* out, hs_file_info* info) {
  if (!path || !out || !info) {
    g_err = "null argument";
    return HS_FMT_EINVAL;
  }
  *out = nullptr;
  int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) {
    g_err = std::string("cannot open ") + path + ": " + std::strerror(errno);
    return HS_FMT_EIO;
  }
  struct stat st;
  if (fstat(fd, &st) != 0) {
    g_err = std::string("cannot stat ") + path;
    ::close(fd);
    return HS_FMT_EIO;
  }
  hs_file* f = new hs_file;
  f->size = size_t(st.st_size);
  if (f->size) {
    f->map = mmap(nullptr, f->size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (f->map == MAP_FAILED) {
      ::close(fd);
      delete f;
      g_err = std::string("cannot map ") + path;
      return HS_FMT_EIO;
    }
    madvise(f->map, f->size, MADV_SEQUENTIAL | MADV_WILLNEED);
  }
  ::close(fd);
  struct Args { hs_file* f; int32_t kind; } a{f, expect_kind};
  int rc = guard([](void* p) -> int {
    Args* a = static_cast<Args*>(p);
    hs_file* f = a->f;
    static const uint8_t empty[1] = {0};
    Cursor c{f->map ? static_cast<const uint8_t*>(f->map) : empty, 0, f->size};
    int kind = a->kind;
    if (!kind) {
      const char* tags[4] = {"HIDX", "HSIX", "HDPQ", "HYBX"};
      kind = HS_FILE_HIDX;  // unknown magic reports as the composite
      for (int i = 0; i < 4 && f->size >= 4; ++i)
        if (!std::memcmp(c.base, tags[i], 4)) kind = i + 1;
    }
    f->kind = kind;
    switch (kind) {
      case HS_FILE_HIDX: parse_hidx(f, c); break;
      case HS_FILE_HSIX:
        f->sp = parse_hsix(c);
        f->has_sparse = true;
        f->n = f->sp.n;
        f->d_sparse = f->sp.d;
        break;
      case HS_FILE_HDPQ:
        f->dn = parse_hdpq(c);
        f->has_dense = true;
        f->n = f->dn.n;
        f->d_dense = f->dn.d;
        break;
      case HS_FILE_HYBX: parse_hybx(f, c); break;
      default: fail(HS_FMT_EINVAL, "unknown file kind " + std::to_string(kind));
    }
    return HS_FMT_OK;
  }, &a);
  if (rc != HS_FMT_OK) {
    hs_file_close(f);
    return rc;
  }
  std::memset(info, 0, sizeof *info);
  info->kind = f->kind;
  info->n = f->n;
  info->d_sparse = f->d_sparse;
  info->d_dense = f->d_dense;
  info->has_sparse = f->has_sparse;
  info->n_active = f->sp.n_active;
  info->post_nnz = f->sp.nnz;
  info->has_residual = f->has_residual;
  info->res_rows = f->csr.rows;
  info->res_nnz = f->csr.nnz;
  info->has_dense = f->has_dense;
  info->n_subspaces = f->dn.K;
  info->n_centers = f->dn.l;
  info->centers_len = f->dn.centers_len;
  info->codes_bytes = f->dn.codes_bytes;
  info->has_sq = f->dn.has_sq;
  info->has_whitening = f->dn.has_wh;
  info->ds_nnz = f->kind == HS_FILE_HYBX ? f->csr.nnz : 0;
  info->meta_len = f->meta_len;
  *out = f;
  return HS_FMT_OK;
}

void hs_file_close(hs_file_t f) {
  if (!f) return;
  if (f->map && f->map != MAP_FAILED) munmap(f->map, f->size);
  delete f;
}

int hs_file_read_meta(hs_file_t f, char* buf) {
  if (!f || !buf || !f->meta) {
    g_err = "no META section";
    return HS_FMT_EINVAL;
  }
  std::memcpy(buf, f->meta, size_t(f->meta_len));
  return HS_FMT_OK;
}

int hs_file_read_sparse(hs_file_t f, int64_t* order, int64_t* dims, int64_t* ptr, uint32_t* ids,
                        float* w) {
  if (!f || !f->has_sparse || !order || !dims || !ptr || !ids || !w) {
    g_err = "no sparse index in file (or null output)";
    return HS_FMT_EINVAL;
  }
  const SparseView& v = f->sp;
  for (int64_t i = 0; i < v.n; ++i) order[i] = ld<uint32_t>(v.order + 4 * i);
  int64_t a = 0, off = 0;
  ptr[0] = 0;
  for (int64_t j = 0; j < v.d; ++j) {
    uint32_t cnt = ld<uint32_t>(v.counts + 4 * j);
    if (!cnt) continue;
    dims[a] = j;
    off += cnt;
    ptr[++a] = off;
  }
  // de-interleave the (id, w) records: the device layout keeps ids and weights
  // in separate streams
#pragma omp parallel for schedule(static) if (v.nnz > (1 << 20))
  for (int64_t i = 0; i < v.nnz; ++i) {
    ids[i] = ld<uint32_t>(v.recs + 8 * i);
    w[i] = ld<float>(v.recs + 8 * i + 4);
  }
  return HS_FMT_OK;
}

int hs_file_read_csr(hs_file_t f, int64_t* indptr, int32_t* indices, float* data) {
  if (!f || !f->has_residual || !indptr || !indices || !data) {
    g_err = "no CSR block in file (or null output)";
    return HS_FMT_EINVAL;
  }
  const CsrView& v = f->csr;
  std::memcpy(indptr, v.indptr, nb(size_t(v.rows) + 1, 8));
  std::memcpy(data, v.data, nb(size_t(v.nnz), 4));
#pragma omp parallel for schedule(static) if (v.nnz > (1 << 20))
  for (int64_t i = 0; i < v.nnz; ++i) indices[i] = int32_t(ld<uint32_t>(v.indices + 4 * i));
  return HS_FMT_OK;
}

int hs_file_read_dense(hs_file_t f, int64_t* subdims, float* centers, uint8_t* codes, float* sq_lo,
                       float* sq_step, uint8_t* sq_codes, double* wh_mean, double* wh_forward,
                       double* wh_inverse_t) {
  if (!f || !f->has_dense || !subdims || !centers || !codes) {
    g_err = "no dense index in file (or null output)";
    return HS_FMT_EINVAL;
  }
  const DenseView& v = f->dn;
  for (int32_t k = 0; k < v.K; ++k) subdims[k] = ld<uint32_t>(v.subdims + 4 * k);
  std::memcpy(centers, v.centers, size_t(v.centers_len) * 4);
  std::memcpy(codes, v.codes, size_t(v.codes_bytes));
  const size_t d = size_t(v.d);
  if (v.has_sq) {
    if (!sq_lo || !sq_step || !sq_codes) {
      g_err = "null scalar-quant output";
      return HS_FMT_EINVAL;
    }
    std::memcpy(sq_lo, v.sq_lo, d * 4);
    std::memcpy(sq_step, v.sq_step, d * 4);
    std::memcpy(sq_codes, v.sq_codes, size_t(v.n) * d);
  }
  if (v.has_wh) {
    if (!wh_mean || !wh_forward || !wh_inverse_t) {
      g_err = "null whitening output";
      return HS_FMT_EINVAL;
    }
    std::memcpy(wh_mean, v.wh_mean, d * 8);
    std::memcpy(wh_forward, v.wh_fwd, d * d * 8);
    std::memcpy(wh_inverse_t, v.wh_inv, d * d * 8);
  }
  return HS_FMT_OK;
}

int hs_file_read_dataset_dense(hs_file_t f, float* dense) {
  if (!f || f->kind != HS_FILE_HYBX || (!dense && f->n * f->d_dense)) {
    g_err = "not a dataset file (or null output)";
    return HS_FMT_EINVAL;
  }
  std::memcpy(dense, f->ds_dense, nb(nb(size_t(f->n), size_t(f->d_dense)), 4));
  return HS_FMT_OK;
}

}  // extern "C"
