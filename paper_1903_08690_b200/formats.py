"""The reference's on-disk formats, read natively.

Readers go through `libhsbuild.so` (`csrc/formats.cpp`, C ABI in
`include/hsformats.h`): the file is mmap-ed, validated once, and decoded
straight into the CSR arrays the device index consumes — no per-dimension
dict of posting lists.  Writers produce byte-identical files to the
reference's savers.  Names, signatures and exceptions follow the reference:

    save_dataset / load_dataset                  data.py:270-296      (HYBX)
    save_inverted_index / load_inverted_index    sparse.py:369-410    (HSIX)
    save_dense_index / load_dense_index          dense.py:433-516     (HDPQ)
    save_index / load_index                      pipeline.py:362-453  (HIDX)

`load_device_index(path, device, dataset)` is the file -> GPU path: the
decoded arrays go to `hs_index_create` directly.
"""

from __future__ import annotations

import ctypes
import io
import json
import os
import struct
import tempfile
import threading
from dataclasses import asdict

import numpy as np
import scipy.sparse as sp

from .types import (
    LUT16_CENTERS,
    BadMagicError,
    BadVersionError,
    Codebooks,
    DenseIndex,
    FormatError,
    HybridDataset,
    HybridIndex,
    HybridIndexConfig,
    InvertedIndex,
    PQCodes,
    ScalarQuantResidual,
    TruncatedFileError,
    WhiteningTransform,
)

HS_FILE_HIDX, HS_FILE_HSIX, HS_FILE_HDPQ, HS_FILE_HYBX = 1, 2, 3, 4
_EIO, _EBADMAGIC, _EBADVERSION, _ETRUNC, _EINVAL = 1, 2, 3, 4, 5

DATASET_MAGIC, DATASET_VERSION = b"HYBX", 1
INDEX_MAGIC, INDEX_VERSION = b"HSIX", 1
DENSE_MAGIC, DENSE_VERSION = b"HDPQ", 1
COMPOSITE_MAGIC, COMPOSITE_VERSION = b"HIDX", 1
_POSTING_DTYPE = np.dtype([("id", "<u4"), ("w", "<f4")])

i32, i64, P = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class FileInfo(ctypes.Structure):
    _fields_ = [
        ("kind", i32), ("n", i64), ("d_sparse", i64), ("d_dense", i64),
        ("has_sparse", i32), ("n_active", i64), ("post_nnz", i64),
        ("has_residual", i32), ("res_rows", i64), ("res_nnz", i64),
        ("has_dense", i32), ("n_subspaces", i32), ("n_centers", i32),
        ("centers_len", i64), ("codes_bytes", i64), ("has_sq", i32), ("has_whitening", i32),
        ("ds_nnz", i64), ("meta_len", i64),
    ]


_LIB = None
_LIB_LOCK = threading.Lock()


def _lib():
    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            from ._build import LIB_HOST, build_host

            if not os.path.exists(LIB_HOST):
                build_host()
            L = ctypes.CDLL(LIB_HOST)
            L.hs_file_last_error.restype = ctypes.c_char_p
            L.hs_file_open.argtypes = [ctypes.c_char_p, i32, ctypes.POINTER(P), ctypes.POINTER(FileInfo)]
            L.hs_file_close.argtypes = [P]
            L.hs_file_close.restype = None
            L.hs_file_read_meta.argtypes = [P, P]
            L.hs_file_read_sparse.argtypes = [P] + [P] * 5
            L.hs_file_read_csr.argtypes = [P] + [P] * 3
            L.hs_file_read_dense.argtypes = [P] + [P] * 9
            L.hs_file_read_dataset_dense.argtypes = [P, P]
            _LIB = L
        return _LIB


def _check(rc):
    if rc == 0:
        return
    msg = _lib().hs_file_last_error().decode(errors="replace")
    exc = {_EIO: OSError, _EBADMAGIC: BadMagicError, _EBADVERSION: BadVersionError,
           _ETRUNC: TruncatedFileError}.get(rc, FormatError)
    raise exc(msg)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data if a is not None else 0)


class _File:
    """One mapped file (context manager); `info` holds the array sizes."""

    def __init__(self, path_or_file, kind):
        self._tmp = None
        if hasattr(path_or_file, "read"):  # file-like (the reference accepts BytesIO)
            t = tempfile.NamedTemporaryFile(prefix="hsfmt_", delete=False)
            t.write(path_or_file.read())
            t.close()
            self._tmp = path = t.name
        else:
            path = os.fspath(path_or_file)
        self.info = FileInfo()
        self.h = ctypes.c_void_p()
        try:
            _check(_lib().hs_file_open(os.fsencode(path), kind, ctypes.byref(self.h),
                                       ctypes.byref(self.info)))
        except BaseException:
            self._cleanup()
            raise

    def _cleanup(self):
        if self._tmp is not None:
            os.unlink(self._tmp)
            self._tmp = None

    def close(self):
        if self.h:
            _lib().hs_file_close(self.h)
            self.h = ctypes.c_void_p()
        self._cleanup()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- decoders --------------------------------------------------------------
    def sparse_index(self) -> InvertedIndex:
        fi = self.info
        order = np.empty(fi.n, np.int64)
        dims = np.empty(fi.n_active, np.int64)
        ptr = np.empty(fi.n_active + 1, np.int64)
        ids = np.empty(fi.post_nnz, np.uint32)
        w = np.empty(fi.post_nnz, np.float32)
        _check(_lib().hs_file_read_sparse(self.h, _ptr(order), _ptr(dims), _ptr(ptr), _ptr(ids), _ptr(w)))
        return InvertedIndex(fi.n, fi.d_sparse, order, dims=dims, ptr=ptr, ids=ids, w=w)

    def csr(self, n_cols) -> sp.csr_matrix:
        fi = self.info
        nnz = fi.ds_nnz if fi.kind == HS_FILE_HYBX else fi.res_nnz
        indptr = np.empty(fi.res_rows + 1, np.int64)
        indices = np.empty(nnz, np.int32)
        data = np.empty(nnz, np.float32)
        _check(_lib().hs_file_read_csr(self.h, _ptr(indptr), _ptr(indices), _ptr(data)))
        return sp.csr_matrix((data, indices, indptr), shape=(fi.res_rows, n_cols))

    def dense_index(self) -> DenseIndex:
        fi = self.info
        K, l, d, n = fi.n_subspaces, fi.n_centers, fi.d_dense, fi.n
        subdims = np.empty(K, np.int64)
        centers = np.empty(fi.centers_len, np.float32)
        codes = np.empty(fi.codes_bytes, np.uint8)
        sq = [np.empty(d, np.float32), np.empty(d, np.float32), np.empty((n, d), np.uint8)] \
            if fi.has_sq else [None] * 3
        wh = [np.empty(d, np.float64), np.empty((d, d), np.float64), np.empty((d, d), np.float64)] \
            if fi.has_whitening else [None] * 3
        _check(_lib().hs_file_read_dense(self.h, _ptr(subdims), _ptr(centers), _ptr(codes),
                                         *[_ptr(a) for a in sq], *[_ptr(a) for a in wh]))
        blocks, off = [], 0
        for k in range(K):
            m = l * int(subdims[k])
            blocks.append(centers[off:off + m].reshape(l, int(subdims[k])))
            off += m
        cb = Codebooks(subdims=subdims, centers=blocks)
        if l == LUT16_CENTERS:
            pq = PQCodes(n=n, n_subspaces=K, n_centers=l, packed=codes.reshape((K + 1) // 2, n))
        else:
            pq = PQCodes(n=n, n_subspaces=K, n_centers=l, bytes_wide=codes.reshape(n, K))
        residual = ScalarQuantResidual(lo=sq[0], step=sq[1], codes=sq[2]) if fi.has_sq else None
        whitening = (WhiteningTransform(forward=wh[1], inverse_t=wh[2], mean=wh[0])
                     if fi.has_whitening else None)
        return DenseIndex(codebooks=cb, codes=pq, residual=residual, whitening=whitening)


# ----------------------------------------------------------------------------
# HYBX datasets (data.py:250-296)
# ----------------------------------------------------------------------------
def save_dataset(ds: HybridDataset, path) -> None:
    """Write a dataset in the HYBX binary format (bit-exact round trip)."""
    with open(path, "wb") as f:
        f.write(DATASET_MAGIC)
        f.write(struct.pack("<IQQI", DATASET_VERSION, ds.n, ds.d_sparse, ds.d_dense))
        f.write(np.ascontiguousarray(ds.dense, dtype="<f4").tobytes())
        f.write(ds.sparse.indptr.astype("<u8").tobytes())
        f.write(ds.sparse.indices.astype("<u4").tobytes())
        f.write(ds.sparse.data.astype("<f4").tobytes())


def load_dataset(path) -> HybridDataset:
    """Read a HYBX dataset; raises a distinct FormatError per failure mode."""
    with _File(path, HS_FILE_HYBX) as f:
        fi = f.info
        dense = np.empty((fi.n, fi.d_dense), np.float32)
        _check(_lib().hs_file_read_dataset_dense(f.h, _ptr(dense)))
        mat = f.csr(fi.d_sparse)
    return HybridDataset(mat, dense)


# ----------------------------------------------------------------------------
# HSIX sparse scan index (sparse.py:365-410)
# ----------------------------------------------------------------------------
def _inverted_bytes(index) -> bytes:
    if not hasattr(index, "ptr"):  # the reference's dict form
        index = InvertedIndex(index.n, index.d_sparse, index.order, index.lists)
    counts = index.nnz_per_dim
    if np.any(counts >= 2 ** 32):
        raise ValueError("posting list longer than 2^32")
    rec = np.empty(index.nnz, dtype=_POSTING_DTYPE)
    rec["id"] = index.ids
    rec["w"] = index.w
    return b"".join([INDEX_MAGIC, struct.pack("<IQQ", INDEX_VERSION, index.n, index.d_sparse),
                     np.asarray(index.order).astype("<u4").tobytes(),
                     counts.astype("<u4").tobytes(), rec.tobytes()])


def save_inverted_index(index, path_or_file) -> None:
    blob = _inverted_bytes(index)
    if hasattr(path_or_file, "write"):
        path_or_file.write(blob)
    else:
        with open(path_or_file, "wb") as f:
            f.write(blob)


def load_inverted_index(path_or_file) -> InvertedIndex:
    with _File(path_or_file, HS_FILE_HSIX) as f:
        return f.sparse_index()


# ----------------------------------------------------------------------------
# HDPQ dense PQ index (dense.py:423-516)
# ----------------------------------------------------------------------------
def _dense_bytes(idx: DenseIndex) -> bytes:
    cb, codes = idx.codebooks, idx.codes
    out = [DENSE_MAGIC, struct.pack("<IQIII", DENSE_VERSION, codes.n, cb.d_dense,
                                    cb.n_subspaces, cb.n_centers),
           np.asarray(cb.subdims).astype("<u4").tobytes()]
    out += [np.ascontiguousarray(c, dtype="<f4").tobytes() for c in cb.centers]
    arr = codes.packed if codes.packed is not None else codes.bytes_wide
    out.append(np.asarray(arr).astype("<u1").tobytes())
    out.append(struct.pack("<B", 1 if idx.residual is not None else 0))
    if idx.residual is not None:
        r = idx.residual
        out += [r.lo.astype("<f4").tobytes(), r.step.astype("<f4").tobytes(),
                r.codes.astype("<u1").tobytes()]
    out.append(struct.pack("<B", 1 if idx.whitening is not None else 0))
    if idx.whitening is not None:
        w = idx.whitening
        out += [w.mean.astype("<f8").tobytes(), w.forward.astype("<f8").tobytes(),
                w.inverse_t.astype("<f8").tobytes()]
    return b"".join(out)


def save_dense_index(idx: DenseIndex, path_or_file) -> None:
    blob = _dense_bytes(idx)
    if hasattr(path_or_file, "write"):
        path_or_file.write(blob)
    else:
        with open(path_or_file, "wb") as f:
            f.write(blob)


def load_dense_index(path_or_file) -> DenseIndex:
    with _File(path_or_file, HS_FILE_HDPQ) as f:
        return f.dense_index()


# ----------------------------------------------------------------------------
# HIDX composite index (pipeline.py:362-453)
# ----------------------------------------------------------------------------
def _config_to_json(cfg) -> dict:
    raw = asdict(cfg)
    for key, val in raw.items():
        if isinstance(val, np.ndarray):
            raw[key] = val.tolist()
    return raw


def save_index(index: HybridIndex, path) -> None:
    """Write the composite index (the raw dataset is not included)."""
    meta = {"n": index.n, "d_sparse": index.d_sparse, "d_dense": index.d_dense,
            "config": _config_to_json(index.config)}
    res = sp.csr_matrix(index.sparse_residual)
    buf = io.BytesIO()
    buf.write(struct.pack("<QQ", res.shape[0], res.nnz))
    buf.write(res.indptr.astype("<u8").tobytes())
    buf.write(res.indices.astype("<u4").tobytes())
    buf.write(res.data.astype("<f4").tobytes())
    sections = [(b"META", json.dumps(meta, sort_keys=True).encode()),
                (b"SPIX", _inverted_bytes(index.sparse_index)),
                (b"SRES", buf.getvalue())]
    if index.dense_index is not None:
        sections.append((b"DPQX", _dense_bytes(index.dense_index)))
    with open(path, "wb") as f:
        f.write(COMPOSITE_MAGIC)
        f.write(struct.pack("<II", COMPOSITE_VERSION, len(sections)))
        offset = 12 + 20 * len(sections)
        for tag, blob in sections:
            f.write(tag)
            f.write(struct.pack("<QQ", offset, len(blob)))
            offset += len(blob)
        for _, blob in sections:
            f.write(blob)


def load_index(path, dataset: HybridDataset | None = None) -> HybridIndex:
    """Read a composite index; attach ``dataset`` to re-enable exact rerank."""
    with _File(path, HS_FILE_HIDX) as f:
        fi = f.info
        raw = ctypes.create_string_buffer(max(fi.meta_len, 1))
        _check(_lib().hs_file_read_meta(f.h, raw))
        meta = json.loads(raw.raw[:fi.meta_len].decode())
        config = HybridIndexConfig(**meta["config"])
        # META against the blobs: the device upload sizes every array by n
        if (int(meta["n"]) != int(fi.n) or int(meta["d_sparse"]) != int(fi.d_sparse)
                or int(meta["d_dense"]) != int(fi.d_dense)):
            raise FormatError(
                f"META (n={meta['n']}, d_sparse={meta['d_sparse']}, d_dense={meta['d_dense']}) "
                f"does not match the index sections (n={fi.n}, d_sparse={fi.d_sparse}, "
                f"d_dense={fi.d_dense})")
        sparse_index = f.sparse_index()
        residual = f.csr(meta["d_sparse"])
        dense_index = f.dense_index() if fi.has_dense else None
    return HybridIndex(config=config, n=meta["n"], d_sparse=meta["d_sparse"],
                       d_dense=meta["d_dense"], order=sparse_index.order,
                       sparse_index=sparse_index, sparse_residual=residual,
                       dense_index=dense_index, dataset=dataset)


def load_device_index(path, device: int = 0, dataset: HybridDataset | None = None):
    """HIDX file -> device index handle (`DeviceIndex`), cached on the index."""
    from .search import device_index

    index = load_index(path, dataset)
    device_index(index, device)
    return index
