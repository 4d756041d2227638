"""Native readers of the reference's file formats.

Fixtures in tests/golden/formats/ were written by the REFERENCE's savers
(tests/golden/make_formats.py).  CPU tests: our readers decode them into the
arrays the reference's loaders return, our writers reproduce them byte for
byte, and the reference's error classes/messages come back for bad magic,
bad version and every truncation point (test_data.py:150-177 is the
reference's own version of those checks).  GPU test: file -> device index ->
search gives the reference's ids and scores.
"""

from __future__ import annotations

import io
import json
import os
import struct

import numpy as np
import pytest

import paper_1903_08690_b200 as hs

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")
TAGS = ["default", "odd", "sparse_only"]


def path(name):
    return os.path.join(HERE, name)


def expect():
    return np.load(path("expect.npz"))


def raw(name):
    with open(path(name), "rb") as f:
        return f.read()


@pytest.mark.parametrize("tag", TAGS)
def test_hidx_decodes_to_reference_arrays(tag):
    z = expect()
    idx = hs.load_index(path(f"{tag}.hidx"))
    assert np.array_equal(idx.order, z[f"{tag}_order"])
    assert np.array_equal(idx.sparse_index.nnz_per_dim, z[f"{tag}_nnz_per_dim"])
    r = idx.sparse_residual
    assert np.array_equal(r.indptr, z[f"{tag}_res_indptr"])
    assert np.array_equal(r.indices, z[f"{tag}_res_indices"])
    assert np.array_equal(r.data, z[f"{tag}_res_data"])
    assert tuple(r.shape) == tuple(z[f"{tag}_res_shape"])
    assert (idx.dense_index is None) == (tag == "sparse_only")


@pytest.mark.parametrize("tag", TAGS)
def test_writers_reproduce_reference_files(tmp_path, tag):
    idx = hs.load_index(path(f"{tag}.hidx"))
    hs.save_index(idx, tmp_path / "i.hidx")
    assert (tmp_path / "i.hidx").read_bytes() == raw(f"{tag}.hidx")
    ds = hs.load_dataset(path(f"{tag}.hybx"))
    hs.save_dataset(ds, tmp_path / "d.hybx")
    assert (tmp_path / "d.hybx").read_bytes() == raw(f"{tag}.hybx")
    sidx = hs.load_inverted_index(path(f"{tag}.hsix"))
    buf = io.BytesIO()
    hs.save_inverted_index(sidx, buf)
    assert buf.getvalue() == raw(f"{tag}.hsix")
    if tag != "sparse_only":
        di = hs.load_dense_index(io.BytesIO(raw(f"{tag}.hdpq")))  # file-like input
        buf = io.BytesIO()
        hs.save_dense_index(di, buf)
        assert buf.getvalue() == raw(f"{tag}.hdpq")


def test_standalone_blobs_match_composite():
    idx = hs.load_index(path("default.hidx"))
    s = hs.load_inverted_index(path("default.hsix"))
    for a in ("order", "dims", "ptr", "ids", "w"):
        assert np.array_equal(getattr(s, a), getattr(idx.sparse_index, a))
    d = hs.load_dense_index(path("default.hdpq"))
    assert np.array_equal(d.codes.packed, idx.dense_index.codes.packed)
    for a, b in zip(d.codebooks.centers, idx.dense_index.codebooks.centers):
        assert np.array_equal(a, b)


def test_load_index_with_oracle_search_matches_reference():
    """The decoded index drives the CPU oracle to the reference's results."""
    from oracle import hybrid_oracle as O

    z = expect()
    for tag in TAGS:
        ds = hs.load_dataset(path(f"{tag}.hybx"))
        qs = hs.load_dataset(path(f"{tag}_q.hybx"))
        idx = hs.load_index(path(f"{tag}.hidx"), dataset=ds)
        for si, st in enumerate(json.loads(str(z[f"{tag}_settings"]))):
            kw = {k: v for k, v in st.items() if k != "h"}
            res = O.search_batch(idx, qs, st["h"], **kw)
            ids = np.stack([r[0] for r in res])
            np.testing.assert_allclose(np.stack([r[1] for r in res]), z[f"{tag}_s{si}_scores"],
                                       rtol=1e-12, atol=1e-14)
            assert ids.tolist() == z[f"{tag}_s{si}_ids"].tolist(), (tag, si)


# ---- error behaviour (data.py:258-296, sparse.py:393-410, dense.py:478-516,
#      pipeline.py:413-430) ----
KINDS = [("default.hidx", hs.load_index, "not a hybrid index file", "unsupported index version"),
         ("default.hsix", hs.load_inverted_index, "not a sparse index file",
          "unsupported sparse index version"),
         ("default.hdpq", hs.load_dense_index, "not a dense index file",
          "unsupported dense index version"),
         ("default.hybx", hs.load_dataset, "not a dataset file", "unsupported dataset version")]


@pytest.mark.parametrize("name,loader,magic_msg,version_msg", KINDS)
def test_bad_magic_and_version(tmp_path, name, loader, magic_msg, version_msg):
    b = raw(name)
    p = tmp_path / "bad"
    p.write_bytes(b"XXXX" + b[4:])
    with pytest.raises(hs.BadMagicError, match=magic_msg):
        loader(p)
    p.write_bytes(b[:4] + struct.pack("<I", 7) + b[8:])
    with pytest.raises(hs.BadVersionError, match=version_msg + " 7"):
        loader(p)


@pytest.mark.parametrize("name,loader", [(k[0], k[1]) for k in KINDS])
def test_every_truncation_raises(tmp_path, name, loader):
    b = raw(name)
    p = tmp_path / "cut"
    rng = np.random.default_rng(0)
    cuts = sorted(set(list(range(0, 64)) + rng.integers(64, len(b), 40).tolist() + [len(b) - 1]))
    for n in cuts:
        p.write_bytes(b[:n])
        with pytest.raises(hs.TruncatedFileError, match="truncated file while reading"):
            loader(p)
    assert issubclass(hs.TruncatedFileError, hs.FormatError)


def test_truncation_messages_name_the_field(tmp_path):
    b = raw("default.hybx")
    p = tmp_path / "cut"
    for n, what in [(2, "magic"), (10, "header"), (40, "dense block")]:
        p.write_bytes(b[:n])
        with pytest.raises(hs.TruncatedFileError, match=f"while reading {what}$"):
            hs.load_dataset(p)
    s = raw("default.hsix")
    p.write_bytes(s[:-1])
    with pytest.raises(hs.TruncatedFileError, match="while reading postings dim"):
        hs.load_inverted_index(p)
    h = raw("default.hidx")
    p.write_bytes(h[:-1])
    with pytest.raises(hs.TruncatedFileError, match="while reading section b'DPQX'"):
        hs.load_index(p)


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        hs.load_index(tmp_path / "nope.hidx")


def test_native_format_symbols_exported():
    import ctypes

    from paper_1903_08690_b200._build import LIB_HOST, REPO

    L = ctypes.CDLL(LIB_HOST)
    hdr = open(os.path.join(REPO, "include", "hsformats.h")).read()
    import re

    names = set(re.findall(r"\b(hs_file_\w+)\s*\(", hdr))
    assert len(names) >= 7
    for n in names:
        assert hasattr(L, n), n


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_file_to_device_search_matches_reference(tag):
    z = expect()
    ds = hs.load_dataset(path(f"{tag}.hybx"))
    qs = hs.load_dataset(path(f"{tag}_q.hybx"))
    idx = hs.load_device_index(path(f"{tag}.hidx"), 0, dataset=ds)
    for si, st in enumerate(json.loads(str(z[f"{tag}_settings"]))):
        kw = {k: v for k, v in st.items() if k != "h"}
        res = hs.search_batch(idx, qs, st["h"], **kw)
        assert np.stack([r.ids for r in res]).tolist() == z[f"{tag}_s{si}_ids"].tolist(), (tag, si)
        np.testing.assert_allclose(np.stack([r.scores for r in res]), z[f"{tag}_s{si}_scores"],
                                   rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_corrupt_index_rejected_before_upload():
    """A posting id or layout slot outside [0, n) (a damaged file) is refused
    by hs_index_create instead of being dereferenced on the device."""
    idx = hs.load_index(path("default.hidx"))
    idx.sparse_index.ids[3] = idx.n + 5
    with pytest.raises(ValueError, match="posting id out of range"):
        hs.DeviceIndex(idx, device=0)
    idx = hs.load_index(path("default.hidx"))
    idx.order[0] = idx.n
    with pytest.raises(ValueError, match="layout order out of range"):
        hs.DeviceIndex(idx, device=0)


def test_meta_must_match_the_sections(tmp_path):
    """A hand-edited META n (the loop bound of the device upload) that
    disagrees with the section arrays is rejected at load time."""
    b = raw("default.hidx")
    assert b.count(b'"n": 3000') == 1
    p = tmp_path / "meta.hidx"
    p.write_bytes(b.replace(b'"n": 3000', b'"n": 9000'))
    with pytest.raises(hs.FormatError, match="does not match the index sections"):
        hs.load_index(p)


@pytest.mark.gpu
def test_corrupt_csr_rejected_before_upload():
    """Residual / dataset CSR row pointers that are not monotone (scipy only
    checks the first and last entry) are refused by hs_index_create."""
    import scipy.sparse as sp

    idx = hs.load_index(path("default.hidx"))
    r = idx.sparse_residual
    ptr = r.indptr.copy()
    ptr[2], ptr[3] = ptr[3] + 5, ptr[2]
    idx.sparse_residual = sp.csr_matrix((r.data, r.indices, ptr), shape=r.shape)
    with pytest.raises(ValueError, match="sparse residual row pointers not monotone"):
        hs.DeviceIndex(idx, device=0)
    idx = hs.load_index(path("default.hidx"))
    r = idx.sparse_residual
    idx.sparse_residual = sp.csr_matrix((r.data, r.indices, r.indptr), shape=r.shape)
    idx.sparse_residual.indices[0] = idx.d_sparse + 1
    with pytest.raises(ValueError, match="sparse residual column index out of range"):
        hs.DeviceIndex(idx, device=0)
