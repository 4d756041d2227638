"""Index build on the GPU from a GPU-resident dataset.

`build_index` (pipeline.py:119-162) for datasets that do not fit the host or
the reference's Python build — config 5 is 10^8 points with 5*10^9 sparse
nonzeros.  The dataset is generated on (or uploaded to) the GPU that will
search it and the index is built in place through `include/hsb200.h`'s
`hs_builder_*` entry points:

    DeviceDataset.generate(law, seed, ...)  the BASELINE data law on the device
                                            (rows keyed by global id: any id
                                            range generates the same rows)
    DeviceDataset.upload(dataset)           a host HybridDataset
    dd.build(config)                        -> GpuBuild (sparse + dense products)
        hs_builder_sparse        thresholds, data-part flags, cache_sort order,
                                 postings (integer products == the reference's)
        hs_builder_dense_moments mean / covariance -> whiten_fit's eigh on the host
        hs_builder_gather_dense  the k-means sample (reference RNG stream), whitened
        train_codebooks          host k-means on that sample (same streams)
        hs_builder_dense_encode  PQ codes + SQ residual, layout order
    build.host_index()                      download -> a reference-compatible
                                            HybridIndex (parity checks, small n)
    build.finish()                          -> DeviceBuiltIndex, searchable with
                                            search_batch / search_topk

The search never sees a host copy of the arrays: `DeviceBuiltIndex` carries
the device handle plus the host metadata the reference API reads (config,
sizes, codebooks, whitening).
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np
import scipy.sparse as sp

from . import _native as nat
from .types import (
    LUT16_CENTERS,
    Codebooks,
    DenseIndex,
    HybridDataset,
    HybridIndex,
    HybridIndexConfig,
    InvertedIndex,
    PQCodes,
    ScalarQuantResidual,
    WhiteningTransform,
)

P = ctypes.c_void_p
i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class GenParams(ctypes.Structure):
    _fields_ = [("n", i64), ("d_sparse", i64), ("d_dense", i64), ("mean_nnz", f64),
                ("zipf_s", f64), ("value_law", i32), ("dense_fp16", i32),
                ("seed", ctypes.c_uint64), ("perm_seed", ctypes.c_uint64), ("row0", i64)]


def _lib():
    L = nat.require_gpu()
    if not getattr(L, "_hsb_builder_bound", False):
        L.hs_builder_generate.argtypes = [ctypes.POINTER(GenParams), ctypes.c_int, ctypes.POINTER(P)]
        L.hs_builder_upload.argtypes = [i64, i64, i64, P, P, P, P, i32, ctypes.c_int,
                                        ctypes.POINTER(P)]
        L.hs_builder_destroy.argtypes = [P]
        L.hs_builder_destroy.restype = None
        L.hs_builder_info.argtypes = [P, P]
        L.hs_builder_phase_times.argtypes = [P, P, i32, ctypes.POINTER(i32), ctypes.c_char_p, i32]
        L.hs_builder_download_rows.argtypes = [P, i64, i64, P, P, P, P]
        L.hs_builder_sparse.argtypes = [P, i64, f64, f64]
        L.hs_builder_download_sparse.argtypes = [P] + [P] * 8
        L.hs_builder_dense_moments.argtypes = [P, P, P]
        L.hs_builder_gather_dense.argtypes = [P, P, i64, P, P, P]
        L.hs_builder_dense_encode.argtypes = [P, i32, P, P, i32, P, P, P]
        L.hs_builder_download_dense.argtypes = [P, P, P, P, P]
        L.hs_builder_finish.argtypes = [P, f64, f64, i64, ctypes.POINTER(P)]
        L.hs_index_gather_rows.argtypes = [P, P, i64, P, P, P, P]
        L._hsb_builder_bound = True
    return L


def _p(a):
    return nat.ptr(a)


class DeviceDataset:
    """A HybridDataset resident on one GPU (an hs_builder_t handle)."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = int(device)
        info = np.zeros(8, dtype=np.int64)
        nat.check(_lib().hs_builder_info(self._h, _p(info)))
        self.n, self.d_sparse, self.d_dense, self.nnz = (int(x) for x in info[:4])
        self.dense_fp16 = bool(info[7])

    # -- construction --
    @classmethod
    def generate(cls, law, seed: int, n: int | None = None, row0: int = 0,
                 mean_nnz: float | None = None, device: int = 0, perm_seed: int | None = None):
        """Rows [row0, row0 + n) of the seeded dataset with `law` (synth.HybridLaw)."""
        from .synth import PERM_SEED

        p = GenParams()
        p.n = int(law.n if n is None else n)
        p.d_sparse, p.d_dense = int(law.d_sparse), int(law.d_dense)
        p.mean_nnz = float(law.mean_nnz if mean_nnz is None else mean_nnz)
        p.zipf_s = float(law.zipf_s)
        p.value_law = 1 if law.value_law == "lognormal" else 0
        p.dense_fp16 = int(bool(law.dense_fp16))
        p.seed = int(seed)
        p.perm_seed = int(PERM_SEED if perm_seed is None else perm_seed)
        p.row0 = int(row0)
        h = P()
        nat.check(_lib().hs_builder_generate(ctypes.byref(p), int(device), ctypes.byref(h)))
        return cls(h, device)

    @classmethod
    def upload(cls, dataset: HybridDataset, device: int = 0, dense_fp16: bool = False):
        s = sp.csr_matrix(dataset.sparse, copy=True)  # canonicalised here, not in place
        s.sum_duplicates()
        s.sort_indices()
        indptr = nat.contig(s.indptr, np.int64)
        idx = nat.contig(s.indices, np.uint32)
        val = nat.contig(s.data, np.float32)
        dense = nat.contig(dataset.dense, np.float32) if dataset.d_dense else None
        h = P()
        nat.check(_lib().hs_builder_upload(int(dataset.n), int(dataset.d_sparse),
                                           int(dataset.d_dense), _p(indptr), _p(idx), _p(val),
                                           _p(dense), int(bool(dense_fp16)), int(device),
                                           ctypes.byref(h)))
        return cls(h, device)

    # -- access --
    def download(self, lo: int = 0, hi: int | None = None) -> HybridDataset:
        """Rows [lo, hi) as a host HybridDataset (fp16 dense upcast to f32)."""
        hi = self.n if hi is None else int(hi)
        m = hi - lo
        indptr = np.zeros(m + 1, dtype=np.int64)
        nat.check(_lib().hs_builder_download_rows(self._h, lo, hi, _p(indptr), None, None, None))
        nnz = int(indptr[-1])
        idx = np.empty(max(nnz, 1), dtype=np.uint32)
        val = np.empty(max(nnz, 1), dtype=np.float32)
        dense = np.empty((m, self.d_dense), dtype=np.float32)
        nat.check(_lib().hs_builder_download_rows(self._h, lo, hi, None, _p(idx), _p(val),
                                                  _p(dense) if self.d_dense else None))
        mat = sp.csr_matrix((val[:nnz], idx[:nnz].astype(np.int32), indptr),
                            shape=(m, self.d_sparse))
        mat.has_sorted_indices = True
        return HybridDataset(mat, dense)

    def phase_times(self) -> dict:
        sec = (ctypes.c_double * 32)()
        cnt = ctypes.c_int32()
        names = ctypes.create_string_buffer(2048)
        nat.check(_lib().hs_builder_phase_times(self._h, sec, 32, ctypes.byref(cnt), names, 2048))
        keys = names.value.decode().split(";") if cnt.value else []
        return {k: float(sec[i]) for i, k in enumerate(keys)}

    def build(self, config: HybridIndexConfig | None = None, order_fn=None) -> "GpuBuild":
        """build_index (pipeline.py:119-162) on the GPU; the dataset stays resident."""
        if order_fn is not None:
            raise ValueError("order_fn is not supported by the GPU build (cache_sort only)")
        return GpuBuild(self, config or HybridIndexConfig())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib().hs_builder_destroy(self._h)
            self._h = P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def whiten_from_moments(mean, cov, ridge_scale: float = 1e-6) -> WhiteningTransform:
    """whiten_fit (dense.py:333-348) from the GPU-computed mean and covariance."""
    d = cov.shape[0]
    if np.trace(cov) == 0.0:
        eye = np.eye(d)
        return WhiteningTransform(forward=eye, inverse_t=eye.copy(), mean=mean)
    ridge = ridge_scale * np.trace(cov) / d
    w, V = np.linalg.eigh(cov + ridge * np.eye(d))
    if np.any(w <= 0):
        raise ValueError("covariance is singular even after ridge")
    forward = (V * (w ** -0.5)) @ V.T
    inverse_t = (V * (w ** 0.5)) @ V.T
    return WhiteningTransform(forward=forward, inverse_t=inverse_t, mean=mean)


def sample_rows(n: int, n_subspaces: int, seed: int, sample, n_centers: int) -> np.ndarray:
    """The k-means training rows train_codebooks draws (dense.py:123-129)."""
    if sample is not None and n_centers <= sample < n:
        seqs = np.random.SeedSequence(seed).spawn(1 + n_subspaces)
        rs = np.random.default_rng(seqs[0])
        return np.sort(rs.choice(n, size=sample, replace=False)).astype(np.int64)
    return np.arange(n, dtype=np.int64)


class GpuBuild:
    """Index products of one GPU build (still owned by the builder handle)."""

    def __init__(self, dd: DeviceDataset, config: HybridIndexConfig):
        from .builder import subspace_widths, train_codebooks

        self.dd = dd
        self.config = config
        L = _lib()
        t0 = time.perf_counter()
        if config.data_threshold is not None:
            dm = np.asarray(config.data_threshold, dtype=np.float64)
            if dm.ndim:
                raise ValueError("the GPU build takes a scalar data_threshold")
            top_t, data_min = -1, float(dm)
        else:
            top_t, data_min = (-1 if config.top_t is None else int(config.top_t)), 0.0
            if config.top_t is None:
                data_min = 0.0  # PruneThresholds: data_min defaults to 0 without top_t
        eps = np.asarray(config.residual_threshold, dtype=np.float64)
        if eps.ndim:
            raise ValueError("the GPU build takes a scalar residual_threshold")
        nat.check(L.hs_builder_sparse(dd._h, top_t, data_min, float(eps)))
        info = np.zeros(8, dtype=np.int64)
        nat.check(L.hs_builder_info(dd._h, _p(info)))
        self.n_active, self.nnz_post, self.n_head = int(info[4]), int(info[5]), int(info[6])
        self.codebooks = None
        self.whitening = None
        self.timing = {"sparse_s": time.perf_counter() - t0}
        if dd.d_dense > 0:
            if config.pq_centers != LUT16_CENTERS:
                raise ValueError("the GPU build supports 16-center (4-bit) codebooks only")
            t1 = time.perf_counter()
            d = dd.d_dense
            mean = np.zeros(d, dtype=np.float64)
            wt = None
            if config.use_whitening:
                cov = np.zeros((d, d), dtype=np.float64)
                nat.check(L.hs_builder_dense_moments(dd._h, _p(mean), _p(cov)))
                wt = whiten_from_moments(mean, cov)
            K = config.pq_subspaces or max(1, math.ceil(d / 2))
            widths = subspace_widths(d, K)
            rows = sample_rows(dd.n, K, config.seed, config.train_sample, config.pq_centers)
            x = np.empty((len(rows), d), dtype=np.float64)
            fwd = nat.contig(wt.forward, np.float64) if wt is not None else None
            wm = nat.contig(wt.mean, np.float64) if wt is not None else None
            nat.check(L.hs_builder_gather_dense(dd._h, _p(rows), len(rows), _p(wm), _p(fwd),
                                                _p(x)))
            self.timing["whiten_fit_sample_s"] = time.perf_counter() - t1
            t2 = time.perf_counter()
            cb = train_codebooks(x, K, n_centers=config.pq_centers, n_iters=config.kmeans_iters,
                                 seed=config.seed, sample=None)
            self.timing["kmeans_s"] = time.perf_counter() - t2
            t3 = time.perf_counter()
            sub = nat.contig(cb.subdims, np.int32)
            cen = nat.contig(np.concatenate([c.reshape(-1) for c in cb.centers]), np.float32)
            inv = nat.contig(wt.inverse_t, np.float64) if wt is not None else None
            nat.check(L.hs_builder_dense_encode(dd._h, K, _p(sub), _p(cen), cb.n_centers, _p(wm),
                                                _p(fwd), _p(inv)))
            self.timing["dense_encode_s"] = time.perf_counter() - t3
            self.codebooks, self.whitening = cb, wt
            del widths
        self.timing.update({f"gpu_{k}_s": v for k, v in dd.phase_times().items()})

    # -- parity helpers (download; small n) --
    def sparse_products(self) -> dict:
        dd = self.dd
        order = np.empty(dd.n, dtype=np.int64)
        dims = np.empty(max(self.n_active, 1), dtype=np.uint32)
        ptr = np.empty(self.n_active + 1, dtype=np.int64)
        ids = np.empty(max(self.nnz_post, 1), dtype=np.uint32)
        w = np.empty(max(self.nnz_post, 1), dtype=np.float32)
        mask = np.empty(max((dd.nnz + 31) // 32, 1), dtype=np.uint32)
        hd = np.empty(max(self.n_head, 1), dtype=np.uint32)
        ht = np.empty(max(self.n_head, 1), dtype=np.float32)
        nat.check(_lib().hs_builder_download_sparse(dd._h, _p(order), _p(dims), _p(ptr), _p(ids),
                                                    _p(w), _p(mask), _p(hd), _p(ht)))
        return dict(order=order, dims=dims[:self.n_active].astype(np.int64), ptr=ptr,
                    ids=ids[:self.nnz_post], w=w[:self.nnz_post], dmask=mask,
                    head_dims=hd[:self.n_head], head_thr=ht[:self.n_head])

    def dense_products(self) -> dict:
        dd = self.dd
        if dd.d_dense == 0:
            return {}
        K = self.codebooks.n_subspaces
        packed = np.empty(((K + 1) // 2, dd.n), dtype=np.uint8)
        lo = np.empty(dd.d_dense, dtype=np.float32)
        step = np.empty(dd.d_dense, dtype=np.float32)
        sq = np.empty((dd.n, dd.d_dense), dtype=np.uint8)
        nat.check(_lib().hs_builder_download_dense(dd._h, _p(packed), _p(lo), _p(step), _p(sq)))
        return dict(packed=packed, sq_lo=lo, sq_step=step, sq_codes=sq)

    def host_index(self, dataset: HybridDataset | None = None) -> HybridIndex:
        """The built index as a reference-compatible host HybridIndex."""
        dd = self.dd
        ds = dataset if dataset is not None else dd.download()
        s = self.sparse_products()
        sidx = InvertedIndex(dd.n, dd.d_sparse, s["order"], dims=s["dims"], ptr=s["ptr"],
                             ids=s["ids"], w=s["w"])
        m = sp.csr_matrix(ds.sparse)
        bits = np.unpackbits(s["dmask"].view(np.uint8), bitorder="little")[:m.nnz].astype(bool)
        eps = float(np.asarray(self.config.residual_threshold))
        keep = ~bits & (np.abs(m.data.astype(np.float64)) >= eps)
        # (copies: eliminate_zeros compacts the index arrays in place)
        res = sp.csr_matrix((np.where(keep, m.data, 0).astype(np.float32), m.indices.copy(),
                             m.indptr.copy()), shape=m.shape)
        res.eliminate_zeros()
        res = res[s["order"]].tocsr()
        res.sort_indices()
        dense_index = None
        if dd.d_dense > 0:
            dp = self.dense_products()
            dense_index = DenseIndex(
                codebooks=self.codebooks,
                codes=PQCodes(n=dd.n, n_subspaces=self.codebooks.n_subspaces,
                              n_centers=self.codebooks.n_centers, packed=dp["packed"]),
                residual=ScalarQuantResidual(lo=dp["sq_lo"], step=dp["sq_step"],
                                             codes=dp["sq_codes"]),
                whitening=self.whitening)
        return HybridIndex(config=self.config, n=dd.n, d_sparse=dd.d_sparse, d_dense=dd.d_dense,
                           order=s["order"], sparse_index=sidx, sparse_residual=res,
                           dense_index=dense_index, dataset=ds)

    def finish(self, id_offset: int = 0) -> "DeviceBuiltIndex":
        """Move the products into a search index (the dataset handle is consumed)."""
        dd = self.dd
        h = P()
        builder, dd._h = dd._h, P()
        nat.check(_lib().hs_builder_finish(builder, float(self.config.sparse_weight),
                                           float(self.config.dense_weight), int(id_offset),
                                           ctypes.byref(h)))
        return DeviceBuiltIndex(h, dd, self, id_offset)


class _DeviceDatasetRef:
    """Stands in for `index.dataset` (the raw data lives in the device index)."""

    def __init__(self, n, d_sparse, d_dense):
        self.n, self.d_sparse, self.d_dense = n, d_sparse, d_dense


class _DenseMeta:
    def __init__(self, codebooks, whitening, n):
        self.codebooks = codebooks
        self.whitening = whitening
        self.codes = PQCodes(n=n, n_subspaces=codebooks.n_subspaces,
                             n_centers=codebooks.n_centers, packed=None)
        self.residual = True  # the SQ residual exists on the device


class DeviceBuiltIndex:
    """A HybridIndex whose arrays live on the GPU that built them.

    Exposes what the reference API reads (config, n, d_sparse, d_dense,
    dense_index codebooks / whitening, dataset presence); search_batch and
    search_topk dispatch to the device handle.  Weights are fixed at build.
    """

    def __init__(self, handle, dd: DeviceDataset, build: GpuBuild, id_offset: int):
        from .search import DeviceIndex

        self.config = build.config
        self.n, self.d_sparse, self.d_dense = dd.n, dd.d_sparse, dd.d_dense
        self.dense_index = (_DenseMeta(build.codebooks, build.whitening, dd.n)
                            if dd.d_dense > 0 else None)
        self.dataset = _DeviceDatasetRef(dd.n, dd.d_sparse, dd.d_dense)
        self.id_offset = int(id_offset)
        self.build_timing = dict(build.timing)
        self.n_active, self.nnz_post = build.n_active, build.nnz_post
        self.handle = DeviceIndex.from_handle(handle, dd.device, dd.n, dd.d_sparse, dd.d_dense,
                                              self.config.sparse_weight, self.config.dense_weight)

    def device_handle(self, device: int = 0):
        if device != self.handle.device:
            raise ValueError("a GPU-built index is searched on the GPU that holds it")
        if (float(self.config.sparse_weight) != self.handle.sparse_weight
                or float(self.config.dense_weight) != self.handle.dense_weight):
            raise ValueError("sparse_weight / dense_weight are fixed when a GPU index is built")
        return self.handle

    def memory_bytes(self) -> int:
        return self.handle.memory_bytes()

    def gather_rows(self, ids) -> HybridDataset:
        """Raw rows of local original ids (sampled checks; small m)."""
        ids = nat.contig(ids, np.int64)
        m = len(ids)
        L = _lib()
        indptr = np.zeros(m + 1, dtype=np.int64)
        nat.check(L.hs_index_gather_rows(self.handle.handle, _p(ids), m, _p(indptr), None, None,
                                         None))
        nnz = int(indptr[-1])
        idx = np.empty(max(nnz, 1), dtype=np.uint32)
        val = np.empty(max(nnz, 1), dtype=np.float32)
        dense = np.empty((m, self.d_dense), dtype=np.float32)
        nat.check(L.hs_index_gather_rows(self.handle.handle, _p(ids), m, _p(indptr), _p(idx),
                                         _p(val), _p(dense) if self.d_dense else None))
        mat = sp.csr_matrix((val[:nnz], idx[:nnz].astype(np.int64), indptr),
                            shape=(m, self.d_sparse))
        return HybridDataset(mat, dense)
