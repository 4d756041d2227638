"""Seeded synthetic inputs with the BASELINE.json configs' laws.

BASELINE.json names no public dataset; these generators stand in for it
(SURVEY Appendix B): Poisson nnz per row, distinct Zipf(s) dimension ranks
mapped through one seeded bijection shared by data and queries, |N(0,1)| or
lognormal(0,1) values, N(0,1) dense part, rows L2-normalised over the
concatenated vector (f64 norm, f32 storage).  Generation is native
(`hsb_gen_hybrid`, OpenMP, counter-based RNG: identical output for any
thread count).  Data and queries are generated once and the same bytes feed
both the GPU path and the CPU oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .builder import _hostlib, _ptr
from .types import HybridDataset, HybridIndexConfig

PERM_SEED = 0x5EED_1903_0869


@dataclass
class HybridLaw:
    n: int
    d_sparse: int
    d_dense: int
    mean_nnz: float
    zipf_s: float
    value_law: str = "absnormal"  # or "lognormal"
    dense_fp16: bool = False


@dataclass
class BaselineConfig:
    name: str
    data: HybridLaw
    n_queries: int
    query_mean_nnz: float
    index: dict = field(default_factory=dict)     # HybridIndexConfig kwargs
    search: dict = field(default_factory=dict)    # h, overfetch, retain, exact_final_rerank
    note: str = ""

    def index_config(self, **over) -> HybridIndexConfig:
        kw = dict(self.index)
        kw.update(over)
        return HybridIndexConfig(**kw)


# BASELINE.json "configs" mapped onto the reference API
CONFIGS = {
    "cfg1": BaselineConfig(
        "cfg1", HybridLaw(100_000, 1_000_000, 128, 50.0, 1.1, "absnormal"), 1000, 50.0,
        index=dict(pq_subspaces=64, pq_centers=16, kmeans_iters=10, seed=0),
        search=dict(h=10, overfetch=20.0, retain=20.0, exact_final_rerank=True),
        note="configs[0]: small hybrid, top-10 after exact rerank of 200"),
    "cfg2": BaselineConfig(
        "cfg2", HybridLaw(1_000_000, 10_000_000, 256, 100.0, 1.1, "lognormal"), 1000, 100.0,
        index=dict(pq_subspaces=128, pq_centers=16, seed=0),
        search=dict(h=10, overfetch=50.0, retain=50.0, exact_final_rerank=True),
        note="configs[1]: medium hybrid, top-10 after exact rerank of 500"),
    "cfg3": BaselineConfig(
        "cfg3", HybridLaw(10_000_000, 0, 128, 0.0, 1.1), 10_000, 0.0,
        index=dict(pq_subspaces=64, pq_centers=16, seed=0),
        search=dict(h=100, overfetch=1.0, retain=1.0, exact_final_rerank=False),
        note="configs[2]: dense-only LUT16 roofline, top-100 of stage-1 scores"),
    "cfg4": BaselineConfig(
        "cfg4", HybridLaw(10_000_000, 100_000_000, 0, 80.0, 1.05, "absnormal"), 10_000, 30.0,
        index=dict(top_t=None, seed=0),
        search=dict(h=10, overfetch=1.0, retain=1.0, exact_final_rerank=False),
        note="configs[3]: sparse-only posting stream, exact top-10"),
    # generated and built on the GPU (devbuild.py): 10^8 points do not fit the host
    "cfg5": BaselineConfig(
        "cfg5", HybridLaw(100_000_000, 1_000_000_000, 256, 50.0, 1.1, "absnormal",
                          dense_fp16=True), 10_000, 50.0,
        index=dict(pq_subspaces=128, pq_centers=16, seed=0),
        search=dict(h=100, overfetch=10.0, retain=10.0, exact_final_rerank=True),
        note="configs[4]: large hybrid, top-100 after exact rerank of 1000 candidates "
             "(per shard)"),
}


def replica_law(law: HybridLaw, n: int) -> HybridLaw:
    """The same law at n points with the sparse dimensionality scaled by
    n / law.n (so postings per dim, and the pruning they see, stay alike)."""
    d = max(1000, int(round(law.d_sparse * n / law.n))) if law.d_sparse else 0
    return HybridLaw(n, d, law.d_dense, law.mean_nnz, law.zipf_s, law.value_law,
                     law.dense_fp16)


def generate(law: HybridLaw, seed: int, n: int | None = None, mean_nnz: float | None = None,
             perm_seed: int = PERM_SEED) -> HybridDataset:
    """One seeded HybridDataset with the given law (n / mean_nnz overridable)."""
    n = law.n if n is None else int(n)
    mean = law.mean_nnz if mean_nnz is None else float(mean_nnz)
    L = _hostlib()
    indptr = np.zeros(n + 1, dtype=np.int64)
    vl = 1 if law.value_law == "lognormal" else 0
    L.hsb_gen_hybrid(n, law.d_sparse, law.d_dense, mean, law.zipf_s, vl, seed, perm_seed,
                     int(law.dense_fp16), _ptr(indptr), None, None, None)
    nnz = int(indptr[-1])
    indices = np.empty(max(nnz, 1), dtype=np.int32)
    data = np.empty(max(nnz, 1), dtype=np.float32)
    dense = np.empty((n, law.d_dense), dtype=np.float32)
    L.hsb_gen_hybrid(n, law.d_sparse, law.d_dense, mean, law.zipf_s, vl, seed, perm_seed,
                     int(law.dense_fp16), _ptr(indptr), _ptr(indices), _ptr(data), _ptr(dense))
    m = sp.csr_matrix((data[:nnz], indices[:nnz], indptr), shape=(n, law.d_sparse))
    m.has_sorted_indices = True
    return HybridDataset(m, dense)


def make_config(name: str, n: int | None = None, n_queries: int | None = None,
                data_seed: int = 0, query_seed: int = 1):
    """(dataset, queries, BaselineConfig) for a BASELINE config, optionally
    scaled down in n / n_queries with the same laws."""
    cfg = CONFIGS[name]
    ds = generate(cfg.data, data_seed, n=n)
    qs = generate(cfg.data, query_seed, n=cfg.n_queries if n_queries is None else n_queries,
                  mean_nnz=cfg.query_mean_nnz)
    return ds, qs, cfg


def k1_of(cfg: BaselineConfig, n: int) -> int:
    s = cfg.search
    return min(n, math.ceil(s["overfetch"] * s["h"]))
