"""Shared fixtures: golden-fixture loaders and the `gpu` marker."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def csr_from(z, prefix):
    shape = tuple(int(x) for x in z[f"{prefix}_shape"])
    return sp.csr_matrix((z[f"{prefix}_data"], z[f"{prefix}_indices"], z[f"{prefix}_indptr"]),
                         shape=shape)


def golden_config(z, key="config"):
    from paper_1903_08690_b200 import HybridIndexConfig

    return HybridIndexConfig(**json.loads(str(z[key])))


def golden_index(z, prefix="", with_dataset=True, config=None):
    """Rebuild the reference-built index stored in a fixture as our types."""
    from paper_1903_08690_b200 import (
        Codebooks, DenseIndex, HybridDataset, HybridIndex, InvertedIndex, PQCodes,
        ScalarQuantResidual, WhiteningTransform,
    )

    g = lambda k: z[prefix + k]
    cfg = config or golden_config(z, prefix + "config")
    n, ds_, dd = int(g("n")), int(g("d_sparse")), int(g("d_dense"))
    order = g("order")
    sidx = InvertedIndex(n, ds_, order, dims=g("post_dims"), ptr=g("post_ptr"),
                         ids=g("post_ids"), w=g("post_w"))
    res = csr_from(z, prefix + "res")
    di = None
    if int(g("has_dense")):
        sub = g("subdims")
        flat = g("centers_flat")
        l = int(g("n_centers"))
        centers, off = [], 0
        for w in sub:
            centers.append(flat[off:off + l * int(w)].reshape(l, int(w)))
            off += l * int(w)
        cb = Codebooks(subdims=sub, centers=centers)
        codes = PQCodes(n=n, n_subspaces=len(sub), n_centers=l, packed=g("packed"))
        sq = (ScalarQuantResidual(lo=g("sq_lo"), step=g("sq_step"), codes=g("sq_codes"))
              if int(g("has_sq")) else None)
        wt = (WhiteningTransform(forward=g("wh_forward"), inverse_t=g("wh_inverse_t"),
                                 mean=g("wh_mean")) if int(g("has_whitening")) else None)
        di = DenseIndex(codebooks=cb, codes=codes, residual=sq, whitening=wt)
    ds = None
    if with_dataset and "ds_dense" in z.files:
        ds = HybridDataset(csr_from(z, "ds"), z["ds_dense"])
    return HybridIndex(config=cfg, n=n, d_sparse=ds_, d_dense=dd, order=order, sparse_index=sidx,
                       sparse_residual=res, dense_index=di, dataset=ds)


def golden_queries(z):
    from paper_1903_08690_b200 import HybridDataset

    return HybridDataset(csr_from(z, "q"), z["q_dense"])


PIPELINE_CASES = ["pipe_default", "pipe_nowhite", "pipe_unpruned", "pipe_odd", "pipe_dense_only",
                  "pipe_sparse_only"]


@pytest.fixture(params=PIPELINE_CASES)
def pipeline_case(request):
    z = golden(request.param)
    return request.param, z
