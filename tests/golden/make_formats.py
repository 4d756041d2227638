"""Generate the on-disk format fixtures (HIDX/HSIX/HDPQ/HYBX) with the REFERENCE.

Run in the dev container (where `/root/reference` exists):

    python tests/golden/make_formats.py

The reference's own `save_index`, `save_inverted_index`, `save_dense_index`
and `save_dataset` (pipeline.py:377-410, sparse.py:369-385, dense.py:433-460,
data.py:270-279) write small files into `tests/golden/formats/`; the
reference's `load_index` + `search_batch` on them give the expected results in
`formats/expect.npz`.  Nothing at test time reads `/root/reference`.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import PIPELINE_CASES, _dataset, _ref, csr_arrays  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")
CASES = ["pipe_default", "pipe_odd", "pipe_sparse_only"]


def main():
    hs = _ref()
    from hybridsearch import data, dense, pipeline, sparse

    os.makedirs(OUT, exist_ok=True)
    expect = {}
    for name in CASES:
        kind, seed, cfg_kw, settings = PIPELINE_CASES[name]
        ds, qs = _dataset(hs, kind, seed)
        cfg = hs.HybridIndexConfig(seed=seed, **cfg_kw)
        idx = hs.build_index(ds, cfg)
        tag = name[len("pipe_"):]
        pipeline.save_index(idx, os.path.join(OUT, f"{tag}.hidx"))
        data.save_dataset(ds, os.path.join(OUT, f"{tag}.hybx"))
        data.save_dataset(qs, os.path.join(OUT, f"{tag}_q.hybx"))
        sparse.save_inverted_index(idx.sparse_index, os.path.join(OUT, f"{tag}.hsix"))
        if idx.dense_index is not None:
            dense.save_dense_index(idx.dense_index, os.path.join(OUT, f"{tag}.hdpq"))
        # what the reference's loaders return from those files
        back = pipeline.load_index(os.path.join(OUT, f"{tag}.hidx"), dataset=ds)
        expect[f"{tag}_order"] = np.asarray(back.order, np.int64)
        expect[f"{tag}_nnz_per_dim"] = np.asarray(back.sparse_index.nnz_per_dim, np.int64)
        for k, v in csr_arrays("res", back.sparse_residual).items():
            expect[f"{tag}_{k}"] = v
        expect[f"{tag}_settings"] = np.array(json.dumps(settings))
        for si, st in enumerate(settings):
            h = st.get("h")
            kw = {k: v for k, v in st.items() if k != "h"}
            res = hs.search_batch(back, qs, h, **kw)
            expect[f"{tag}_s{si}_ids"] = np.stack([r.ids for r in res])
            expect[f"{tag}_s{si}_scores"] = np.stack([r.scores for r in res])
    np.savez_compressed(os.path.join(OUT, "expect.npz"), **expect)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
