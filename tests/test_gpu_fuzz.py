"""Shape fuzz of the dense scan paths (tools/tc_fuzz.py): random subspace counts
and batch sizes through the filtered stage 1 — tensor-core pass for >= 16
queries, streamed PRMT scan below — against the unfiltered CUDA-core scan.
The chunk count per block, the query-group width and the TMEM ring depth all
follow from the shape, so this walks the kernels' launch-shape space."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [["5", "11"], ["5", "12", "small"]])
def test_scan_shape_fuzz(args):
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "tc_fuzz.py")] + args,
                       capture_output=True, text=True, timeout=900, cwd=REPO)
    assert r.returncode == 0, (r.stdout[-1500:], r.stderr[-1500:])
    assert "0 mismatching" in r.stdout
