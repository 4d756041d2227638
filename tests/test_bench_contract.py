"""bench.py contract checks that need no GPU: the reference arm (the oracle
port on the host cores, index from oracle/build_oracle.py — no product library
on that arm) prints the driver's JSON line, and the roofline denominators
resolve to recorded measurements."""

from __future__ import annotations

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--replica-n",
         "20000", "--ref-queries", "16", "--steps", "1", "--warmup", "1", "--ref-step-seconds",
         "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["unit"] == "queries/s" and line["value"] > 0
    assert line["config"]["workload"] == "cfg5" and line["config"]["n"] == 100_000_000
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_maps_no_product_library():
    """Run the arm in-process and read /proc/self/maps afterwards: neither
    libhsb200.so nor libhsbuild.so may be loaded (the driver checks the same)."""
    code = (
        "import sys, runpy\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--replica-n', '20000', '--ref-queries', '8',"
        " '--steps', '1', '--warmup', '1', '--ref-step-seconds', '1']\n"
        "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
        "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') if 'libhsb' in l}))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "MAPS []"


def test_roofline_denominators_resolve():
    sys.path.insert(0, REPO)
    import bench

    peak, kind = bench._tensor_peak()
    assert peak > 1000 and isinstance(kind, str)
    hbm, hkind = bench._peaks()
    assert 3000 < hbm < 9000 and isinstance(hkind, str)
    t = bench._traffic("cfg4")
    assert t == {} or t["dram_bytes_per_launch"] > 0
