# Round-end self-check: GPU tests, smoke, default bench line.
O=gpurun_out/check
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -2; cat $O/bench_cfg2.json
