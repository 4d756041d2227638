# Session start state: GPU tests, smoke, default bench (cfg5), cfg3 and cfg4 lines.
O=gpurun_out/state
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --workload cfg3 --steps 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg4 --steps 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 1200 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
for w in 3 4 5; do cut -c1-400 $O/bench_cfg$w.json; tail -2 $O/bench_cfg$w.err; done
