# Round-2 evidence: full GPU test run (no -x), smoke, default bench line (cfg5),
# reference arm, and the ncu launch list of the same bench command (search
# kernels only: the generator/build launches would use up the capture count).
O=gpurun_out/r02
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:k_lut|k_fuse|k_stage|k_select|k_sample|k_sparse_b|k_bucket|k_map_dims|k_tlim|k_shard' -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity --qb1 0 --truth-queries 4 > $O/ncu_launch.log 2>&1
echo "ncu rc=$?" >> $O/ncu_launch.log
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; cut -c1-600 $O/bench_cfg5.json; cut -c1-600 $O/bench_ref.json; tail -2 $O/ncu_launch.log
