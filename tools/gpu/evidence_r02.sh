# Round-2 evidence: full GPU test run, smoke, default bench line (cfg5), reference arm, cfg3/cfg4 lines,
# the ncu launch list of the bench command (search kernels only), the tcgen05 issue-rate microbenchmark,
# one ncu --set full capture of the tensor-core filter kernel, the debug-library test run, cfg1/cfg2 lines.
O=gpurun_out/r02
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
[ -x tools/mma_bench2 ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench2 tools/mma_bench2.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > $O/u8_peak.txt; ./tools/mma_bench2 >> $O/u8_peak.txt 2>&1; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $O/u8_peak.txt
timeout 1200 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --workload cfg3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:k_lut|k_fuse|k_stage|k_select|k_sample|k_sparse_b|k_bucket|k_map_dims|k_tlim|k_shard' -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity --qb1 0 --truth-queries 4 > $O/ncu_launch.log 2>&1
echo "ncu rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/tc_cfg5law \
  python bench.py --n 10000000 --no-cpu --no-parity --qb1 0 --steps 1 --warmup 0 --truth-queries 8 --queries 1152 > $O/ncu_tc.log 2>&1
echo "ncu tc rc=$?" >> $O/ncu_tc.log
# compute-sanitizer is closed on this pool (profiles/r02/sanitizer_refused.log): the debug library's device asserts instead
bash tools/gpu/debug_asserts.sh
timeout 900 python bench.py --workload cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --workload cfg1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/u8_peak.txt; cut -c1-300 $O/bench_cfg5.json; cut -c1-300 $O/bench_ref.json; tail -n 2 $O/ncu_launch.log; tail -n 2 $O/ncu_tc.log
