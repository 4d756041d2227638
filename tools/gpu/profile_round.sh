# Round evidence: bench lines (cfg2 default + cfg3 + cfg4 + reference arm),
# the cfg2 launch list, and ncu --set full captures of the dominant kernels.
# Output: gpurun_out/prof/ (copied into profiles/<round>/ by hand).
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --workload cfg3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --workload cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/tc_cfg2 \
  python bench.py --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > $O/ncu_tc_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/tc_cfg3 \
  python bench.py --no-cpu --workload cfg3 --queries 2048 --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > $O/ncu_tc_cfg3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage1 -c 1 -f -o $O/s1_cfg4 \
  python bench.py --no-cpu --workload cfg4 --queries 2048 --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > $O/ncu_s1_cfg4.log 2>&1
ls -la $O
