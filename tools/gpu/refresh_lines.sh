# Refresh the bench lines (cfg2 default, cfg3, cfg4, reference arm) and the cfg2 launch list.
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --workload cfg3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --workload cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_launch.log 2>&1
ls -la $O; tail -c 600 $O/bench_cfg2.json; tail -c 300 $O/bench_cfg4.json; tail -c 300 $O/bench_ref.json
