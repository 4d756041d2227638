mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python bench.py --workload cfg4 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -c 1500 gpurun_out/bench_cfg4.json
python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -c 2500 gpurun_out/bench_cfg2.json
