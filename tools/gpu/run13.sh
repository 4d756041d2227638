# dev: GPU tests + cfg4 bench (no CPU arm)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python bench.py --workload cfg4 --no-cpu --qb1 2 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print('cfg4',d['value'],d['e2e']['value'],d['roofline']['frac'],d['config']['recall_at_10'],d['kernel_ms_per_step'])"
