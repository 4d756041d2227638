# dev: GPU tests + cfg2 / cfg3 bench (no CPU arm)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg2.json'));print('cfg2',d['value'],d['e2e']['value'],d['roofline']['frac'],d['kernel_ms_per_step'])"
if [ "${CFG3:-1}" = 1 ]; then
python bench.py --no-cpu --workload cfg3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg3.json'));print('cfg3',d['value'],d['e2e']['value'],d['roofline']['frac'],d['kernel_ms_per_step'])"
fi
