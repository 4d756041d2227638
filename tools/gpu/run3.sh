# dev: cfg4 bench only (+ optional env)
mkdir -p gpurun_out
python bench.py --workload cfg4 --no-cpu --qb1 2 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print(d['value'],d['roofline']['frac'],d['kernel_ms_per_step'])"
HSB200_WS=0 python bench.py --workload cfg4 --no-cpu --qb1 2 --steps 3 > gpurun_out/bench_cfg4_nows.json 2> gpurun_out/bench_cfg4_nows.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_nows.json'));print('nows',d['value'],d['roofline']['frac'],d['kernel_ms_per_step'])"
