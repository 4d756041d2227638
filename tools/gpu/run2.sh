# dev: GPU tests, cfg4 + cfg2 bench, one ncu capture of the cfg4 stage-1 kernel
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python bench.py --workload cfg4 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -c 1500 gpurun_out/bench_cfg4.json
python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg2.json'));print(d['value'],d['e2e']['value'],d['kernel_ms_per_step'])"
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage1 -c 1 -f -o gpurun_out/s1_cfg4 \
  python bench.py --workload cfg4 --queries 2048 --steps 1 --warmup 0 --no-cpu --qb1 1 > gpurun_out/ncu_cfg4.log 2>&1; tail -3 gpurun_out/ncu_cfg4.log
fi
