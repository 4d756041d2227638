# dev: GPU tests, cfg2 bench with the totals-only sample threshold vs the exact sample
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
for v in 0 1; do
HSB200_EXACT_SAMPLE=$v python bench.py --no-cpu > gpurun_out/b9_$v.json 2> gpurun_out/b9_$v.err; python -c "import json;d=json.load(open('gpurun_out/b9_$v.json'));print('exact=$v',d['value'],d['e2e']['value'],d['config']['recall_at_10'],d['kernel_ms_per_step'])"
done
