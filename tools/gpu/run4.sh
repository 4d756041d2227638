# dev: cfg4 stage-1 variants (env knobs)
mkdir -p gpurun_out
for v in "HSB200_RING_KB=48" "HSB200_RING_KB=64" "HSB200_RING_KB=100"; do
  env $v python bench.py --workload cfg4 --no-cpu --qb1 2 --steps 3 > gpurun_out/b4.json 2> gpurun_out/b4.err; python -c "import json;d=json.load(open('gpurun_out/b4.json'));print('$v',d['value'],d['roofline']['frac'],d['kernel_ms_per_step']['stage1'])"
done
