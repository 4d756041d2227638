# dev: cfg4 stage-1 timing (4096 queries) for A/B library tags (TAGS="a b", "" = default)
mkdir -p gpurun_out
for t in ${TAGS:-""}; do
HSB200_LIB_TAG=$t python bench.py --workload cfg4 --queries ${NQ:-10000} --no-cpu --qb1 0 --steps 2 --warmup 3 --truth-queries 8 > gpurun_out/b14.json 2> gpurun_out/b14_$t.err; python -c "import json;d=json.load(open('gpurun_out/b14.json'));print('cfg4 tag=$t',d['value'],d['roofline']['frac'],d['kernel_ms_per_step']['stage1'])"
done
