# dev: cfg2 sample-size sweep (HSB200_FUSE_SAMPLE)
mkdir -p gpurun_out
for m in 43008 86016 172032; do
HSB200_FUSE_SAMPLE=$m python bench.py --no-cpu --qb1 0 --truth-queries 8 > gpurun_out/b18.json 2> gpurun_out/b18.err; python -c "import json;d=json.load(open('gpurun_out/b18.json'));k=d['kernel_ms_per_step'];print('m=$m',round(d['value']),round(d['e2e']['value']),k['sample'],k['lut16_tc'],k['fuse'],k['fuse_select'],k['fallback'])"
done
