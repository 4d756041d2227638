# dev: k_fuse_cands phase knock-outs (HSB200_FUSE_EXP), cfg2 timings only
mkdir -p gpurun_out
for e in 0 1 2 3; do
HSB200_FUSE_EXP=$e python bench.py --no-cpu --qb1 0 --steps 3 --truth-queries 8 > gpurun_out/b10.json 2> gpurun_out/b10_$e.err
python -c "import json;d=json.load(open('gpurun_out/b10.json'));k=d['kernel_ms_per_step'];print('exp=$e',k['fuse'],k['fuse_select'],k['fallback'])"
done
