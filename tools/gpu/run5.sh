# dev: k_lut16_tc phase knock-outs on cfg2 (HSB200_TC_EXP), timings only
mkdir -p gpurun_out
for e in 0 1 3 5 9 11 13 15; do
  HSB200_TC_EXP=$e python bench.py --no-cpu --qb1 1 --steps 3 --truth-queries 8 > gpurun_out/b5.json 2> gpurun_out/b5_$e.err
  python -c "import json;d=json.load(open('gpurun_out/b5.json'));print('exp=$e', round(d['kernel_ms_per_step']['lut16_tc'],4), round(d['kernel_ms_per_step']['sample'],4))"
done
