# Sustained vs isolated k_lut16_tc: a cfg5-law index of 10^7 points, 1152 queries (six full 192-query groups),
# 20 back-to-back steps with the clock/power samples, then the per-kernel breakdown of the same run.
O=gpurun_out/tc_sustain
mkdir -p $O
timeout 900 python bench.py --n 10000000 --queries ${QUERIES:-1152} --steps 20 --warmup 3 --no-cpu --no-parity --qb1 0 --truth-queries 8 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/tc_sustain/bench.json'))
print('ms/step', d['ms_per_step'], 'QPS', d['value'])
print('kernel ms', d['kernel_ms_per_step'])
print('roof', {k: d['roofline'][k] for k in ('achieved','peak','frac','issue_peak','frac_of_issue_peak') if k in d['roofline']})
print('clocks', d['clocks'])
PY
