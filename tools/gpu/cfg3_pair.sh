# cfg3 (K = 64): single-CTA groups of 160 queries vs CTA pairs with groups of 192
O=gpurun_out/cfg3pair
mkdir -p $O
for p in default 1; do
E=""; [ "$p" = 1 ] && E="HSB200_TC_PAIR=1"
env $E timeout 900 python bench.py --workload cfg3 --steps 3 --no-cpu --qb1 0 > $O/bench_$p.json 2> $O/bench_$p.err
python - $p <<'PY'
import json,sys
d=json.load(open('gpurun_out/cfg3pair/bench_%s.json' % sys.argv[1]))
print('pair', sys.argv[1], 'QPS', round(d['value']), 'tc ms', d['kernel_ms_per_step'].get('lut16_tc'), 'frac', round(d['roofline']['frac'],3), 'recall', d['config']['recall_at_10'], d.get('parity'))
PY
done
