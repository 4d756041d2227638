# cfg5 step vs the candidate budget (HSB200_FUSE_ECAND = expected dense candidates per k1)
O=gpurun_out/ecand
mkdir -p $O
for e in ${ES:-30 40}; do
HSB200_FUSE_ECAND=$e timeout 900 python bench.py --steps 3 --no-cpu --no-parity --qb1 0 --truth-queries 32 > $O/bench_$e.json 2> $O/bench_$e.err
python - $e <<'PY'
import json,sys
d=json.load(open('gpurun_out/ecand/bench_%s.json' % sys.argv[1]))
print('ecand', sys.argv[1], 'QPS', round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'recall', d['config']['recall_at_10'])
print('  ', d['kernel_ms_per_step'])
PY
done
