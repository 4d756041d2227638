# cfg5 step vs the stage-1 scratch budget (query chunk = whole tensor-core groups that fit it)
O=gpurun_out/scratch
mkdir -p $O
for g in ${GS:-8 16}; do
HSB200_SCRATCH_GB=$g timeout 900 python bench.py --steps 3 --no-cpu --no-parity --qb1 0 --truth-queries 32 > $O/bench_$g.json 2> $O/bench_$g.err
python - $g <<'PY'
import json,sys
d=json.load(open('gpurun_out/scratch/bench_%s.json' % sys.argv[1]))
print('scratch GB', sys.argv[1], 'QPS', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step'],1), 'launches', d['gpu_launches'], 'recall', d['config']['recall_at_10'])
print('  ', d['kernel_ms_per_step'])
PY
tail -2 $O/bench_$g.err
done
