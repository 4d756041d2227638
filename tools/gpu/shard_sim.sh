# One shard of an 8-GPU cfg5 run, simulated on one GPU: the cfg5 law at N = 1.25e7 (d_sparse scaled alike), all 10K queries.
O=gpurun_out/shard
mkdir -p $O
for n in ${NS:-12500000}; do
timeout 900 python bench.py --n $n --steps 3 --no-cpu --no-parity --qb1 0 --truth-queries 16 > $O/bench_$n.json 2> $O/bench_$n.err
python - $n <<'PY'
import json,sys
d=json.load(open('gpurun_out/shard/bench_%s.json' % sys.argv[1]))
print('n', sys.argv[1], 'QPS', round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'recall', d['config']['recall_at_10'])
print('  ', d['kernel_ms_per_step'])
PY
done
