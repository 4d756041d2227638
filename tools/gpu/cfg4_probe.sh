# cfg4 posting stream: sparse parity tests, a short bench line per library tag (TAGS), optional ncu capture (NCU=1)
O=gpurun_out/cfg4
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or cfg4 or streamed_sparse" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for tag in ${TAGS:-main}; do
T=$tag; [ "$tag" = main ] && T=""
HSB200_LIB_TAG=$T timeout 900 python bench.py --workload cfg4 --steps 3 --no-cpu --qb1 4 > $O/bench_cfg4_$tag.json 2> $O/bench_cfg4_$tag.err
python - $tag <<'PY'
import json,sys
d=json.load(open('gpurun_out/cfg4/bench_cfg4_%s.json' % sys.argv[1]))
r=d['roofline']
print(sys.argv[1], 'cfg4 QPS', d['value'], 'frac', r['frac'], 'ms', r['kernel_ms_per_step'], 'recall', d['config']['recall_at_10'])
PY
done
if [ -n "$NCU" ]; then
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_stage1 -s 2 -c 1 -f -o $O/s1_cfg4 \
  python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu --qb1 0 --truth-queries 4 > $O/ncu.log 2>&1; echo "ncu rc=$?"
fi
