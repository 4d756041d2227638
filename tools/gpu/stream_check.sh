# Streamed LUT16 path: GPU tests, then the cfg3 bench line (qb1 view) and a short cfg5 line.
O=gpurun_out/stream
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
timeout 900 python bench.py --workload cfg3 --no-cpu --steps 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/stream/bench_cfg3.json'))
print(d['value'], d['roofline'].get('qb1'))
PY
tail -3 $O/bench_cfg3.err
