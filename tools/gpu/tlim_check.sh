# k_sample_tlim rework: fused-path parity tests, then a short cfg5 line (sample pass time)
O=gpurun_out/tlim
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_synth_parity.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
timeout 1200 python bench.py --steps 3 --no-cpu --qb1 2 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/tlim/bench_cfg5.json'))
print('QPS', d['value'], 'e2e', d['e2e']['value'], 'recall', d['config']['recall_at_10'], 'postings', d['config'].get('index_postings_rank0'))
print(d['kernel_ms_per_step']); print(d['parity'])
PY
tail -3 $O/bench_cfg5.err
