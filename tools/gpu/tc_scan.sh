# k_lut16_tc ms per step vs batch size on the cfg5-law 10^7-point index
for q in "$@"; do
  timeout 600 python bench.py --n 10000000 --queries $q --no-cpu --no-parity --qb1 0 --steps 3 > gpurun_out/scan_$q.out 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/scan_$q.out').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
ops=2.0*1e7*$q*16*128
print('q=$q', round(d['value']), 'tc ms', k.get('lut16_tc'), 'POPS', round(ops/k['lut16_tc']/1e9,2), 'sample', k.get('sample'), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/scan_$q.out
done
