# A/B of tagged library builds / env knobs on the cfg5-law 10^7-point index:
#   bash tools/gpu/ab_tc.sh base pg0 "base:HSB200_TC_PAIR=0" ...
for spec in "$@"; do
  t=${spec%%:*}; envs=""; [ "$spec" != "$t" ] && envs=${spec#*:}
  if [ "$t" = "base" ]; then tt=""; else tt="$t"; fi
  name=$(echo "$spec" | tr ':= ' '___')
  env HSB200_LIB_TAG=$tt $envs timeout 600 python bench.py --n 10000000 --queries ${QUERIES:-2304} --no-cpu --no-parity --qb1 0 --steps 3 > gpurun_out/ab_$name.out 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$name.out').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']; print('$spec', round(d['value']), 'tc', k.get('lut16_tc'), 'sample', k.get('sample'), 'fuse', k.get('fuse'), 'sel', k.get('fuse_select'))" || tail -3 gpurun_out/ab_$name.out
done
