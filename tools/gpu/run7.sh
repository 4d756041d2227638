# dev: k_lut16_tc per-role wait cycles (HSB200_TC_EXP=16), cfg2
mkdir -p gpurun_out
HSB200_TC_EXP=16 python bench.py --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > gpurun_out/b7.json 2> gpurun_out/b7.err
python - <<PY
import re
rows=[l for l in open('gpurun_out/b7.json').read().splitlines() if l.startswith('TCPROF') and 'items=5' in l and 'items=50 ' not in l]
print(len(rows))
for l in rows[-42:]:
    w=int(re.search(r"warp=(\d+)",l).group(1))
    if w in (0,4,8,12,13,16,17,20): print(l)
PY
