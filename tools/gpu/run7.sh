# dev: k_lut16_tc per-role wait cycles (HSB200_TC_EXP=16)
mkdir -p gpurun_out
for w in cfg2 cfg3; do
HSB200_TC_EXP=16 python bench.py --workload $w --queries 2000 --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > gpurun_out/b7_$w.json 2> gpurun_out/b7_$w.err
python - <<PY
import re
rows=[l for l in open('gpurun_out/b7_$w.json').read().splitlines() if l.startswith('TCPROF')]
print('$w', len(rows))
for l in rows[-42:]:
    w=int(re.search(r"warp=(\d+)",l).group(1))
    if w in (0,1,4,5,8,12,16,17,20): print(l)
PY
done
