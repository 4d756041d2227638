# dev: per-launch durations of the cfg2 step (ncu launch list)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > gpurun_out/n11.csv 2> gpurun_out/n11.err
grep '^"' gpurun_out/n11.csv | python -c "
import sys,csv
from collections import defaultdict
d=defaultdict(list)
for r in csv.reader(sys.stdin):
    if len(r)<10 or r[0]=='ID': continue
    d[r[4][:60]].append(float(r[-1]))
for k,v in sorted(d.items(), key=lambda kv:-sum(kv[1])): print(round(sum(v)/1e3,3), len(v), round(max(v)/1e3,3), k)
" | head -30
