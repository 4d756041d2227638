# dev: per-launch durations of the Qb=1 path (cfg3)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  python bench.py --workload cfg3 --queries 256 --no-cpu --qb1 6 --steps 1 --warmup 1 --truth-queries 8 > gpurun_out/n16.csv 2> gpurun_out/n16.err
grep '^"' gpurun_out/n16.csv | tail -60 | python -c "
import sys,csv
for r in csv.reader(sys.stdin):
    if len(r)<10 or r[0]=='ID': continue
    print(r[4][:50], r[-3], r[-1])
" | tail -24
