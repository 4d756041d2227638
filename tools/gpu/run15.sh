# dev: k_lut16_tc ring shape sweep (HSB200_TC_KC / HSB200_TC_SLOTS), cfg2 launch durations
mkdir -p gpurun_out
for v in "0 8" "8 8" "8 10" "0 5"; do
  set -- $v
  HSB200_TC_KC=$1 HSB200_TC_SLOTS=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_lut16_tc --csv \
    python bench.py --no-cpu --qb1 0 --steps 2 --warmup 1 --truth-queries 8 > gpurun_out/n15.csv 2> gpurun_out/n15.err
  grep '^"' gpurun_out/n15.csv | grep "k_lut16_tc<16, 1" | python -c "
import sys,csv
v=sorted(float(r[-1]) for r in csv.reader(sys.stdin))
print('kc=$1 slots=$2', len(v), v[len(v)//2]/1e3 if v else None)"
done
