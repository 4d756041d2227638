# dev: k_lut16_tc phase knock-outs on cfg2 under ncu (per-launch durations)
mkdir -p gpurun_out
for e in ${EXPS:-0 1 2 3 8}; do
  HSB200_TC_EXP=$e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_lut16_tc --csv \
    python bench.py --no-cpu --qb1 0 --steps 2 --warmup 1 --truth-queries 8 > gpurun_out/n6_$e.csv 2> gpurun_out/n6_$e.err
  echo "exp=$e"; grep -o '"k_lut16_tc<[^"]*".*' gpurun_out/n6_$e.csv | awk -F'","' '{print $1, $NF}' | sort | uniq -c | head -8
done
