# ncu --set full of the filter-mode k_lut16_tc (CTA-pair variant) on a cfg5-law index of 10^7 points
O=gpurun_out/prof
mkdir -p $O
TAG=${1:-tc5}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/$TAG \
  python bench.py --n 10000000 --no-cpu --no-parity --qb1 0 --steps 1 --warmup 0 --truth-queries 8 --queries 1152 > $O/ncu_$TAG.log 2>&1
echo ncu rc=$?
ncu -i $O/$TAG.ncu-rep --page details --csv > $O/$TAG.details.csv 2>/dev/null
python tools/ncu_lines.py $O/$TAG.ncu-rep 60 > $O/$TAG.lines_top.txt 2>&1
python tools/ncu_sass.py $O/$TAG.ncu-rep 60 > $O/$TAG.sass_top.txt 2>&1
