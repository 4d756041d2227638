# ncu --set full of the filter-mode k_lut16_tc (the second k_lut16_tc launch of a step: the first is the sample's totals pass)
O=gpurun_out/prof
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/tc_cfg2 \
  python bench.py --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > $O/ncu_tc_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_tc -s 1 -c 1 -f -o $O/tc_cfg3 \
  python bench.py --no-cpu --workload cfg3 --queries 2048 --qb1 0 --steps 1 --warmup 0 --truth-queries 8 > $O/ncu_tc_cfg3.log 2>&1
