# dev: ncu --set full of one single-query (Qb=1) k_stage1<1,0,0> launch, cfg3
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage1 -s ${SKIP:-7} -c 1 -f -o gpurun_out/qb1 \
  python bench.py --workload cfg3 --queries 256 --no-cpu --qb1 6 --steps 1 --warmup 0 --truth-queries 8 > gpurun_out/qb1.log 2>&1; tail -2 gpurun_out/qb1.log
