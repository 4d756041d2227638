# dev: ncu --set full of one kernel launch in the cfg2 bench (KERNEL regex)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KERNEL} -s ${SKIP:-0} -c 1 -f -o gpurun_out/${NAME} \
  python bench.py --no-cpu --qb1 0 --steps 1 --warmup 0 --truth-queries 8 ${ARGS} > gpurun_out/${NAME}.log 2>&1; tail -2 gpurun_out/${NAME}.log
