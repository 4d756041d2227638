# per-role wait cycles of k_lut16_tc (library built with -DHS_TCPROF, tag prof): cfg5-law index of 10^7 points, 192 queries
O=gpurun_out/tcprof
mkdir -p $O
HSB200_LIB_TAG=prof timeout 600 python tools/tcprof_probe.py 10000000 > $O/tcprof.log 2>&1
grep TCPROF $O/tcprof.log | tail -60
