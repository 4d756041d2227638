O=gpurun_out/build2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -x -q > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
tail -15 $O/pytest_new.log
timeout 600 python tools/dense_build_probe.py 2000000 > $O/probe.json 2> $O/probe.err; cat $O/probe.json; tail -3 $O/probe.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_pq_encode|k_sq_encode" --csv --log-file $O/ncu_build.csv python tools/dense_build_probe.py 2000000 > $O/ncu.log 2>&1
grep -E "k_pq|k_sq" $O/ncu_build.csv | cut -c1-300 | tail -8
