O=gpurun_out/build
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_formats.py -m gpu -x -q > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
tail -15 $O/pytest_new.log
timeout 600 python tools/dense_build_probe.py 2000000 > $O/probe.json 2> $O/probe.err; cat $O/probe.json; tail -3 $O/probe.err
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; cat $O/bench_cfg2.json; tail -3 $O/bench_cfg2.err
