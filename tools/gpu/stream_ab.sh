# k_lut16_stream: parity tests of the streamed path, the probe at the cfg3 / cfg5 row shapes, one ncu capture.
O=gpurun_out/stream_ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_synth_parity.py -m gpu -q -x -k "streamed" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python tools/stream_probe.py 10000000 64 d s > $O/probe_k64.log 2>&1; grep -v "^{" $O/probe_k64.log | cut -c1-200
timeout 600 python tools/stream_probe.py 10000000 128 d s > $O/probe_k128.log 2>&1; grep -v "^{" $O/probe_k128.log | cut -c1-200
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lut16_stream -s 9 -c 1 -o $O/stream_k64 -f \
  python tools/stream_probe.py 10000000 64 d > $O/ncu.log 2>&1; echo "ncu rc=$?"
