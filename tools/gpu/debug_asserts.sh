# compute-sanitizer is closed on this pool: the substitute is the debug library (HS_DCHECK device asserts on
# every posting slice, chunk bound and ring slot; -DHS_DEBUG) under the GPU parity tests of the barrier-heavy paths.
O=gpurun_out/debug
mkdir -p $O
HSB200_LIB_TAG="" HSB200_DEBUG=1 timeout 2400 python -m pytest tests/test_gpu_synth_parity.py tests/test_gpu_parity.py -m gpu -q > $O/pytest_debug_lib.log 2>&1; echo "pytest rc=$?" >> $O/pytest_debug_lib.log
tail -4 $O/pytest_debug_lib.log
