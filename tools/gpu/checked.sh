# the GPU suite and tools/sanitize_run.py against the bounds-checked build (AQR_CHECKS=1):
# compute-sanitizer is closed on this pool
AQR_LIB_VARIANT=checked python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
AQR_LIB_VARIANT=checked python tools/sanitize_run.py > gpurun_out/${TAG}_sanitize.log 2>&1; tail -2 gpurun_out/${TAG}_sanitize.log
grep -c "AQR_CHECKS" gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_sanitize.log
