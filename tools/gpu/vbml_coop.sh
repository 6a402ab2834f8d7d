AQR_LIB_VARIANT=chk timeout 900 python -m pytest tests/test_gpu_coop.py tests/test_gpu_visited.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python tools/perf.py --config C4 --ef 2480 --vbits -2 --reps 3 --variants default --wpq 1,4 > gpurun_out/${TAG}_c4.log 2>&1
python tools/perf.py --config C4 --ef 2480 --vbits -2 --nq 8000 --reps 2 --variants default --wpq 1,4 > gpurun_out/${TAG}_c4s.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c*.log | grep -v summary
