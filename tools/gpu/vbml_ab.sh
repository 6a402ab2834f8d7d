# visited bitmap tested by an L2 load + RED (AQR_VBM_LOAD) vs one atomicOr per neighbour
AQR_LIB_VARIANT=vbmlchk timeout 900 python -m pytest tests/test_gpu_visited.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python tools/perf.py --config C4 --ef 2480 --vbits -2 --reps 3 --variants default,vbml,default,vbml > gpurun_out/${TAG}_c4.log 2>&1
python tools/perf.py --config C1 --ef 64 --vbits -2 --reps 5 --variants default,vbml,default,vbml > gpurun_out/${TAG}_c1.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c*.log | grep -v summary
