set -x
python tools/perf.py --config C2 --ef 784 --reps 5 --variants base,shar,default > gpurun_out/ab1_perf.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sq8.py -x -q > gpurun_out/ab1_pytest.log 2>&1
tail -5 gpurun_out/ab1_pytest.log
grep variant gpurun_out/ab1_perf.log
