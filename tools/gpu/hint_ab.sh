python -m pytest tests/test_gpu_parity.py tests/test_gpu_coop.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python tools/perf.py --config C2 --ef 784 --reps 5 --variants default,nohint,default,nohint > gpurun_out/${TAG}_c2.log 2>&1
python tools/perf.py --config C3 --ef 5888 --nq 3000 --reps 1 --variants default,nohint --wpq 1,4 > gpurun_out/${TAG}_c3.log 2>&1
python tools/perf.py --config C4 --ef 2480 --vbits -2 --reps 2 --variants default,nohint > gpurun_out/${TAG}_c4.log 2>&1
python tools/perf.py --config C5 --ef 128 --vbits 10 --reps 5 --variants default,nohint > gpurun_out/${TAG}_c5.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c*.log | grep -v summary
