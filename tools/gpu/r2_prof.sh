# full GPU suite, then one ncu capture of the C2 search kernel at the bench point
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/${TAG}_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_prof python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/${TAG}_ncu.log 2>&1
grep variant gpurun_out/${TAG}_perf.log | head -1
