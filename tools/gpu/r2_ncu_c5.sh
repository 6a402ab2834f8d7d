python tools/perf.py --config C5 --ef 128 --reps 2 --variants default --vbits -1 > gpurun_out/${TAG}_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_prof python tools/perf.py --config C5 --ef 128 --reps 2 --variants default --vbits -1 > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?
