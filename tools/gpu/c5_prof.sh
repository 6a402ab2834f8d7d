python tools/perf.py --config C5 --ef 128 --reps 2 --vbits 10 --variants default > gpurun_out/${TAG}_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_c5_prof python tools/perf.py --config C5 --ef 128 --reps 2 --vbits 10 --variants default > gpurun_out/${TAG}_c5_ncu.log 2>&1
echo c5 rc=$?
grep variant gpurun_out/${TAG}_c5.log | grep -v summary
