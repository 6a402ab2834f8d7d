python tools/perf.py --config C4 --ef 2480 --reps 3 --vbits -2 --wpq 4 --variants default,coop6,coop7 > gpurun_out/${TAG}_c4.log 2>&1
python tools/perf.py --config C3 --ef 5888 --nq 3000 --reps 1 --vbits -1 --wpq 4 --variants default,coop6,coop7 > gpurun_out/${TAG}_c3.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c*.log | grep -v summary
python tools/perf.py --config C3 --ef 5888 --nq 1200 --reps 1 --wpq 4 --variants default > gpurun_out/${TAG}_c3p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 1 -c 1 -o gpurun_out/${TAG}_c3_prof python tools/perf.py --config C3 --ef 5888 --nq 1200 --reps 1 --wpq 4 --variants default > gpurun_out/${TAG}_c3_ncu.log 2>&1
echo c3 rc=$?
