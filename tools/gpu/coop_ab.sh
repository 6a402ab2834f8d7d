# one-warp vs cooperative (4 warps per query) search kernel on the large-ef / few-query configs
python tools/perf.py --config C4 --ef 2480 --reps 3 --vbits -2 --wpq 1,4 --variants default > gpurun_out/${TAG}_c4.log 2>&1
python tools/perf.py --config C3 --ef 5888 --nq 3000 --reps 1 --vbits -1 --wpq 1,4 --variants default > gpurun_out/${TAG}_c3.log 2>&1
python tools/perf.py --config C1 --ef 64 --reps 20 --vbits 13 --wpq 1,4 --variants default > gpurun_out/${TAG}_c1.log 2>&1
python tools/perf.py --config C2 --ef 784 --reps 3 --vbits -1 --wpq 1,4 --variants default > gpurun_out/${TAG}_c2.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c*.log | grep -v summary
