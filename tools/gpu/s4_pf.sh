# L2 prefetch variants (AQR_PF_PASSES: later gather passes; AQR_PF_ROW: the likely next adjacency row)
python tools/perf.py --config C2 --ef 784 --reps 5 --variants default,pf1,pf2,pfr,pfb,default > gpurun_out/${TAG}_c2.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c2.log | grep -v summary
python tools/perf.py --config C5 --ef 128 --reps 5 --vbits 10 --variants default,pf1,pf2,pfr,pfb > gpurun_out/${TAG}_c5.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c5.log | grep -v summary
python tools/perf.py --config C1 --ef 64 --reps 20 --vbits 13 --variants default,pf1,pfr,pfb > gpurun_out/${TAG}_c1.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c1.log | grep -v summary
python tools/perf.py --config C3 --ef 1024 --reps 2 --variants default,pf1,pfr,pfb > gpurun_out/${TAG}_c3.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c3.log | grep -v summary
