# ncu capture of the cooperative kernel (C3 ef 5888, 1200 queries; C4 ef 2480 bitmap)
python tools/perf.py --config C3 --ef 5888 --nq 1200 --reps 1 --wpq 4 --variants default > gpurun_out/${TAG}_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 1 -c 1 -o gpurun_out/${TAG}_c3_prof python tools/perf.py --config C3 --ef 5888 --nq 1200 --reps 1 --wpq 4 --variants default > gpurun_out/${TAG}_c3_ncu.log 2>&1
echo c3 rc=$?
python tools/perf.py --config C4 --ef 2480 --reps 1 --vbits -2 --wpq 4 --variants default > gpurun_out/${TAG}_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 1 -c 1 -o gpurun_out/${TAG}_c4_prof python tools/perf.py --config C4 --ef 2480 --reps 1 --vbits -2 --wpq 4 --variants default > gpurun_out/${TAG}_c4_ncu.log 2>&1
echo c4 rc=$?
