# full ncu captures of the large-ef search kernels (C3 ef 5888 on 2k queries, C4 ef 2480 with the bitmap)
python tools/perf.py --config C3 --ef 5888 --nq 2000 --reps 1 --variants default > gpurun_out/${TAG}_c3_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_c3_prof python tools/perf.py --config C3 --ef 5888 --nq 2000 --reps 1 --variants default > gpurun_out/${TAG}_c3_ncu.log 2>&1
echo c3 rc=$?
python tools/perf.py --config C4 --ef 2480 --reps 2 --variants default --vbits -2 > gpurun_out/${TAG}_c4_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_c4_prof python tools/perf.py --config C4 --ef 2480 --reps 2 --variants default --vbits -2 > gpurun_out/${TAG}_c4_ncu.log 2>&1
echo c4 rc=$?
grep -h '"variant"' gpurun_out/${TAG}_c3_perf.log gpurun_out/${TAG}_c4_perf.log | grep -v summary
