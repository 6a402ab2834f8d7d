# final captures of the benched binary: (1) the launch list of the bench command (per-launch device
# times, ncu's single-metric pass), (2) one full ncu capture of the C2 search kernel at the bench point
CMD="python bench.py --steps 3 --warmup 3 --ef 784 --no-cpu --no-oracle"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launch_run.log 2>&1
echo launches rc=$?
python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/${TAG}_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/${TAG}_prof python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/${TAG}_ncu.log 2>&1
echo full rc=$?
