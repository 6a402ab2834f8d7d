set -x
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
python bench.py --steps 10 --warmup 3 --ef 784 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.log
python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/r2b_perf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/r2b_prof python tools/perf.py --config C2 --ef 784 --reps 2 --variants default > gpurun_out/r2b_ncu.log 2>&1
echo done
