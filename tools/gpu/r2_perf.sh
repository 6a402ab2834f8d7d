# A/B of built variants on one index: VARIANTS, CFG, EF (defaults: default / C2 / 784)
python tools/perf.py --config ${CFG:-C2} --ef ${EF:-784} --reps 5 --variants ${VARIANTS:-default} ${PERF_ARGS} > gpurun_out/${TAG:-pf}_perf.log 2>&1
grep '"variant"' gpurun_out/${TAG:-pf}_perf.log | grep -v summary
tail -2 gpurun_out/${TAG:-pf}_perf.log | grep -i error
