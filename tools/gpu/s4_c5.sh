# micro-variant A/B (AQR_CMIN_GUARD, AQR_PF_FINISH), C5 bench with its cpu_baseline leg, ncu capture of the C5 shard kernel
python tools/perf.py --config C2 --ef 784 --reps 5 --variants default,g1,pff,default > gpurun_out/${TAG}_c2.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c2.log | grep -v summary
python tools/perf.py --config C5 --ef 128 --reps 5 --vbits 10 --variants default,g1,pff,default > gpurun_out/${TAG}_c5.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c5.log | grep -v summary
python bench.py --config C5 --scale 0.02 --nq 500 --steps 2 --warmup 3 > gpurun_out/${TAG}_c5small.json 2> gpurun_out/${TAG}_c5small.log; echo c5small rc=$?
tail -c 600 gpurun_out/${TAG}_c5small.log
python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_C5.json 2> gpurun_out/${TAG}_C5.log; echo C5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_C5.json')); print(d['value'], d['roofline']['frac'], d['cpu_baseline'])"
TAG=${TAG}p bash tools/gpu/c5_prof.sh
