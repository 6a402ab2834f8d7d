# final build (two-way table only in the CAP > 56 kernels): GPU suite + smoke + C2 bench, launch list + full ncu capture, C5 bench
export TAG=s4final2
bash tools/gpu/r2_full.sh
bash tools/gpu/r2_ncu.sh
python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_C5.json 2> gpurun_out/${TAG}_C5.log; echo C5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_C5.json')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['ids_equal_frac'])"
