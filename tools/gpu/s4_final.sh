# final build: GPU suite + smoke + C2 bench, launch list + full ncu capture, C5 bench, then the bounds-checked build
export TAG=s4final
bash tools/gpu/r2_full.sh
bash tools/gpu/r2_ncu.sh
python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_C5.json 2> gpurun_out/${TAG}_C5.log; echo C5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_C5.json')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['ids_equal_frac'])"
python bench.py --config C1 --steps 20 --warmup 3 > gpurun_out/${TAG}_C1.json 2> gpurun_out/${TAG}_C1.log; echo C1 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_C1.json')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['config'].get('ef'), d['config'].get('recall@10'))"
TAG=s4final_checked bash tools/gpu/checked.sh
