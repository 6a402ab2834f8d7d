# GPU suite + smoke + C2 bench (the driver's round-end sequence), outputs under gpurun_out/${TAG}_*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print(d['value'], d['config']['ef'], d['config']['recall@10'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['cores'], d['clocks'])"
