python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py --config C3 --ef 5888 --rerank exact --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.log; echo c3 rc=$?
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.log; echo c5 rc=$?
python -c "
import json
for c in ['c3','c5']:
    d=json.load(open('gpurun_out/${TAG}_'+c+'.json')); print(c, d['value'], d['config'].get('ef'), d['config'].get('recall@10'), d['roofline']['frac'], d['ms_per_step'])"
