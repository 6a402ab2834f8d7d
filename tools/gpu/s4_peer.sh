# peer-memory exchange: GPU tests, then the C5 bench at small and full scale with --exchange peer (world 1)
python -m pytest tests/test_gpu_peer.py tests/test_gpu_sharded.py tests/test_abi.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -15 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --config C5 --scale 0.02 --nq 500 --steps 2 --warmup 3 --exchange peer --check-exchange --no-cpu > gpurun_out/${TAG}_small.json 2> gpurun_out/${TAG}_small.log; echo small rc=$?
grep -h "peer exchange\|Error\|error" gpurun_out/${TAG}_small.log | tail -5
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --exchange peer --check-exchange --no-cpu > gpurun_out/${TAG}_C5peer.json 2> gpurun_out/${TAG}_C5peer.log; echo C5peer rc=$?
grep -h "peer exchange\|Error\|error" gpurun_out/${TAG}_C5peer.log | tail -5
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_C5peer.json')); print(d['value'], d['ms_per_step'], d['config']['recall@10'], d['config']['exchange'], d['e2e'], d['gpu_launches'])"
