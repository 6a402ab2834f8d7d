# C3 / C4 bench lines on the final build
for c in C3 C4; do
  X=""; [ $c = C4 ] && X="--stream 8000"
  python bench.py --config $c --steps 5 --warmup 3 $X > gpurun_out/s4final_$c.json 2> gpurun_out/s4final_$c.log; echo $c rc=$?
done
python - <<'P'
import json
for c in ['C3','C4']:
    d=json.loads(open('gpurun_out/s4final_%s.json' % c).read().strip().splitlines()[-1])
    print(c, d['metric'], d['value'], d['config'].get('ef'), d['config'].get('recall@10'), d['roofline']['frac'], d['roofline']['kernel_ms'], d['ms_per_step'], d['e2e']['value'], d.get('steady_state'))
P
