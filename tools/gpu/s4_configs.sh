# bench lines of every config on the head build (default invocation per config), then CTA-shape A/B on C2
for c in C1 C3 C4 C5; do
  X=""; [ $c = C4 ] && X="--stream 8000"
  python bench.py --config $c --steps 5 --warmup 3 $X > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.log; echo $c rc=$?
done
python - <<'P'
import json, os
for c in ['C1','C3','C4','C5']:
    try:
        d=json.loads(open('gpurun_out/%s_%s.json' % (os.environ['TAG'], c)).read().strip().splitlines()[-1])
        print(c, d['metric'], d['value'], d['config'].get('ef'), d['config'].get('recall@10'), d['roofline']['frac'], d['roofline']['kernel_ms'], d['ms_per_step'], d['e2e']['value'])
    except Exception as e:
        print(c, 'ERR', e)
P
python tools/perf.py --config C2 --ef 784 --reps 5 --variants default,w8c3,w2c12,w3c8,w6c4,default > gpurun_out/${TAG}_shape.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_shape.log | grep -v summary
python tools/perf.py --config C2 --ef 784 --reps 3 --vbits -2 --variants default > gpurun_out/${TAG}_c2_vbm.log 2>&1
grep -h '"variant"' gpurun_out/${TAG}_c2_vbm.log | grep -v summary
