for vb in -1 10 12 -2; do
  python tools/perf.py --config C5 --ef 128 --reps 3 --variants hprobe,default --vbits $vb 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C5 vb=$vb /"
done
for vb in -1 12 13 -2; do
  python tools/perf.py --config C1 --ef 64 --reps 5 --variants hprobe,default --vbits $vb 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C1 vb=$vb /"
done
for vb in -1 12; do
  python tools/perf.py --config C2 --ef 784 --reps 3 --variants default --vbits $vb 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C2 vb=$vb /"
done
