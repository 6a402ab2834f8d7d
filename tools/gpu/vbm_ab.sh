python tools/perf.py --config C4 --ef 2480 --reps 3 --variants novh,default,novh,default --vbits -2 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C4 /"
python tools/perf.py --config C1 --ef 64 --reps 5 --variants novh,default --vbits -2 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C1 /"
