# visited table associativity: direct (h1w), two-way (default), four-way (h4w)
for vb in 10 11 12; do
  python tools/perf.py --config C5 --ef 128 --reps 5 --vbits $vb --variants h1w,default,h4w,default,h4w 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C5 vb=$vb /"
done
python tools/perf.py --config C1 --ef 64 --reps 20 --vbits 13 --variants h1w,default,h4w,default,h4w 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C1 vb=13 /"
AQR_LIB_VARIANT=h4w python -m pytest tests/test_gpu_visited.py tests/test_gpu_configs.py tests/test_gpu_coop.py -x -q 2>&1 | tail -3
