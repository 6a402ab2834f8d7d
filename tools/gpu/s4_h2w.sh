# two-way set-associative 16-bit-tag visited table (AQR_HASH_2WAY) vs direct-mapped
for vb in 9 10 11; do
  python tools/perf.py --config C5 --ef 128 --reps 5 --vbits $vb --variants default,h2w,default,h2w 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C5 vb=$vb /"
done
for vb in 12 13; do
  python tools/perf.py --config C1 --ef 64 --reps 20 --vbits $vb --variants default,h2w,default,h2w 2>&1 | grep '"variant"' | grep -v summary | sed "s/^/C1 vb=$vb /"
done
AQR_LIB_VARIANT=h2w python -m pytest tests/test_gpu_visited.py tests/test_gpu_configs.py tests/test_gpu_coop.py -x -q 2>&1 | tail -3
