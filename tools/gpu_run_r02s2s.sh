#!/bin/bash
# batch-buffer cap and wavefront chunk size with S = 24
O=gpurun_out/s2s
mkdir -p $O
for rep in 1 2; do
for v in b26s24 b25s24 b27s24 b27s16 p21s24 p23s24; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
