#!/bin/bash
# chunk 2^22 / 2^23 / 2^24 paths x batch cap, cfg3 + cfg4 crop
O=gpurun_out/s2s2
mkdir -p $O
for rep in 1 2 3; do
for v in b26s24 b27s24 p23s24 p23b26 p24s24; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" | tail -1 >> $O/sweep.log
done
done
