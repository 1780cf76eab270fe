#!/bin/bash
# samples per path per march round (2): 20 / 24 / 28 vs 32, cfg3 + cfg1 + cfg4 crop
O=gpurun_out/s2r2
mkdir -p $O
for rep in 1 2; do
for v in s32 s20 s24 s28; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" | tail -1 >> $O/sweep.log
done
done
