#!/bin/bash
# encode-team rounds per chunk (with 12 TEX levels in team rounds)
O=gpurun_out/s2q
mkdir -p $O
for rep in 1 2; do
for v in tr3 tr4 tr5 tr7; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
