#!/bin/bash
# TEX / LSU level split for the F = 4 (cfg4) field: finest N levels through TEX
O=gpurun_out/s2o
mkdir -p $O
for rep in 1 2; do
for v in tx8 tx4 tx12 tx16; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "stage|rror" | tail -1 >> $O/sweep.log
done
done
