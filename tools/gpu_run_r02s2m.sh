#!/bin/bash
# any-hit node fetch split: how many box float4s come through TEX (3 = current)
O=gpurun_out/s2m
mkdir -p $O
for rep in 1 2; do
for v in qt3 qt4 qt5 qt6; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "stage|rror" | tail -1 >> $O/sweep.log
done
done
