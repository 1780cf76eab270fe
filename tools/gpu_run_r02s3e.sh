#!/bin/bash
# session 3: k_step composite - the rows after the first batch prefetched into L2 up front
# (pf; pf2 with 2-row batches) vs base; cfg3 frame + cfg1, 2 runs each
O=gpurun_out/s3e
mkdir -p $O
for rep in 1 2; do
for v in base pf pf2; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|stages|rror" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
