#!/bin/bash
# tile-ring depth, tail-round sizing, small-round samples per path (cfg3 + cfg4 crop + cfg1)
O=gpurun_out/s2t
mkdir -p $O
for rep in 1 2; do
for v in base st4 st8 tt4 tt16 sm32 sm64; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
