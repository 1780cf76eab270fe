#!/bin/bash
# k_step occupancy sweep (HRT_STEP_MINB / HRT_STEP_THREADS / HRT_COMP_BATCH) on cfg3, cfg4 1/16, cfg1
O=gpurun_out/s
mkdir -p $O
for v in m3 m4 m5 m4t256 m4b2 m3 m4; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [3]|rror|stage" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> $O/sweep.log
done
