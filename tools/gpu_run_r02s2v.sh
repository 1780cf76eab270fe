#!/bin/bash
# host check cadence, tail-mode threshold, small-round threshold (cfg3 N=1 and its 8-GPU share, cfg4 crop, cfg1)
O=gpurun_out/s2v
mkdir -p $O
for rep in 1 2; do
for v in base rc8 rc16 tl4k tl8k sl100 sl400; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/scale_probe.py 3 8 3 2>&1 | grep -E "world 8|rror" | tail -1 >> $O/sweep.log
done
done
