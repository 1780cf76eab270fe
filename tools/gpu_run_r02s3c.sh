#!/bin/bash
# session 3: shadow tracer refill threshold (idle lanes that trigger a warp refill) 2 / 4 / 8 (base) / 16,
# cfg4 960x540 x 64 spp crop frame (shadow stage), 2 runs each
O=gpurun_out/s3c
mkdir -p $O
for rep in 1 2; do
for v in base rl2 rl4 rl16; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|stages|rror" | tail -2 >> $O/sweep.log
done
done
