#!/bin/bash
# cfg4 with F = 4 encode teams: rounds per chunk run with teams (HRT_TEAM_ROUNDS)
O=gpurun_out/tr
mkdir -p $O
for v in tr3 tr5 tr8 tr3; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
done
