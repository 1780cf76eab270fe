#!/bin/bash
# per-round encode-teams selection: sweep HRT_TEAM_ROUNDS, then parity on the default build
mkdir -p gpurun_out
for v in base team2 team3 team5 base team3; do
  echo "== $v" >> gpurun_out/sweep_r02t.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [23]|rror" >> gpurun_out/sweep_r02t.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> gpurun_out/sweep_r02t.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" >> gpurun_out/sweep_r02t.log
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02t.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r02t.log
