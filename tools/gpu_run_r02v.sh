#!/bin/bash
# deferred stage hand-off (HRT_DEFER_ST) and row-record L1 prefetch (HRT_ROW_PREFETCH) sweep
mkdir -p gpurun_out
for v in d0 d1 d2 d1pf1 d0pf1 d0 d1 d2; do
  echo "== $v" >> gpurun_out/sweep_r02v.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [3]|rror" >> gpurun_out/sweep_r02v.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> gpurun_out/sweep_r02v.log
done
HRT_LIB=tools/_variants/libhrt_d2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r02v_d2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r02v_d2.log
