#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stats.py -q -x > gpurun_out/pytest_stats_r02d.log 2>&1; echo "exit $?" >> gpurun_out/pytest_stats_r02d.log
for v in base pair pair_if1; do
  echo "== $v" >> gpurun_out/sweep_r02d.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2" -A1 >> gpurun_out/sweep_r02d.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3" -A1 >> gpurun_out/sweep_r02d.log
done
HRT_LIB=tools/_variants/libhrt_pair.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/pytest_pair_r02d.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair_r02d.log
