#!/bin/bash
mkdir -p gpurun_out
for v in base clamp base clamp; do
  echo "== $v" >> gpurun_out/sweep_r02n.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" -A1 >> gpurun_out/sweep_r02n.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> gpurun_out/sweep_r02n.log
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py -q -x > gpurun_out/pytest_clamp_r02n.log 2>&1; echo "exit $?" >> gpurun_out/pytest_clamp_r02n.log
