#!/bin/bash
# k_paths_bounce (per-bounce compacted closest-hit launches) vs the fused per-path k_paths
mkdir -p gpurun_out
for v in pb0 pb1 pb0 pb1; do
  echo "== $v" >> gpurun_out/sweep_r02x.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [3]|rror|stage" >> gpurun_out/sweep_r02x.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> gpurun_out/sweep_r02x.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" >> gpurun_out/sweep_r02x.log
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02x.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r02x.log
