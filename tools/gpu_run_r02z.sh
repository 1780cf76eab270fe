#!/bin/bash
# path-major shadow set-up walk (HRT_SHADOW_PATH_MAJOR): coherent tracer queue
O=gpurun_out/z4
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_configs.py -q -x -k "at_scale or shadows" > $O/pytest_scale.log 2>&1; echo "exit $?" >> $O/pytest_scale.log
for v in pm0 pm1 pm0 pm1; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
done
