#!/bin/bash
# shadow entry table: exactness tests, counts, cfg4 timing on / off
O=gpurun_out/s2e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "entry or shadow" > $O/pytest_entry.log 2>&1; echo "exit $?" >> $O/pytest_entry.log
HRT_LIB=tools/_variants/libhrt_cnt.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 > $O/cnt_cfg4.log 2>&1
for rep in 1 2; do
for e in 0 1; do
  echo "== entry $e" >> $O/sweep.log
  HRT_SHADOW_ENTRY=$e timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
done
done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
