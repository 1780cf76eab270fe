#!/bin/bash
# shadow set-up: row and path loads issued together (hs) vs before (hs0)
O=gpurun_out/s2n
mkdir -p $O
for rep in 1 2; do
for v in hs0 hs; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "stage|rror" | tail -1 >> $O/sweep.log
done
done
HRT_LIB=tools/_variants/libhrt_hs.so timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "entry or shadow" > $O/pytest_hs.log 2>&1; echo "exit $?" >> $O/pytest_hs.log
