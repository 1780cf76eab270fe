#!/bin/bash
# any-hit child order (deepest crossing first) and a finer shadow entry table (64^3 x 16^2)
O=gpurun_out/s2f
mkdir -p $O
for v in deep_cnt g64p16_cnt; do
  echo "== $v" >> $O/cnt.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 1 2>&1 | grep -E "shadow trace|rror" | tail -1 >> $O/cnt.log
done
for rep in 1 2; do
for v in base deep g64p16; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
done
done
HRT_LIB=tools/_variants/libhrt_deep.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_scale.py -q -x -k "entry or shadow or any" > $O/pytest_deep.log 2>&1; echo "exit $?" >> $O/pytest_deep.log
