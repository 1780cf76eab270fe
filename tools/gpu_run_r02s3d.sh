#!/bin/bash
# session 3: bottom 8 / 16 / 24 entries of the any-hit tracer's stack in shared memory vs all
# local (base); cfg4 960x540 x 64 spp crop frame, 2 runs each; shadow tests on ss16
O=gpurun_out/s3d
mkdir -p $O
for rep in 1 2; do
for v in base ss8 ss16 ss24; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|stages|rror" | tail -2 >> $O/sweep.log
done
done
HRT_LIB=tools/_variants/libhrt_ss16.so timeout 900 python -m pytest tests -m gpu -q -k "shadow or any_hit or cfg4" > $O/pytest_ss16.log 2>&1; echo "exit $?" >> $O/pytest_ss16.log
