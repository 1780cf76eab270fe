#!/bin/bash
# session 3: encode teams per coherent round, T = 2 (base) vs T = 4 (four teams of 4 warps,
# each thread all 16 levels of its row, one level in flight, four tiles per SM); team rounds
# 3 / 5 / all; TEX levels 12 / 16. cfg3 frame + field, cfg1, images compared with base.
O=gpurun_out/s3a
mkdir -p $O
for rep in 1 2; do
for v in base t4 t4r5 t4all t4x16; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|stages|rror" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
for v in t4 t4r5; do
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/parity_$v.log 2>&1; echo "exit $?" >> $O/parity_$v.log
done
