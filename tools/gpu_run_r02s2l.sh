#!/bin/bash
# dense-level x-pair records (one 16-B load per x-corner pair)
O=gpurun_out/s2l
mkdir -p $O
for v in dp0 dp1; do HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/dump_frame.py $O/frame_$v.npy >> $O/dump.log 2>&1; done
python -c "import numpy as np; a=np.load('$O/frame_dp0.npy'); b=np.load('$O/frame_dp1.npy'); print('identical', np.array_equal(a,b), abs(a-b).max())" >> $O/dump.log 2>&1
for rep in 1 2; do
for v in dp0 dp1; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
