#!/bin/bash
# samples per round 24 vs 32 at the N-GPU rank shares of cfg3
O=gpurun_out/s2r3
mkdir -p $O
for v in s32 s24; do
  echo "== $v" >> $O/scale.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 900 python tools/scale_probe.py 5 1,2,4,8 3 >> $O/scale.log 2>&1
done
