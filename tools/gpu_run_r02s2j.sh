#!/bin/bash
# per-round engine time: teams (base) vs T = 1 everywhere vs T = 1 + rolling pipeline everywhere
O=gpurun_out/s2j
mkdir -p $O
for v in base t0 t0roll; do
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/round_profile.py 3 > $O/rounds_$v.json 2>&1
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/round_profile.py 1 > $O/rounds_cfg1_$v.json 2>&1
done
