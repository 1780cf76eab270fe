#!/bin/bash
# level interleave / 80-register cap / encode-only and MLP-only ceilings on cfg3 and cfg1
O=gpurun_out/s2b
mkdir -p $O
for rep in 1 2; do
for v in il0 il1 il0r80 il1r80 smlp_il0 smlp_il1 senc; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
for v in il0 il1r80 smlp_il1 senc; do
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/round_profile.py 3 > $O/rounds_$v.json 2>&1
done
HRT_LIB=tools/_variants/libhrt_il1r80.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_il1r80.log 2>&1; echo "exit $?" >> $O/pytest_il1r80.log
