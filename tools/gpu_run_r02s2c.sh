#!/bin/bash
# cp.async row-record prefetch in the encode warps (rs) vs base (il0)
O=gpurun_out/s2c
mkdir -p $O
for rep in 1 2; do
for v in il0 rs; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|rror" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" | tail -1 >> $O/sweep.log
done
done
HRT_LIB=tools/_variants/libhrt_rs.so timeout 300 python tools/round_profile.py 3 > $O/rounds_rs.json 2>&1
HRT_LIB=tools/_variants/libhrt_rs.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_rs.log 2>&1; echo "exit $?" >> $O/pytest_rs.log
