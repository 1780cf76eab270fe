#!/bin/bash
# session-2 start: state check at HEAD (GPU tests, cfg3 frames, role accounting, ncu of a coherent field round)
O=gpurun_out/s2a
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 > $O/qb_cfg3.log 2>&1
timeout 300 python tools/round_profile.py 3 > $O/rounds_cfg3.log 2>&1
HRT_LIB=tools/_variants/libhrt_wsprof.so timeout 300 python tools/ws_profile.py 3 > $O/wsprof_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 0 -c 1 -o $O/field_round0 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 5 -c 1 -o $O/field_round5 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
ls -la $O
