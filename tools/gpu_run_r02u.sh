#!/bin/bash
# current build: bench line, full captures of a coherent (teams) and an incoherent field round and k_step round 2
O=gpurun_out/u
mkdir -p $O
cp paper_2309_04581_b200/libhrt.so $O/libhrt_u.so
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 1 -c 1 -o $O/field_round1 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 5 -c 1 -o $O/field_round5 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o $O/step_round2 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
ls -la $O
