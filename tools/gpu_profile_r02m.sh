#!/bin/bash
# cfg4 shadow tracer (largest launch) and cfg3 k_step: full ncu captures.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_shadow_trace -s 0 -c 1 -o gpurun_out/shtrace0_cfg4_r02m python tools/quick_bench.py 4 960x540 64 1 > gpurun_out/ncu_shtrace0_r02m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/step2_cfg3_r02m python tools/quick_bench.py 3 1920x1080 8 1 > gpurun_out/ncu_step2_r02m.log 2>&1
