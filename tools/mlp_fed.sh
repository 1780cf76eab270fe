#!/bin/bash
# Measurement: the field engine with the hash-grid gathers replaced by
# position-derived features (HRT_SYNTH_ENCODE=1 build in tools/_variants):
# how fast the tcgen05 MLP pipeline runs when it is fed, vs the real engine.
for v in base synth; do
  lib=tools/_variants/libhrt_$v.so; [ $v = base ] && lib=paper_2309_04581_b200/libhrt.so
  echo "== $v"; HRT_LIB=$lib timeout 300 python tools/quick_bench.py 1 800x800 1 3 2>&1 | tail -2
  HRT_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:k_field_ws -s 3 -c 1 --csv python tools/quick_bench.py 1 800x800 1 1 2>/dev/null | grep -E '"(gpu__|sm__|smsp)' | awk -F'","' '{print $(NF-2), $NF}'
done
