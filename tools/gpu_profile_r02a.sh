#!/bin/bash
# Round-2 first evidence run: cfg3 (the metric's 1080p config) stage profile,
# per-launch list of one frame, field-engine L2 traffic over the frame, and
# one full capture of a large field-engine launch and of k_step.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_r02a.txt 2>&1
timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 > gpurun_out/qb_cfg3_r02a.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_r02a.csv python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_field_ws --csv --log-file gpurun_out/field_traffic_cfg3_r02a.csv python tools/quick_bench.py 3 1920x1080 8 1 > gpurun_out/ft_cfg3_r02a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 8 -c 1 -o gpurun_out/field_cfg3_r02a python tools/quick_bench.py 3 1920x1080 8 1 > gpurun_out/ncu_full_field_r02a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 8 -c 1 -o gpurun_out/step_cfg3_r02a python tools/quick_bench.py 3 1920x1080 8 1 > gpurun_out/ncu_full_step_r02a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_paths -c 1 -o gpurun_out/paths_cfg3_r02a python tools/quick_bench.py 3 1920x1080 8 1 > gpurun_out/ncu_full_paths_r02a.log 2>&1
ls -la gpurun_out | tail -20
