#!/bin/bash
# cfg4 field-engine traffic capture (every k_field_ws launch of a 960x540x64 crop frame), then the cfg4 bench line
O=gpurun_out/s2h
mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_field_ws --csv --log-file $O/field_traffic_cfg4.csv python tools/quick_bench.py 4 960x540 64 1 > $O/field_traffic_cfg4.log 2>&1
echo "exit $?" >> $O/field_traffic_cfg4.log
