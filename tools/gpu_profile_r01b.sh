#!/bin/bash
# Round-1 (session 2) evidence run: bench line, launch list, per-launch field-engine
# sectors/DRAM, one full capture of a large field-engine launch. Output in gpurun_out/.
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_list.log 2>&1
python tools/quick_bench.py 1 800x800 1 1 > gpurun_out/qb1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_tex_mem_texture.sum --clock-control none -k regex:k_field_ws --csv --log-file gpurun_out/field_launches_r01b.csv python tools/quick_bench.py 1 800x800 1 1 > gpurun_out/qb1_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 5 -c 1 -o gpurun_out/field_r01b python tools/quick_bench.py 1 800x800 1 1 > gpurun_out/ncu_full.log 2>&1
python tools/gather_peak.py > gpurun_out/gather_peak.log 2>&1
ls -la gpurun_out
