#!/bin/bash
# Round-2 session-2 final evidence run (one B200), one commit for every file: GPU tests
# (+ the bounds-checked build), smoke, the field engine's traffic over a cfg3 frame and a
# cfg4 crop frame (converted on the box to profiles/r02s3_field_traffic_*.json, which the
# bench lines then read), the cfg3 / cfg4 bench lines, the reference arm, the 2-rank flow,
# the bench's launch list, per-round rows, full ncu captures and the scale probe.
set -x
O=${O:-gpurun_out/ev4}
mkdir -p $O
C=$(cat .commit 2>/dev/null)
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
M=gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct
timeout 900 ncu --metrics $M --clock-control none -k regex:k_field_ws --csv --log-file $O/field_traffic_cfg3.csv python tools/quick_bench.py 3 1920x1080 8 1 > $O/field_traffic.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_field_ws --csv --log-file $O/field_traffic_cfg4.csv python tools/quick_bench.py 4 960x540 64 1 > $O/field_traffic_cfg4.log 2>&1
E3=$(grep -o "evaluated [0-9,]*" $O/field_traffic.log | tail -1 | tr -dc 0-9)
E4=$(grep -o "evaluated [0-9,]*" $O/field_traffic_cfg4.log | tail -1 | tr -dc 0-9)
python tools/field_traffic.py $O/field_traffic_cfg3.csv $E3 profiles/r02s3_field_traffic_cfg3.json cfg3 $C > $O/ft3.log 2>&1
python tools/field_traffic.py $O/field_traffic_cfg4.csv $E4 profiles/r02s3_field_traffic_cfg4.json cfg4 $C "fws::k_field_ws<64,4,T> (T = 2: encode teams, first 5 march rounds of a chunk), cfg4 960x540 x 64 spp crop frame (1/16 of the 4K frame)" > $O/ft4.log 2>&1
cp profiles/r02s3_field_traffic_cfg3.json profiles/r02s3_field_traffic_cfg4.json $O/ 2>/dev/null
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
HRT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extra > $O/bench_gloo2.json 2> $O/bench_gloo2.err
HRT_LIB=tools/_variants/libhrt_checked.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_checked.log 2>&1; echo "exit $?" >> $O/pytest_gpu_checked.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv $CMD > $O/ncu_list.log 2>&1
timeout 300 python tools/round_profile.py 3 > $O/rounds_cfg3.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 1 -c 1 -o $O/field_round1 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 9 -c 1 -o $O/field_round9 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o $O/step_round2 python tools/quick_bench.py 3 1920x1080 8 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_shadow_trace -s 6 -c 1 -o $O/shtrace_cfg4 python tools/quick_bench.py 4 960x540 64 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_shadow$ -s 6 -c 1 -o $O/shadow_setup_cfg4 python tools/quick_bench.py 4 960x540 64 1 > /dev/null 2>&1
timeout 900 python tools/scale_probe.py 5 1,2,4,8 3 > $O/scale_probe_cfg3.log 2>&1
ls -la $O
