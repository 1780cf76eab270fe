#!/bin/bash
# cfg4: field-engine L2 traffic over one 960x540x64 frame (-> profiles/r02_field_traffic_cfg4.json),
# encode teams for F = 4 (HRT_TEAMS_F4), F = 4 gather probe test, then the cfg4 bench line
O=gpurun_out/t4
mkdir -p $O
C=$(cat $O/../.commit_hint 2>/dev/null || echo unknown)
timeout 300 python -m pytest tests/test_gpu_measure.py -q -x > $O/pytest_measure.log 2>&1; echo "exit $?" >> $O/pytest_measure.log
for v in tf0 tf4 tf0 tf4; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror|stage" | tail -2 >> $O/sweep.log
done
timeout 1200 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_field_ws --csv --log-file $O/field_traffic_cfg4.csv python tools/quick_bench.py 4 960x540 64 1 > $O/field_traffic.log 2>&1
N=$(grep -o "evaluated [0-9,]*" $O/field_traffic.log | head -1 | tr -d ',' | awk '{print $2}')
python tools/field_traffic.py $O/field_traffic_cfg4.csv $N $O/r02_field_traffic_cfg4.json cfg4 "$C" "fws::k_field_ws<64,4,1> (cfg4 at 960x540x64, 1/16 of the 4K frame)" > $O/field_traffic_json.log 2>&1
cp $O/r02_field_traffic_cfg4.json profiles/
timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
