#!/bin/bash
# k_step occupancy / batch sweep, and full captures of the cfg4 shadow stage (set-up + tracer)
O=gpurun_out/y
mkdir -p $O
cp paper_2309_04581_b200/libhrt.so $O/libhrt_y.so
for v in st34 st28 st44 st42 st33 st34; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [3]|rror|stage" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> $O/sweep.log
done
timeout 300 python tools/quick_bench.py 4 960x540 64 2 > $O/cfg4_stages.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_shadow_trace -s 6 -c 1 -o $O/shtrace python tools/quick_bench.py 4 960x540 64 1 > $O/ncu_shtrace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_shadow$" -s 6 -c 1 -o $O/shadow python tools/quick_bench.py 4 960x540 64 1 > $O/ncu_shadow.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg4_launches.csv python tools/quick_bench.py 4 960x540 64 1 > /dev/null 2>&1
ls -la $O
