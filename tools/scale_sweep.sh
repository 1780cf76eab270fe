#!/bin/bash
# Dev aid: scale_probe over libhrt variants + a launch list of the 1/8 share
for v in base "$@"; do
  echo "== $v"; HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/scale_probe.py 10 1,8 2>&1 | tail -2
done
HRT_LIB=tools/_variants/libhrt_base.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w8.csv python tools/scale_probe.py 2 8 > /dev/null 2>&1
