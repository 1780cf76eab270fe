#!/bin/bash
O=gpurun_out/s2d
mkdir -p $O
HRT_LIB=tools/_variants/libhrt_cnt.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 > $O/cnt_cfg4.log 2>&1
