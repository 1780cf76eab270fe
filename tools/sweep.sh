#!/bin/bash
# Dev aid: quick_bench over libhrt variants: tools/sweep.sh CFG RES SPP v1 v2 ...
cfg=$1; res=$2; spp=$3; shift 3
for v in "$@"; do
    echo "== $v"
    HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py $cfg $res $spp 3 2>&1 | grep -E "iter 2|Error|error" -A1 | head -4
done
