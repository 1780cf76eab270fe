#!/bin/bash
# Dev aid: scale_probe (world 1 and 8) over libhrt variants in tools/_variants/
for v in "$@"; do
  echo "== $v"; HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/scale_probe.py 10 1,8 2>&1 | tail -2
done
