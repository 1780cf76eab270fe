#!/bin/bash
# Dev build of libhrt.so with ptxas resource report (same flags as __graft_entry__.build()).
cd "$(dirname "$0")/../paper_2309_04581_b200" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared -Xptxas -v -o libhrt.so csrc/hrt.cu csrc/bvh_build.cpp 2> /tmp/ptxas.log
rc=$?
grep -E "error|warning" /tmp/ptxas.log | head -20
exit $rc
