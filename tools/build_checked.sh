#!/bin/bash
# Checked build of libhrt.so (device bounds asserts, -DHRT_CHECKS=1) into
# tools/_variants/libhrt_checked.so; run the GPU suite against it with
#   HRT_LIB=tools/_variants/libhrt_checked.so python -m pytest tests -m gpu
cd "$(dirname "$0")/.." || exit 1
mkdir -p tools/_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared -DHRT_CHECKS=1 -o tools/_variants/libhrt_checked.so \
    paper_2309_04581_b200/csrc/hrt.cu paper_2309_04581_b200/csrc/bvh_build.cpp
