#!/bin/bash
# Dev aid: build libhrt.so variants with extra -D flags into tools/_variants/
# usage: tools/variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
cd "$(dirname "$0")/.." || exit 1
mkdir -p tools/_variants
pids=()
while [ $# -ge 2 ]; do
    name=$1; flags=$2; shift 2
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
        -Xcompiler -fPIC -shared $flags -o tools/_variants/libhrt_$name.so \
        paper_2309_04581_b200/csrc/hrt.cu paper_2309_04581_b200/csrc/bvh_build.cpp &
    pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
ls tools/_variants
exit $rc
