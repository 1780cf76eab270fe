#!/bin/bash
# bench.py on cfg3 (new headline), the 2-rank self-spawn on one GPU, GPU tests.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench exit $?" >> gpurun_out/bench_r02b.err
HRT_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 3 --warmup 1 --no-extra > gpurun_out/bench2_r02b.json 2> gpurun_out/bench2_r02b.err; echo "bench2 exit $?" >> gpurun_out/bench2_r02b.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02b.log
