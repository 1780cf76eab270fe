#!/bin/bash
# final bench lines after the L2-window gather probe (cfg3 default, cfg4 full frame), GPU tests
O=gpurun_out/s2i
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "exit $?" >> $O/bench_cfg4.err
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
