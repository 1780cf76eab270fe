#!/bin/bash
# final state check: GPU tests, smoke, bench lines (cfg3 default, cfg4, reference arm), 2-rank flow
O=gpurun_out/fin
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "exit $?" >> $O/bench_cfg4.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
HRT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extra > $O/bench_gloo2.json 2> $O/bench_gloo2.err
