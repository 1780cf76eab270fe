#!/bin/bash
# session 3: NCCL one-rank gather test + peer tests; team rounds 4, 2^23-path chunks,
# 6-row composite batches vs base (cfg3 frame, cfg1)
O=gpurun_out/s3b
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_peer.py -q -m gpu > $O/pytest_peer.log 2>&1; echo "exit $?" >> $O/pytest_peer.log
for rep in 1 2; do
for v in base tr4 ch23 cb6; do
  echo "== $v" >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 3 2>&1 | grep -E "iter 2|stages|rror" | tail -2 >> $O/sweep.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 2>&1 | grep -E "iter 3|rror" | tail -1 >> $O/sweep.log
done
done
