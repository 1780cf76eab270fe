#!/bin/bash
# table as a persisting L2 window (HRT_L2_PERSIST) / evict-first last read of the row record (HRT_ROW_EVICT)
mkdir -p gpurun_out
python - <<'PY' >> gpurun_out/sweep_r02w.log
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size, "persist max", getattr(p, "persisting_l2_cache_max_size", None))
PY
for v in l2base l2p rev l2prev l2base l2p; do
  echo "== $v" >> gpurun_out/sweep_r02w.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 3 1920x1080 8 4 2>&1 | grep -E "iter [3]|rror" >> gpurun_out/sweep_r02w.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 1 800x800 1 4 2>&1 | grep -E "iter 3|rror" >> gpurun_out/sweep_r02w.log
  HRT_LIB=tools/_variants/libhrt_$v.so timeout 300 python tools/quick_bench.py 4 960x540 64 2 2>&1 | grep -E "iter 1|rror" >> gpurun_out/sweep_r02w.log
done
