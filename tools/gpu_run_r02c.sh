#!/bin/bash
# New parity tests (cfg3/cfg4 full scale, cfg2 statistics, furnace, P5 vs oracle),
# compute-sanitizer runs on smoke() and the 2-process peer-frame test.
mkdir -p gpurun_out
nproc > gpurun_out/nproc_r02c.txt
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_stats.py "tests/test_gpu_configs.py::test_gpu_march_limits_vs_oracle" -q -x --durations=20 > gpurun_out/pytest_new_r02c.log 2>&1; echo "exit $?" >> gpurun_out/pytest_new_r02c.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${tool}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/sanitizer_${tool}_smoke.log
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/sanitizer_memcheck_peer.log 2>&1; echo "exit $?" >> gpurun_out/sanitizer_memcheck_peer.log
