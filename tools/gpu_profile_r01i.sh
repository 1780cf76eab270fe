#!/bin/bash
# Round-1 (session 3, final: 128-thread k_step and k_paths blocks) evidence run: GPU tests, smoke, bench line, launch list, one full
# capture of a large field-engine launch. Output in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_r01i.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01i.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r01i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r01i.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01i.json 2> gpurun_out/bench_ref_r01i.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01i.csv $CMD > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_ws -s 5 -c 1 -o gpurun_out/field_r01i python tools/quick_bench.py 1 800x800 1 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
timeout 600 python tools/scale_probe.py 10 > gpurun_out/scale_probe_r01i.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w8_r01i.csv python tools/scale_probe.py 2 8 > /dev/null 2>&1
