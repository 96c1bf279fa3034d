#!/bin/bash
# Round check: gpu tests, per-kernel step times, default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for S in 8 64; do
  for K in l2 cluster; do
    AURAS_MEGA_KERNEL=$K timeout 300 python scratch/step_time.py $S pusht >> gpurun_out/step_time.log 2>&1 || echo "fail S=$S K=$K" >> gpurun_out/step_time.log
  done
done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/step_time.log | grep -v "^x"; cat gpurun_out/bench.json
