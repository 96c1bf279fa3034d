#!/bin/bash
# step times over S, then the tight parity tests and the DP GPU tests
mkdir -p gpurun_out
for S in 1 2 3 4 5 6 7 8 16 64; do timeout 120 python scratch/step_time.py $S pusht 2>&1 | grep -E "step|Error|error" | tail -2; done > gpurun_out/steps.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py tests/test_gpu_vit.py tests/test_gpu_dpt.py -q -s 2>&1 | grep -E "err=|passed|failed|Error|assert" | tail -40 > gpurun_out/parity.txt
