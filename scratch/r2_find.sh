#!/bin/bash
mkdir -p gpurun_out
export AURAS_SPIN_TIMEOUT_MS=3000
for i in 1 2 3; do AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/tiny_seq.py 4 2>&1 | grep -v CUDAEvent | tail -1 | cut -c1-60; done > gpurun_out/find.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py tests/test_gpu_robust.py -q -x -p no:cacheprovider 2>&1 | tail -4 >> gpurun_out/find.txt
for S in 1 2 4 8 16 64; do timeout 120 python scratch/step_time.py $S pusht 2>&1 | grep step; done >> gpurun_out/find.txt
