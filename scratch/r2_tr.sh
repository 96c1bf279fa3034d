#!/bin/bash
mkdir -p gpurun_out
for S in 8 64; do timeout 120 python scratch/step_time.py $S pusht 2>&1 | grep step; done > gpurun_out/steps.txt
timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
python scratch/ctrace4.py gpurun_out/ctrace_8.npz > gpurun_out/ctrace4_8.txt 2>&1
