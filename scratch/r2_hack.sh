#!/bin/bash
mkdir -p gpurun_out
for h in 0 1 2 3; do
AURAS_CL_HACK=$h timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
python scratch/ctrace2.py gpurun_out/ctrace_8.npz > gpurun_out/ctrace_8_h$h.txt 2>&1
done
