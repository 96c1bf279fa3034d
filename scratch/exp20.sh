#!/bin/bash
for d in 0 8; do
AURAS_CL_DBG=$d AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp20_$d.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_8.json 2>&1 | head -36 >> gpurun_out/exp20_$d.log
cp gpurun_out/kbtrace_8.npy gpurun_out/kbtrace_8_d$d.npy
done
