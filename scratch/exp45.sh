#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp45.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_8.json 2>&1 | head -36 >> gpurun_out/exp45.log
python scratch/headtail.py gpurun_out/ctrace_8.json gpurun_out/kbtrace_8.npy >> gpurun_out/exp45.log 2>&1
