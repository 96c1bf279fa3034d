#!/bin/bash
AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp13_8.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_8.json 2>&1 | head -36 >> gpurun_out/exp13_8.log
AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht >> gpurun_out/exp13_8.log 2>&1
AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 64 pusht >> gpurun_out/exp13_8.log 2>&1
