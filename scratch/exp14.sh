#!/bin/bash
AURAS_CL_DBG=2 AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp14_8.log 2>&1
nvidia-smi -q -d CLOCK | grep -A4 "^    Clocks$" >> gpurun_out/exp14_8.log
