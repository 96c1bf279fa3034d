#!/bin/bash
AURAS_CL_DBG=1 AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp10_8.log 2>&1
