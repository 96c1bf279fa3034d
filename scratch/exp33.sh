#!/bin/bash
AURAS_CL_BN=64 AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 120 python scratch/step_time.py 8 pusht > gpurun_out/exp33a.log 2>&1; echo "rc $?" >> gpurun_out/exp33a.log
AURAS_CL_BN=32 AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 120 python scratch/step_time.py 8 pusht > gpurun_out/exp33b.log 2>&1; echo "rc $?" >> gpurun_out/exp33b.log
