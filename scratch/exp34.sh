#!/bin/bash
AURAS_LIB=$PWD/paper_2509_09560_b200/libauras_b200_tm.so AURAS_CL_VARIANT=64 AURAS_MEGA_KERNEL=cluster timeout 120 python scratch/step_time.py 8 pusht > gpurun_out/exp34.log 2>&1; echo "rc $?" >> gpurun_out/exp34.log
