#!/bin/bash
AURAS_LIB=$PWD/paper_2509_09560_b200/libauras_b200_na2.so AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht > gpurun_out/exp32.log 2>&1
tail -2 gpurun_out/exp32.log
AURAS_LIB=$PWD/paper_2509_09560_b200/libauras_b200_na2.so AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 tiny >> gpurun_out/exp32.log 2>&1
tail -2 gpurun_out/exp32.log
