#!/bin/bash
for S in 8 64; do
AURAS_CL_VARIANT=64 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp31.log
done
AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scratch/step_time.py 8 pusht > gpurun_out/exp31_san.log 2>&1
