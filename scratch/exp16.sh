#!/bin/bash
for d in 0 4; do for S in 8 64; do
echo "dbg=$d S=$S" >> gpurun_out/exp16.log
AURAS_CL_DBG=$d AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms\|x\[" >> gpurun_out/exp16.log
done; done
