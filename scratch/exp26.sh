#!/bin/bash
for pf in 0 2; do for S in 8 64; do
echo "pf=$pf" >> gpurun_out/exp26.log
AURAS_CL_L2PF=$pf AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp26.log
done; done
