#!/bin/bash
mkdir -p gpurun_out
for pf in 1 0; do
echo "L2PF=$pf" >> gpurun_out/exp1.log
AURAS_CL_L2PF=$pf AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace >> gpurun_out/exp1.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_8.json 2>&1 | head -40 >> gpurun_out/exp1.log
cp gpurun_out/kbtrace_8.npy gpurun_out/kbtrace_8_pf$pf.npy
cp gpurun_out/ctrace_8.json gpurun_out/ctrace_8_pf$pf.json
done
