#!/bin/bash
mkdir -p gpurun_out
for pf in 0 4 5 0 4 5; do for S in 8 64; do echo "pf=$pf $(AURAS_CL_L2PF=$pf timeout 120 python scratch/step_time.py $S pusht | grep step)"; done; done > gpurun_out/pf.txt 2>&1
AURAS_CL_L2PF=4 timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
python scratch/ctrace2.py gpurun_out/ctrace_8.npz > gpurun_out/ctrace_8_pf4.txt 2>&1
