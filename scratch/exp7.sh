#!/bin/bash
for pf in 0 1; do
AURAS_CL_L2PF=$pf AURAS_MEGA_KERNEL=cluster timeout 600 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 4 -c 1 -o gpurun_out/clus_pf$pf -f python scratch/step_time.py 8 pusht > gpurun_out/exp7_pf$pf.log 2>&1
done
