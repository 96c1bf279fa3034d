#!/bin/bash
AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 600 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 4 -c 1 -o gpurun_out/clus_cur -f python scratch/step_time.py 8 pusht > gpurun_out/exp12.log 2>&1
