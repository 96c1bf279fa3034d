#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 3 -c 1 -o gpurun_out/prof_r2_S8 python scratch/step_time.py 8 pusht > gpurun_out/ncu_log.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 3 -c 1 -o gpurun_out/prof_r2_S64 python scratch/step_time.py 64 pusht >> gpurun_out/ncu_log.txt 2>&1
