#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cocc scratch/ubench/cluster_occ.cu && /tmp/cocc > gpurun_out/cluster_occ.txt 2>&1
for S in 1 2 3 4 5 6 7 8 16 64; do timeout 120 python scratch/step_time.py $S pusht | grep step; done > gpurun_out/steps.txt 2>&1
timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
python scratch/ctrace2.py gpurun_out/ctrace_8.npz > gpurun_out/ctrace_8.txt 2>&1
