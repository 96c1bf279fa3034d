#!/bin/bash
mkdir -p gpurun_out
timeout 120 python scratch/step_time.py 64 pusht trace > /dev/null 2>&1
python scratch/ctrace2.py gpurun_out/ctrace_64.npz > gpurun_out/ctrace_64.txt 2>&1
