#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:dpt_persist -s 2 -c 1 -f -o gpurun_out/dptp python scratch/dpt_step.py 8 once > gpurun_out/ncu_dptp.log 2>&1
tail -5 gpurun_out/ncu_dptp.log
