#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:dpt_persist -s 3 -c 1 -f -o gpurun_out/dptp python scratch/dpt_step.py 8 once > gpurun_out/ncu_dptp.log 2>&1
AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 8 > gpurun_out/dptp_trace8.txt 2>&1
AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 1 > gpurun_out/dptp_trace1.txt 2>&1
