#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dpt.py -q -x -s -p no:cacheprovider 2>&1 | grep -E "hoisted|DDIM|passed|failed|Error|error|assert" | tail -15 > gpurun_out/dptpf.txt
for pf in ${PFS:-0 1}; do for S in 8; do echo "pf=$pf"; AURAS_DPT_PF=$pf AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py $S; done; done >> gpurun_out/dptpf.txt 2>&1
