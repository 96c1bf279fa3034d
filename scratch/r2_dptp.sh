#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dpt.py -q -x -s -p no:cacheprovider 2>&1 | grep -E "hoisted|DDIM|passed|failed|Error|error|assert" | tail -15 > gpurun_out/dptp.txt
for S in 1 8; do AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py $S; AURAS_DPT_PERSIST=0 timeout 300 python scratch/dpt_step.py $S; done >> gpurun_out/dptp.txt 2>&1
