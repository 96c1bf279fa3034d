#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dpt.py -q -x -s -p no:cacheprovider 2>&1 | grep -E "hoisted|DDIM|passed|failed|Error|error|assert" | tail -15 > gpurun_out/dptdbg.txt
for d in ${DBGS:-0}; do for pf in 1; do echo "dbg=$d pf=$pf"; AURAS_DPT_PF=$pf AURAS_DPT_DBG=$d AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 8 2>&1 | grep -vE "^  op (10|11|12|13|14)[: ] *(prod|B|A|MMA|epilogue)"; done; done >> gpurun_out/dptdbg.txt 2>&1
echo "no trace:" >> gpurun_out/dptdbg.txt
for S in 1 8; do timeout 300 python scratch/dpt_step.py $S; done >> gpurun_out/dptdbg.txt 2>&1
