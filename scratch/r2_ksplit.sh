#!/bin/bash
# K-split ff2 in the persistent DP-T kernel: parity, trace, bench (each under its own timeout)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dpt.py -x -q -s > gpurun_out/ks_test.log 2>&1; echo rc=$? >> gpurun_out/ks_test.log
AURAS_DPT_TRACE=1 timeout 120 python scratch/dpt_step.py 8 > gpurun_out/ks_trace.txt 2>&1
timeout 400 python bench.py --config vit_dpt --no-cpu > gpurun_out/ks_bench.log 2>&1
