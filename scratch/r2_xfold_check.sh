#!/bin/bash
# Folded cross-attention: sanitizer runs on the persistent DP-T kernel (S = 8, one
# launch), the per-phase trace, then the whole GPU suite.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/xf_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 5 --kernel-name kns=dpt_persist --target-processes all python scratch/dpt_step.py 8 once > gpurun_out/xf_san_$tool.txt 2>&1
  echo "dpt_persist (folded, S=8) $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/xf_san_$tool.txt | tail -1)" >> gpurun_out/xf_summary.txt
done
AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 8 > gpurun_out/xf_trace.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/xf_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xf_summary.txt
