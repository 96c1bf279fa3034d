#!/bin/bash
mkdir -p gpurun_out
for v in "" "AURAS_CL_VARIANT=64" "AURAS_CL_VARIANT=128" "AURAS_CL_DUAL=0" "AURAS_CL_VARIANT=128 AURAS_CL_DUAL=0" "AURAS_CL_VARIANT=64 AURAS_CL_DUAL=0"; do
  for S in 16 64; do echo "[$v] $(env $v timeout 120 python scratch/step_time.py $S pusht 2>&1 | grep step)"; done
done > gpurun_out/s64.txt 2>&1
