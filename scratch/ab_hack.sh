#!/bin/bash
mkdir -p gpurun_out
for h in 0 1 2 3; do
  for S in 8 64; do
    AURAS_CL_HACK=$h timeout 120 python scratch/step_time.py $S pusht | grep "step ms" | sed "s|^|hack=$h |"
  done
  AURAS_CL_HACK=$h timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
  cp gpurun_out/ctrace_8.json gpurun_out/ctrace_8_h$h.json
done
