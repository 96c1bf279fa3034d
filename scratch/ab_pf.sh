#!/bin/bash
# A/B: L2 prefetch modes of the cluster kernel (AURAS_CL_L2PF), step alone at S=8 / S=64, plus a traced S=8 run per mode
mkdir -p gpurun_out
for rep in 1 2; do
for m in 0 1 2 3; do
  for S in 8 64; do
    AURAS_CL_L2PF=$m timeout 120 python scratch/step_time.py $S pusht | grep "step ms" | sed "s|^|pf=$m |"
  done
done
done
for m in 0 1 2; do
  AURAS_CL_L2PF=$m timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
  cp gpurun_out/ctrace_8.json gpurun_out/ctrace_8_pf$m.json
done
