#!/bin/bash
# same-box A/B: round-start kernel (scratch/wt_base) vs the working tree, S = 8 and 64, 3 passes
mkdir -p gpurun_out
for pass in 1 2 3; do
  for S in 8 64; do
    echo "base $(cd scratch/wt_base && timeout 120 python scratch/step_time.py $S pusht | grep step)"
    echo "cur  $(timeout 120 python scratch/step_time.py $S pusht | grep step)"
  done
done > gpurun_out/base_ab.txt 2>&1
