#!/bin/bash
# A/B of env knobs on the step time: usage r2_ab.sh VAR "v1 v2 ..." ; two passes
mkdir -p gpurun_out
VAR=$1; VALS=$2
for pass in 1 2; do for v in $VALS; do for S in 8 64; do
  echo "$VAR=$v $(env $VAR=$v timeout 120 python scratch/step_time.py $S pusht | grep step)"
done; done; done > gpurun_out/ab_$VAR.txt 2>&1
