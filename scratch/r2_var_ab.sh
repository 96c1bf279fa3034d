#!/bin/bash
mkdir -p gpurun_out
for pass in 1 2; do
  for v in base new newnr newpw all3; do
    if [ $v = base ]; then d=scratch/wt_base; elif [ $v = cur ]; then d=.; else d=scratch/var_$v; fi
    echo "$v $(cd $d && timeout 120 python scratch/step_time.py 8 pusht | grep step)"
  done
done > gpurun_out/var_ab.txt 2>&1
