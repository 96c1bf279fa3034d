#!/bin/bash
for v in head v1 cur; do
  if [ $v = cur ]; then L=""; else L=$PWD/paper_2509_09560_b200/libauras_b200_$v.so; fi
  for S in 8 64; do
    echo "$v S=$S" >> gpurun_out/exp15.log
    AURAS_LIB=$L AURAS_CL_L2PF=0 AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp15.log
  done
done
