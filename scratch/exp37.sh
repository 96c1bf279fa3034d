#!/bin/bash
for L in "" $PWD/paper_2509_09560_b200/libauras_b200_nf.so; do
for S in 8 64; do echo "lib=$L" >> gpurun_out/exp37.log; AURAS_LIB=$L AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms\|x\[" >> gpurun_out/exp37.log; done
done
