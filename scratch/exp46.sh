#!/bin/bash
for L in "" $PWD/paper_2509_09560_b200/libauras_b200_wr.so; do
for S in 8 64; do echo "lib=$L" >> gpurun_out/exp46.log; AURAS_LIB=$L AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp46.log; done
done
AURAS_LIB=$PWD/paper_2509_09560_b200/libauras_b200_wr.so AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp46_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp46_pytest.log
