#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp25_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp25_pytest.log
for b in 8 2 1; do for S in 8 64; do
echo "bch<=$b" >> gpurun_out/exp25.log
AURAS_CL_BCH=$b AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp25.log
done; done
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py 8 pusht trace > gpurun_out/exp25_8.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_8.json 2>&1 | head -36 >> gpurun_out/exp25_8.log
