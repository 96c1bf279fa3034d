#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp30_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp30_pytest.log
AURAS_CL_VARIANT=128 AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp30_pytest128.log 2>&1; echo "rc $?" >> gpurun_out/exp30_pytest128.log
for v in 64 128; do for S in 8 16 32 64; do
echo "v=$v" >> gpurun_out/exp30.log
AURAS_CL_VARIANT=$v AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms\|x\[\|Error\|error" >> gpurun_out/exp30.log
done; done
