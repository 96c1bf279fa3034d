#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp27_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp27_pytest.log
for S in 8 64; do
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht trace > gpurun_out/exp27_$S.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_$S.json 2>&1 | head -36 >> gpurun_out/exp27_$S.log
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht >> gpurun_out/exp27_$S.log 2>&1
done
