#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp35_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp35_pytest.log
for S in 8 64; do AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht 2>&1 | grep "step ms" >> gpurun_out/exp35.log; done
