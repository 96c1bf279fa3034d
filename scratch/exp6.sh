#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp11_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp11_pytest.log
for pf in 0 1; do
for S in 8 64; do
echo "pf=$pf" >> gpurun_out/exp11_$S.log
AURAS_CL_L2PF=$pf AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht trace >> gpurun_out/exp11_$S.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_$S.json 2>&1 | head -36 >> gpurun_out/exp11_$S.log
cp gpurun_out/kbtrace_$S.npy gpurun_out/kbtrace_${S}_pf$pf.npy; cp gpurun_out/ctrace_$S.json gpurun_out/ctrace_${S}_pf$pf.json
done
done
