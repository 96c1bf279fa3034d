#!/bin/bash
# one iteration of the kernel work: step time alone (S=8, 64), traced S=8 run, tight parity tests
mkdir -p gpurun_out
export AURAS_CL_HACK=${HACK:-0}
for S in 8 64; do timeout 120 python scratch/step_time.py $S pusht | grep step; done
timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null 2>&1
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3; fi
