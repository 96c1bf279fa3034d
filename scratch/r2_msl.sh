#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/msl.txt
for m in 16 8 4 2 1; do echo "mslices=$m" >> gpurun_out/msl.txt; AURAS_DPT_MSLICES=$m AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 8 2>&1 | grep -E "iteration|total|per phase|op 16 MMA|op 11|op 9:" >> gpurun_out/msl.txt; done
AURAS_DPT_MSLICES=4 timeout 300 python -m pytest tests/test_gpu_dpt.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/msl.txt
