#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dpt.py tests/test_gpu_vit.py -q -x -s -p no:cacheprovider 2>&1 | grep -E "hoisted|DDIM|passed|failed|Error|error|assert" | tail -12 > gpurun_out/prep.txt
AURAS_DPT_TRACE=1 timeout 300 python scratch/dpt_step.py 8 2>&1 | grep -E "iteration|total|per phase" >> gpurun_out/prep.txt
timeout 600 python bench.py --config vit_dpt --no-cpu --steps 24 > gpurun_out/bench_vitdpt.json 2> gpurun_out/bench_vitdpt.err
