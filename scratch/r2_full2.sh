#!/bin/bash
# full GPU suite + both bench configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/full_gpu.txt 2>&1
tail -3 gpurun_out/full_gpu.txt
timeout 600 python bench.py --config vit_dpt --no-cpu > gpurun_out/bench_vitdpt.json 2> gpurun_out/bench_vitdpt.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
