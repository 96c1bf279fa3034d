#!/bin/bash
mkdir -p gpurun_out
( time timeout -s ABRT 400 python -X faulthandler bench.py --config vit_dpt --no-cpu --steps 8 --warmup 3 > gpurun_out/bench_vitdpt.json 2> gpurun_out/bench_vitdpt.err ) 2> gpurun_out/bench_vitdpt.time
echo "rc=$?" >> gpurun_out/bench_vitdpt.err
