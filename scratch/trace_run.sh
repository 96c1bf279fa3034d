#!/bin/bash
mkdir -p gpurun_out
for S in 8 64; do
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/step_time.py $S pusht trace > gpurun_out/trace_$S.log 2>&1
python scratch/ctrace.py gpurun_out/ctrace_$S.json >> gpurun_out/trace_$S.log 2>&1
done
timeout 600 python bench.py --agents 8 --no-depth1 --no-cpu --no-e2e > gpurun_out/bench_a8.json 2>gpurun_out/bench_a8.err
