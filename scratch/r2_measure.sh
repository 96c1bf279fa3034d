#!/bin/bash
# round-2 evidence: launch list of the bench command (ncu, serialised; our kernels only)
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:auras:: -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-depth1 > gpurun_out/r2_launches_bench.log 2>&1
python profiles/launches.py gpurun_out/r2_launches.csv > gpurun_out/r2_launches.txt 2>&1
