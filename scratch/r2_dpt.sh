#!/bin/bash
mkdir -p gpurun_out
for S in 1 8 64; do timeout 300 python scratch/dpt_step.py $S; done > gpurun_out/dpt_steps.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:auras:: -s 200 -c 150 --csv --log-file gpurun_out/dpt_launches.csv python scratch/dpt_step.py 8 once > /dev/null 2>&1
python profiles/launches.py gpurun_out/dpt_launches.csv 130 > gpurun_out/dpt_launches.txt 2>&1
