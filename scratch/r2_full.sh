#!/bin/bash
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/gputest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpt_persist -s 3 -c 1 -o gpurun_out/prof_dpt python scratch/dpt_step.py 8 > gpurun_out/ncu_dpt_log.txt 2>&1
