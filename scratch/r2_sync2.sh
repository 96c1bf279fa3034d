#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool synccheck --print-limit 5 --kernel-regex kns=dpt_persist --target-processes all python scratch/dpt_step.py 1 once > gpurun_out/san_dpt_synccheck.txt 2>&1; echo "dpt synccheck rc=$?" > gpurun_out/san2_summary.txt
timeout 1200 $CS --tool racecheck --print-limit 5 --kernel-regex kns=dpt_persist --target-processes all python scratch/dpt_step.py 1 once > gpurun_out/san_dpt_racecheck.txt 2>&1; echo "dpt racecheck rc=$?" >> gpurun_out/san2_summary.txt
timeout 1200 $CS --tool memcheck --print-limit 5 --kernel-regex kns=dpt_persist --target-processes all python scratch/dpt_step.py 1 once > gpurun_out/san_dpt_memcheck.txt 2>&1; echo "dpt memcheck rc=$?" >> gpurun_out/san2_summary.txt
timeout 1200 $CS --tool synccheck --print-limit 5 --kernel-regex kns=unet_cluster --target-processes all python scratch/sanitize_driver.py tiny > gpurun_out/san_tiny_synccheck2.txt 2>&1; echo "tiny synccheck rc=$?" >> gpurun_out/san2_summary.txt
