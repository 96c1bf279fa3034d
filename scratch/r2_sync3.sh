#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool racecheck --print-limit 5 --kernel-name kns=dpt_persist --target-processes all python scratch/dpt_step.py 1 once > gpurun_out/san_dpt_racecheck.txt 2>&1; echo "dpt racecheck rc=$?" > gpurun_out/san3_summary.txt
timeout 1200 $CS --tool racecheck --racecheck-memcheck-mode all --print-limit 5 --kernel-name kns=unet_cluster --target-processes all python scratch/sanitize_driver.py tiny > gpurun_out/san_tiny_racecheck2.txt 2>&1; echo "tiny racecheck rc=$?" >> gpurun_out/san3_summary.txt
