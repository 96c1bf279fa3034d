#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --target-processes all python scratch/sanitize_driver.py ring > gpurun_out/san_ring_$tool.txt 2>&1; echo "ring $tool rc=$?" >> gpurun_out/san_summary.txt
  timeout 1500 $CS --tool $tool --print-limit 20 --target-processes all python scratch/sanitize_driver.py tiny > gpurun_out/san_tiny_$tool.txt 2>&1; echo "tiny $tool rc=$?" >> gpurun_out/san_summary.txt
done
timeout 1500 $CS --tool memcheck --print-limit 20 --target-processes all python scratch/sanitize_driver.py pusht > gpurun_out/san_pusht_memcheck.txt 2>&1; echo "pusht memcheck rc=$?" >> gpurun_out/san_summary.txt
