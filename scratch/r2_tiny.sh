#!/bin/bash
mkdir -p gpurun_out
AURAS_MEGA_KERNEL=cluster timeout 300 python scratch/tiny_seq.py 4 2>&1 | grep -v CUDAEvent | tail -3 > gpurun_out/tiny_cl.txt
AURAS_MEGA_KERNEL=l2 timeout 300 python scratch/tiny_seq.py 4 2>&1 | grep -v CUDAEvent | tail -3 > gpurun_out/tiny_l2.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python scratch/tiny_seq.py 4 > gpurun_out/tiny_memcheck.txt 2>&1
