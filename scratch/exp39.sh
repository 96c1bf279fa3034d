#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_toy.py -x -q -k "par_dec" > gpurun_out/exp39.log 2>&1; echo "rc $?" >> gpurun_out/exp39.log
