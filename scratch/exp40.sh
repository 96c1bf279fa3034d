#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_dp.py -x -q -k "par_dec" > gpurun_out/exp40.log 2>&1; echo "rc $?" >> gpurun_out/exp40.log
