#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_tuner.py -x -q > gpurun_out/exp47.log 2>&1; echo "rc $?" >> gpurun_out/exp47.log
