#!/bin/bash
AURAS_MEGA_KERNEL=cluster timeout 600 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/exp29_pytest.log 2>&1; echo "rc $?" >> gpurun_out/exp29_pytest.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp29_pytest_all.log 2>&1; echo "rc $?" >> gpurun_out/exp29_pytest_all.log
timeout 600 python bench.py --no-cpu --no-depth1 --steps 24 > gpurun_out/exp29_bench.json 2> gpurun_out/exp29_bench.err
timeout 600 python bench.py --no-cpu --no-depth1 --no-e2e --agents 8 --steps 16 > gpurun_out/exp29_bench_a8.json 2> gpurun_out/exp29_bench_a8.err
