#!/bin/bash
# Round-1 measurement pass: gpu tests, bench lines, ncu launch list + one full capture of the denoise kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest.log 2>&1; echo "rc $?" >> gpurun_out/m_pytest.log
timeout 600 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
timeout 600 python bench.py --agents 8 --no-depth1 --no-cpu > gpurun_out/m_bench_a8.json 2> gpurun_out/m_bench_a8.err
timeout 600 python bench.py --sweep --no-cpu --no-e2e --steps 16 > gpurun_out/m_bench_sweep.json 2> gpurun_out/m_bench_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(?!.*(elementwise|distribution|fill|copy|reduce|cat|index)).*" -c 500 --csv --log-file gpurun_out/m_launches.csv python scratch/prof_run.py 12 > gpurun_out/m_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 4 -c 1 -o gpurun_out/m_clus_S8 -f python scratch/step_time.py 8 pusht > gpurun_out/m_ncu8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 4 -c 1 -o gpurun_out/m_clus_S64 -f python scratch/step_time.py 64 pusht > gpurun_out/m_ncu64.log 2>&1
