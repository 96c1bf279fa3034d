#!/bin/bash
# Round-1 measurement pass: gpu tests, smoke, bench lines, ncu launch list + one full capture of the denoise kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest.log 2>&1; echo "rc $?" >> gpurun_out/m_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/m_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err
timeout 600 python bench.py --agents 8 --no-depth1 --no-cpu > gpurun_out/m_bench_a8.json 2> gpurun_out/m_bench_a8.err
timeout 900 python bench.py --no-cpu --no-e2e --no-depth1 --baselines --merged-prefill > gpurun_out/m_bench_extra.json 2> gpurun_out/m_bench_extra.err
timeout 600 python bench.py --config vit_dpt > gpurun_out/m_bench_vitdpt.json 2> gpurun_out/m_bench_vitdpt.err
timeout 600 python bench.py --config vit > gpurun_out/m_bench_vit.json 2> gpurun_out/m_bench_vit.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(?!.*(elementwise|distribution|fill|copy|reduce|cat|index)).*" -c 500 --csv --log-file gpurun_out/m_launches.csv python scratch/prof_run.py 12 > gpurun_out/m_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unet_cluster -s 4 -c 1 -o gpurun_out/m_clus_S8 -f python scratch/step_time.py 8 pusht > gpurun_out/m_ncu8.log 2>&1
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:tf_block --launch-skip 2 -c 1 -o gpurun_out/m_tf_block -f python scratch/tf_ncu.py > gpurun_out/m_ncu_tf.log 2>&1
echo done
