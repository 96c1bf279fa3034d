#!/bin/bash
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/exp38_smoke.log 2>&1; echo "rc $?" >> gpurun_out/exp38_smoke.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/exp38_ref.json 2> gpurun_out/exp38_ref.err; echo "rc $?" >> gpurun_out/exp38_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu --no-depth1 > gpurun_out/exp38_trun.json 2> gpurun_out/exp38_trun.err; echo "rc $?" >> gpurun_out/exp38_trun.err
