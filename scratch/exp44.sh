#!/bin/bash
for i in 1 2; do
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp44_$i.log 2>&1; echo "rc $?" >> gpurun_out/exp44_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/exp44_smoke.log 2>&1; echo "rc $?" >> gpurun_out/exp44_smoke.log
