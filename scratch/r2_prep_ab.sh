#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/prep_ab.txt
for v in 1 0 1 0; do
  AURAS_DPT_INKERNEL_PREP=$v timeout 600 python bench.py --config vit_dpt --no-cpu --no-depth1 --steps 24 > gpurun_out/pab_$v.json 2>/dev/null
  python - "$v" >> gpurun_out/prep_ab.txt <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/pab_{v}.json").read().strip().splitlines()[-1])
print("inkernel_prep", v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "step_ms", round(d["roofline"]["step_ms"], 4))
PY
done
AURAS_DPT_INKERNEL_PREP=0 timeout 300 python -m pytest tests/test_gpu_dpt.py -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/prep_ab.txt
