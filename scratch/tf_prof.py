import json, sys, torch, bench
print(json.dumps(bench.merged_prefill_bench(), indent=1))
