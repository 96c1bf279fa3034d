for v in 1 0; do
  echo "interleave=$v"; AURAS_INTERLEAVE_PG=$v timeout 200 python bench.py --no-cpu --no-e2e --no-depth1 --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['step_ms'], d['p99_action_latency_ms'])"
  AURAS_INTERLEAVE_PG=$v AURAS_MEGA_RESERVE=0 timeout 200 python bench.py --no-cpu --no-e2e --no-depth1 --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('res0', d['value'], d['ms_per_step'], d['roofline']['step_ms'])"
done
