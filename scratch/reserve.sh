for r in 8 20 36; do
  echo "reserve=$r"; AURAS_MEGA_RESERVE=$r timeout 200 python bench.py --no-cpu --no-e2e --no-depth1 --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['step_ms'])"
done
