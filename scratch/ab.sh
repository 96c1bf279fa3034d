for lib in "" scratch/tflibs/headab.so "" scratch/tflibs/headab.so; do
  export AURAS_LIB=$lib; [ -z "$lib" ] && unset AURAS_LIB
  python scratch/vit_time.py > /tmp/v.txt; grep "A=1" /tmp/v.txt | sed "s|^|${lib:-new} |"
  timeout 300 python bench.py --config vit_dpt --no-cpu --no-e2e --no-depth1 --steps 16 2>/dev/null > /tmp/b.txt
  python -c "
import json; d=json.loads([l for l in open('/tmp/b.txt') if l.startswith('{')][-1]); print('${lib:-new}', 'dpt', round(d['value'],1), d['roofline']['step_ms'])"
done
