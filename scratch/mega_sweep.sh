for cfg in "0 10" "64 10" "256 10" "0 4" "64 6"; do
  set -- $cfg
  echo "spin=$1 adepth=$2"
  AURAS_MEGA_SPIN_NS=$1 AURAS_MEGA_A_DEPTH=$2 timeout 120 python scratch/mega_trace.py 8 2>&1 | grep "step ms" | tail -1
  AURAS_MEGA_SPIN_NS=$1 AURAS_MEGA_A_DEPTH=$2 timeout 120 python scratch/mega_trace.py 8 2>&1 | grep "^  op 15\|^op 15"
done
