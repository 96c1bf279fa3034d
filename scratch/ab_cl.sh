for v in "" "AURAS_CL_BN=32" "AURAS_CL_DUAL=0" "" "AURAS_CL_BN=32" "AURAS_CL_DUAL=0"; do
  echo "${v:-default} $(env $v python scratch/step_time.py 8 pusht 2>&1 | grep -i 'step ms' | awk '{print $NF}')"
done
