for lib in "" scratch/tflibs/spin32.so scratch/tflibs/spin128.so "" scratch/tflibs/spin32.so scratch/tflibs/spin128.so; do
  if [ -z "$lib" ]; then unset AURAS_LIB; else export AURAS_LIB=$lib; fi
  echo "lib=${lib:-base} $(python scratch/step_time.py 8 pusht 2>&1 | grep -i "step ms")"
done
