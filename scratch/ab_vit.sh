for lib in "" scratch/tflibs/vitqb16.so scratch/tflibs/vitqb32.so "" scratch/tflibs/vitqb16.so scratch/tflibs/vitqb32.so; do
  if [ -z "$lib" ]; then unset AURAS_LIB; else export AURAS_LIB=$lib; fi
  python scratch/vit_time.py > /tmp/v.txt; echo "lib=${lib:-base} $(tr '\n' ' ' < /tmp/v.txt)"
done
