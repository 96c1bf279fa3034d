#!/bin/bash
# A/B libraries x hack modes on the S=8 step (step time + all-rank trace)
mkdir -p gpurun_out
for lib in ${LIBS:-default two}; do
  for h in ${HACKS:-0 2}; do
    if [ $lib = default ]; then unset AURAS_LIB; else export AURAS_LIB=$PWD/scratch/libs/$lib.so; fi
    export AURAS_CL_HACK=$h
    timeout 60 python scratch/step_time.py ${S:-8} pusht 2>&1 | grep -E "step|Error" | sed "s|^|$lib h=$h |"
    timeout 60 python scratch/step_time.py ${S:-8} pusht trace > /dev/null 2>&1 && cp gpurun_out/ctrace_${S:-8}.npz gpurun_out/ct_${lib}_h$h.npz
  done
done
