mkdir -p gpurun_out
for h in 0 4 8 12; do
AURAS_CL_HACK=$h timeout 120 python scratch/step_time.py 8 pusht | grep step | sed "s|^|h=$h |"
AURAS_CL_HACK=$h timeout 120 python scratch/step_time.py 8 pusht trace > /dev/null; cp gpurun_out/ctrace_8.npz gpurun_out/ctrace_8_h$h.npz
done
