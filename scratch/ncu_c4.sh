mkdir -p gpurun_out
# ViT frame (1 image): the linear-layer GEMM, token epilogue and attention; DP-T iteration kernels
PYTHONPATH=. ncu --set full --clock-control none -k "regex:conv_gemm_tc$|vit_attention|tok_epilogue" -s 60 -c 3 -o gpurun_out/c4_vit -f python scratch/vit_once.py > gpurun_out/c4_vit.log 2>&1
AURAS_DPT_GRAPH=0 PYTHONPATH=. ncu --set full --clock-control none -k "regex:dpt_attention|conv_gemm_tc$" -s 400 -c 2 -o gpurun_out/c4_dpt -f python scratch/dpt_prof.py > gpurun_out/c4_dpt.log 2>&1
echo done
