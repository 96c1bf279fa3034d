import sys, os
sys.path.insert(0, os.getcwd())
os.environ["AURAS_DPT_GRAPH"] = "0"
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["vit_dpt"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=16)
run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8), pol, None, 12, clock="device")
print("done")
