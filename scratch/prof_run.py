"""Short steady-state run for ncu launch lists: pusht, depth 8, resident inputs."""
import sys
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS[sys.argv[2] if len(sys.argv) > 2 else "pusht"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=16)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 12
run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8), pol, None, frames, clock="device")
print("done")
