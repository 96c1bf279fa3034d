import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
def go(tag, env):
    for k, v in env.items(): os.environ[k] = v
    pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=16)
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8), pol, None, 30, clock="device")
    ft = res.frame_times
    ends = np.array([ft["end"][i] for i in range(30)]); st = np.array([ft["start"][i] for i in range(30)])
    print(f"{tag:28s} frame ms med {np.median(np.diff(ends)[10:])*1e3:7.2f}  P-start->G-end med {np.median((ends-st)[10:])*1e3:7.2f}", flush=True)
    for k in env: os.environ.pop(k)
go("mega prio res8", {})
go("mega noprio res8", {"AURAS_G_PRIORITY": "0"})
go("mega prio res0", {"AURAS_MEGA_RESERVE": "0"})
go("mega prio res20", {"AURAS_MEGA_RESERVE": "20"})
go("layer prio", {"AURAS_NO_MEGA": "1"})
go("layer noprio", {"AURAS_NO_MEGA": "1", "AURAS_G_PRIORITY": "0"})
