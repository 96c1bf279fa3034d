import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=64)
for k in (3, 4, 6, 8):
    host = []
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=k), pol, None, 30, clock="device",
                        frame_hook=lambda t, d, e: host.append(time.perf_counter()))
    ft = res.frame_times
    ends = np.array([ft["end"][t] for t in range(30)])
    print(k, "dev frame ms", np.round(np.diff(ends) * 1e3, 1).tolist(), flush=True)
    print(k, "host frame ms", np.round(np.diff(host) * 1e3, 1).tolist(), flush=True)
