import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from paper_2509_09560_b200 import run_decoupled, run_parallel, run_pipelined, PipelineConfig
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=64)
print("sequential_cost", pol.sequential_cost, "p_cost", pol.perception.total_cost, "g_cost", pol.generation.total_cost)
for name in ("dec", "par"):
    interval = pol.sequential_cost / 8
    frames = 24 if name == "dec" else 96
    t0 = time.time()
    if name == "dec":
        res = run_decoupled(pol, None, frames, interval, clock="device")
    else:
        res = run_parallel(pol, None, 8, frames, interval, clock="device")
    torch.cuda.synchronize()
    ft = res.frame_times
    d = [ (ft["end"][t] - ft["start"][t]) * 1e3 for t in range(frames)]
    print(name, "host s", round(time.time() - t0, 2), "actions", len(res.actions))
    print(" frame ms", " ".join(f"{x:.1f}" for x in d))
    print(" completions", [r.completion_frame for r in res.requests])
