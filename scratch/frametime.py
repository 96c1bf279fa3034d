import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
cfg = D.PRESETS["pusht"]
w = D.init_weights(cfg, 0, device="cuda")
def go(tag, **kw):
    pol = D.make_diffusion_policy(cfg, weights=w, **kw)
    host = []
    def hook(t, dev, emis):
        host.append(time.perf_counter())
    t0 = time.perf_counter()
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8), pol, None, 40, clock="device", frame_hook=hook)
    el = time.perf_counter() - t0
    ft = res.frame_times
    ends = np.array([ft["end"][t] for t in range(40)])
    starts = np.array([ft["start"][t] for t in range(40)])
    hd = np.diff(host)
    print(f"{tag}: total {el:.2f}s host/frame med {np.median(hd)*1e3:.1f}ms max {hd.max()*1e3:.1f}; dev frame (end diff) med {np.median(np.diff(ends))*1e3:.2f}ms; start-end med {np.median(ends-starts)*1e3:.2f}", flush=True)
    print("   host per frame:", np.round(hd*1e3,1)[:20])
go("resident", resident_frames=64)
go("resident2", resident_frames=64)
go("host")
go("resident-nograph", resident_frames=64, use_graph=False)
