import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
for name, frames in (("tiny", 8), ("pusht", 12)):
    cfg = D.PRESETS[name]
    w = D.init_weights(cfg, 0, device="cuda")
    out = {}
    for mode in ("layer", "mega"):
        if mode == "layer": os.environ["AURAS_NO_MEGA"] = "1"
        else: os.environ.pop("AURAS_NO_MEGA", None)
        pol = D.make_diffusion_policy(cfg, weights=w, resident_frames=16)
        t = time.time()
        res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=8 if name == "pusht" else 2), pol, None, frames, clock="device")
        ft = res.frame_times
        ends = np.array([ft["end"][i] for i in range(frames)])
        out[mode] = np.array([a.values for a in res.actions])
        print(name, mode, "wall", round(time.time() - t, 2), "dev frame ms", np.round(np.diff(ends)[-4:] * 1e3, 2).tolist(), flush=True)
    print(name, "mega==layer", np.array_equal(out["mega"], out["layer"]), "maxdiff", float(np.abs(out["mega"] - out["layer"]).max()), flush=True)
