import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from oracle import dp_model
from oracle import schedule as osched
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
for hoist in ("1", "0"):
    os.environ["AURAS_DPT_HOIST"] = hoist
    for steps, sch in ((16, "ddim"), (100, "ddpm")):
        cfg = D.DPConfig(name="t", encoder="vit_b16", image_hw=64, feat_dim=768, action_dim=7, denoiser="transformer",
                         scheduler=sch, num_inference_steps=steps, vit_depth=4, dpt_layers=2)
        w = D.init_weights(cfg, 3, device="cpu")
        pol = D.make_diffusion_policy(cfg, dtype="bf16", weights=w)
        gen = pol.generation
        pcfg = dict(pp_perception=1, pp_generation=4, fetch_offset=-1)
        res = run_pipelined(PipelineConfig(**pcfg), pol, None, 8)
        orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol.perception.layer_costs, gen.step_cost)
        ref = osched.run_pipelined(pcfg, orc, None, 8)
        g = np.array([a.values for a in res.actions]); r = np.array([a.values for a in ref.actions])
        print("hoist", hoist, sch, "err", float(np.abs(g - r).max() / np.abs(r).max()), "per-action", [round(float(np.abs(g[i]-r[i]).max()/np.abs(r).max()),3) for i in range(len(g))])
