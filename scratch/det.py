import numpy as np, sys
sys.path.insert(0, '.')
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D
from oracle import dp_model, schedule as osched
w = D.init_weights(D.PRESETS["tiny"], 0, device="cpu")
cfg = PipelineConfig(pp_perception=1, pp_generation=2, fetch_offset=0)
def run(g, dt="bf16"):
    return np.array([x.values for x in run_pipelined(cfg, D.make_diffusion_policy("tiny", dtype=dt, weights=w, use_graph=g), None, 6).actions])
pol = D.make_diffusion_policy("tiny", dtype="bf16", weights=w)
orc = dp_model.OracleDP(w, pol.generation.cfg, 0, 0, pol.perception.layer_costs, pol.generation.step_cost)
ref = np.array([a.values for a in osched.run_pipelined(dict(pp_perception=1, pp_generation=2, fetch_offset=0), orc, None, 6).actions])
for dt in ("bf16", "fp32"):
    g1, g2, e1, e2 = run(True, dt), run(True, dt), run(False, dt), run(False, dt)
    err = lambda a: float(np.abs(a-ref).max()/np.abs(ref).max())
    print(dt, "graph self", np.array_equal(g1, g2), "eager self", np.array_equal(e1, e2), "g-e", float(np.abs(g1-e1).max()),
          "err graph", err(g1), err(g2), "err eager", err(e1), err(e2))
