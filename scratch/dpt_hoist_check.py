import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import dp_model
from paper_2509_09560_b200 import _lib
from paper_2509_09560_b200 import diffusion as D
cfg = D.DPConfig(name="dpt_ddim_test", encoder="vit_b16", image_hw=64, feat_dim=768, action_dim=7,
                 denoiser="transformer", scheduler="ddim", num_inference_steps=16, vit_depth=4, dpt_layers=2)
w = D.init_weights(cfg, 3, device="cpu")
model = D.DeviceModel(cfg, w, "bf16")
S = 4
rng = np.random.default_rng(1)
T, A = cfg.horizon, cfg.action_dim
steps = np.array([0, 5, 10, 15], dtype=np.int32)
x0 = rng.standard_normal((S, 1, T * A)).astype(np.float32)
slot_floats = (cfg.gc_dim + 7) // 8 * 8 + 16
ring = np.zeros((S, 2, slot_floats), dtype=np.float32)
gcs = rng.standard_normal((S, cfg.gc_dim)).astype(np.float32)
ring[:, 1, :cfg.gc_dim] = gcs
sched = D.scheduler_tables(cfg)
for hoist in ("1", "0"):
    os.environ["AURAS_DPT_HOIST"] = hoist
    den = D.DPTDenoiser(model, 8)
    dev = torch.device("cuda")
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(agents=np.arange(S, dtype=np.int32), lanes=np.zeros(S, dtype=np.int32), steps=steps, x=x0.copy(), ring=ring).items()}
    fetched = torch.tensor([1, 7, 3], dtype=torch.int64, device=dev)
    st_t = {k: torch.tensor(v, dtype=torch.int32 if k == "timestep" else torch.float32, device=dev) for k, v in sched.items()}
    sc = _lib.Sched()
    for k in ("timestep", "sqrt_ab", "sqrt_1mab", "c_x0", "c_xt", "c_eps", "sigma"):
        setattr(sc, k, st_t[k].data_ptr())
    sc.n_steps, sc.clip_sample, sc.ddpm = cfg.num_inference_steps, 1, 0
    stream = torch.cuda.current_stream()
    den.frame_cond(S, t["x"].data_ptr(), 1, t["ring"].data_ptr(), 2 * slot_floats, slot_floats, fetched.data_ptr(), stream)
    den.iterate(S, t["agents"].data_ptr(), t["lanes"].data_ptr(), t["steps"].data_ptr(), t["x"].data_ptr(), 1,
                t["ring"].data_ptr(), 2 * slot_floats, slot_floats, fetched.data_ptr(), 0, sc, stream)
    torch.cuda.synchronize()
    eps = den.eps[:S].cpu().numpy()
    errs = []
    for s in range(S):
        want = dp_model.dpt_eps(w, cfg, torch.from_numpy(x0[s, 0].reshape(T, A)), int(sched["timestep"][steps[s]]), torch.from_numpy(gcs[s])).numpy()
        errs.append(float(np.linalg.norm(eps[s] - want) / np.linalg.norm(want)))
    print("hoist", hoist, "eps rel errs", [round(e, 4) for e in errs])
