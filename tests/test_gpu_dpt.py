"""DP-T transformer denoiser (BASELINE configs[3]) on the B200 vs the CPU
restatement (oracle/dp_model.py dpt_eps, pinned against torch's
TransformerDecoderLayer).  A batch of samples at different inference steps,
each reading its agent's ring slot: eps within 3e-2 normwise relative (bf16
weights and activations, fp32 accumulation), and the scheduler update of the
request lanes within the same tolerance of the oracle's step."""

import numpy as np
import pytest
import torch

from oracle import dp_model
from paper_2509_09560_b200 import _lib
from paper_2509_09560_b200 import diffusion as D

pytestmark = pytest.mark.gpu


def _dpt_iteration(hoist, monkeypatch, xfold=True, S=5):
    """One DP-T iteration of S samples (5: a partial 128-row tile; 8: every
    CTA of the persistent kernel has rows) at steps 0..99 on the device; returns
    (cfg, weights, inputs, eps, updated lanes, cross-attention time rows)."""
    monkeypatch.setenv("AURAS_DPT_HOIST", "1" if hoist else "0")
    monkeypatch.setenv("AURAS_DPT_XFOLD", "1" if xfold else "0")
    cfg = D.DPConfig(name="dpt_gpu_test", encoder="vit_b16", image_hw=224, feat_dim=768, action_dim=7,
                     denoiser="transformer")
    w = D.init_weights(cfg, 4, device="cpu")
    model = D.DeviceModel(cfg, w, "bf16")
    den = D.DPTDenoiser(model, 8)
    rng = np.random.default_rng(1)
    T, A = cfg.horizon, cfg.action_dim
    steps = np.array([0, 13, 50, 98, 99, 1, 77, 42][:S], dtype=np.int32)
    agents = np.arange(S, dtype=np.int32)
    lanes = np.zeros(S, dtype=np.int32)
    x0 = rng.standard_normal((S, 1, T * A)).astype(np.float32)
    noise = rng.standard_normal((S, 1, cfg.num_inference_steps, T * A)).astype(np.float32)
    slot_floats = _lib_round(cfg.gc_dim, 8) + 16
    ring = np.zeros((S, 2, slot_floats), dtype=np.float32)
    gcs = rng.standard_normal((S, cfg.gc_dim)).astype(np.float32)
    ring[:, 1, :cfg.gc_dim] = gcs                      # the frame fetched slot 1
    dev = torch.device("cuda")
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(agents=agents, lanes=lanes, steps=steps, x=x0, noise=noise,
                                                         ring=ring).items()}
    fetched = torch.tensor([1, 7, 3], dtype=torch.int64, device=dev)
    sched = D.scheduler_tables(cfg)
    st_t = {k: torch.tensor(v, dtype=torch.int32 if k == "timestep" else torch.float32, device=dev)
            for k, v in sched.items()}
    sc = _lib.Sched()
    for k in ("timestep", "sqrt_ab", "sqrt_1mab", "c_x0", "c_xt", "c_eps", "sigma"):
        setattr(sc, k, st_t[k].data_ptr())
    sc.n_steps, sc.clip_sample, sc.ddpm = cfg.num_inference_steps, int(cfg.clip_sample), 1
    stream = torch.cuda.current_stream()
    den.frame_cond(S, t["x"].data_ptr(), 1, t["ring"].data_ptr(), 2 * slot_floats, slot_floats, fetched.data_ptr(),
                   stream)
    den.iterate(S, t["agents"].data_ptr(), t["lanes"].data_ptr(), t["steps"].data_ptr(), t["x"].data_ptr(), 1,
                t["ring"].data_ptr(), 2 * slot_floats, slot_floats, fetched.data_ptr(), t["noise"].data_ptr(), sc,
                stream)
    den.memory_rows(S, t["agents"].data_ptr(), t["steps"].data_ptr(), stream)
    torch.cuda.synchronize()
    assert den.xfold == (hoist and xfold) and (bool(den.pplan) or not hoist)
    return dict(cfg=cfg, w=w, S=S, steps=steps, x0=x0, noise=noise, gcs=gcs, sched=sched,
                eps=den.eps[:S].cpu().numpy(), xs=t["x"].cpu().numpy(), kv=den.kv2[:S].float().cpu().numpy())


def _oracle_eps(r):
    cfg, w, steps, x0, gcs, sched = (r[k] for k in ("cfg", "w", "steps", "x0", "gcs", "sched"))
    T, A = cfg.horizon, cfg.action_dim
    out = []
    for s in range(r["S"]):
        with torch.no_grad():
            out.append(dp_model.dpt_eps(w, cfg, torch.from_numpy(x0[s, 0].reshape(T, A)),
                                        int(sched["timestep"][steps[s]]), torch.from_numpy(gcs[s])).numpy())
    return np.stack(out)


@pytest.mark.parametrize("xfold,S", [(True, 5), (False, 5), (True, 8), (False, 8)])
def test_dpt_iteration_matches_oracle(monkeypatch, xfold, S):
    r = _dpt_iteration(True, monkeypatch, xfold, S)
    cfg, w, S, steps, x0, noise, gcs, sched = (r[k] for k in ("cfg", "w", "S", "steps", "x0", "noise", "gcs", "sched"))
    eps, xs = r["eps"], r["xs"]
    T, A = cfg.horizon, cfg.action_dim
    osch = dp_model.Scheduler(cfg)
    for s in range(S):
        xin = torch.from_numpy(x0[s, 0].reshape(T, A))
        with torch.no_grad():
            want = dp_model.dpt_eps(w, cfg, xin, int(sched["timestep"][steps[s]]), torch.from_numpy(gcs[s])).numpy()
            wx = osch.step(int(steps[s]), xin, torch.from_numpy(want),
                           torch.from_numpy(noise[s, 0, steps[s]].reshape(T, A))).numpy()
        err = np.linalg.norm(eps[s] - want) / np.linalg.norm(want)
        assert err <= 3e-2, (s, err)
        xerr = np.linalg.norm(xs[s, 0].reshape(T, A) - wx) / np.linalg.norm(wx)
        assert xerr <= 3e-2, (s, xerr)


def test_hoisted_cross_attention_memory_matches_per_iteration_program(monkeypatch):
    """The hoisted cross-attention memory (time rows from a table built once,
    observation rows once per frame) against the per-iteration device program
    that recomputes cond tokens -> memory -> K|V every iteration
    (AURAS_DPT_HOIST=0): the K|V rows may differ only by bf16 rounding flips,
    and the iteration's eps by the same order."""
    h = _dpt_iteration(True, monkeypatch, xfold=False)
    p = _dpt_iteration(False, monkeypatch)
    kv_err = np.abs(h["kv"] - p["kv"]).max() / np.abs(p["kv"]).max()
    eps_err = np.linalg.norm(h["eps"] - p["eps"]) / np.linalg.norm(p["eps"])
    print(f"hoisted vs per-iteration: K|V rows {kv_err:.2e}, eps {eps_err:.2e}")
    assert kv_err <= 1e-2, kv_err
    assert eps_err <= 1e-2, eps_err


def test_folded_cross_attention_matches_unfolded(monkeypatch):
    """The persistent iteration with the cross-attention folded into per-memory-
    token vectors (one DP_XATTN phase per layer instead of ca_in GEMM,
    attention, ca_out GEMM; auras_dpt_xfold) against the unfolded phases: eps
    within 1.5e-2 of each other (each is ~1.1e-2 from the fp32 oracle with
    these random weights, measured 9.4e-3 apart: the fold skips the bf16
    roundings of q and of the attention output), both within the 3e-2 bar of
    the fp32 oracle, and the fold no farther from the oracle than the unfolded
    program + 2e-3 (measured 1.10e-2 vs 1.14e-2)."""
    f = _dpt_iteration(True, monkeypatch, xfold=True)
    u = _dpt_iteration(True, monkeypatch, xfold=False)
    want = _oracle_eps(f)
    d = np.linalg.norm(f["eps"] - u["eps"]) / np.linalg.norm(u["eps"])
    ef = np.linalg.norm(f["eps"] - want) / np.linalg.norm(want)
    eu = np.linalg.norm(u["eps"] - want) / np.linalg.norm(want)
    print(f"folded vs unfolded eps {d:.2e}; vs fp32 oracle: folded {ef:.2e}, unfolded {eu:.2e}")
    assert d <= 1.5e-2, d
    assert ef <= 3e-2 and eu <= 3e-2, (ef, eu)
    assert ef <= eu + 2e-3, (ef, eu)


def _lib_round(x, m):
    return (x + m - 1) // m * m


def _ddim_pipeline_err(hoist, monkeypatch):
    from oracle import schedule as osched
    from paper_2509_09560_b200 import PipelineConfig, run_pipelined
    monkeypatch.setenv("AURAS_DPT_HOIST", "1" if hoist else "0")
    cfg = D.DPConfig(name="dpt_ddim_test", encoder="vit_b16", image_hw=64, feat_dim=768, action_dim=7,
                     denoiser="transformer", scheduler="ddim", num_inference_steps=16, vit_depth=4, dpt_layers=2)
    w = D.init_weights(cfg, 3, device="cpu")
    pol = D.make_diffusion_policy(cfg, dtype="bf16", weights=w)
    gen = pol.generation
    pcfg = dict(pp_perception=1, pp_generation=4, fetch_offset=-1)
    res = run_pipelined(PipelineConfig(**pcfg), pol, None, 8)
    orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol.perception.layer_costs, gen.step_cost)
    ref = osched.run_pipelined(pcfg, orc, None, 8)
    g = np.array([a.values for a in res.actions])
    r = np.array([a.values for a in ref.actions])
    assert g.shape == r.shape and len(g) > 0
    assert [q.context_versions for q in res.requests] == [q.context_versions for q in ref.requests]
    return float(np.abs(g - r).max() / np.abs(r).max())


def test_small_vit_dpt_ddim_pipeline_matches_oracle(monkeypatch):
    """The DP-T path with a DDIM scheduler (16 steps), a 4-block ViT at 64x64
    and a 2-layer denoiser: pipelined at depth 4 vs the fp32 oracle pipeline.

    DDIM (eta = 0) is a deterministic chain whose coefficients amplify the
    ~0.5 % per-step bf16 eps error of these random weights (per-step bar 3e-2,
    test above) to several % on the action, so the absolute bar is 1e-1, for
    the hoisted path and for the per-iteration path (AURAS_DPT_HOIST=0) alike.
    Which of the two lands closer to the fp32 oracle is rounding noise of that
    chaotic chain (measured 7.0e-2 vs 4.9e-2); whether the hoist changes the
    arithmetic is checked where nothing amplifies it, per iteration
    (test_hoisted_cross_attention_memory_matches_per_iteration_program)."""
    e_hoist = _ddim_pipeline_err(True, monkeypatch)
    e_plain = _ddim_pipeline_err(False, monkeypatch)
    print(f"DDIM DP-T pipeline vs fp32 oracle: hoisted {e_hoist:.3e}, per-iteration {e_plain:.3e}")
    assert e_plain <= 1e-1, e_plain
    assert e_hoist <= 1e-1, e_hoist
