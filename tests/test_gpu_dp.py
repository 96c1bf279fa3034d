"""Diffusion Policy plugin on the B200 vs the CPU oracle.

Both sides run the same weights, the same synthetic frames and the same
host-drawn noise.  The oracle is the restated reference scheduler
(oracle/schedule.py, pinned bit-exact to the reference) driving the torch-CPU
fp32 network restatement (oracle/dp_model.py).

Tolerances (normwise, on the emitted horizon of every action):
  fp32 path  : max|a - a_ref| <= 1e-3 * max|a_ref|     (north_star: 1e-3 relative)
  bf16 path  : max|a - a_ref| <= 6e-2 * max|a_ref|     (bf16 weights+activations,
               fp32 accumulation/normalisation; stated tolerance)
Context versions consumed by every request must match the oracle exactly.
"""

import numpy as np
import pytest
import torch

from oracle import dp_model
from oracle import schedule as osched
from paper_2509_09560_b200 import PipelineConfig, run_decoupled, run_parallel, run_pipelined, run_sequential
from paper_2509_09560_b200 import diffusion as D

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-3, "bf16": 6e-2}
_W = {}


def weights(name, seed=0):
    if (name, seed) not in _W:
        _W[(name, seed)] = D.init_weights(D.PRESETS[name], seed, device="cpu")
    return _W[(name, seed)]


def oracle_run(policy, cfg_dict, duration, agent=0, mode="pipe"):
    gen = policy.generation
    orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, agent, policy.perception.layer_costs,
                            gen.step_cost)
    if mode == "pipe":
        return osched.run_pipelined(cfg_dict, orc, None, duration)
    return osched.run_sequential(orc, None, duration)


def rel_err(got, want):
    g = np.array([a.values for a in got])
    w = np.array([a.values for a in want])
    assert g.shape == w.shape, (g.shape, w.shape)
    return float(np.abs(g - w).max() / np.abs(w).max())


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("pp,off", [((1, 2), 0), ((1, 2), -1), ((1, 4), 0), ((2, 2), 0), ((3, 2), -1)])
def test_tiny_pipelined_matches_oracle(dtype, pp, off):
    pol = D.make_diffusion_policy("tiny", dtype=dtype, weights=weights("tiny"))
    cfg = dict(pp_perception=pp[0], pp_generation=pp[1], fetch_offset=off)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 9)
    ref = oracle_run(pol, cfg, 9)
    assert [r.context_versions for r in res.requests] == [r.context_versions for r in ref.requests]
    err = rel_err(res.actions, ref.actions)
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_tiny_sequential_matches_oracle(dtype):
    pol = D.make_diffusion_policy("tiny", dtype=dtype, weights=weights("tiny"))
    res = run_sequential(pol, None, 4)
    ref = oracle_run(pol, None, 4, mode="seq")
    err = rel_err(res.actions, ref.actions)
    assert err <= TOL[dtype], err


def test_multi_agent_batching_matches_per_agent_oracle():
    pol = D.make_diffusion_policy("tiny", dtype="fp32", weights=weights("tiny"), agents=3)
    cfg = dict(pp_perception=1, pp_generation=3, fetch_offset=0)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 8, agents=3)
    for a in range(3):
        ref = oracle_run(pol, cfg, 8, agent=a)
        err = rel_err(res.agent_actions[a], ref.actions)
        assert err <= TOL["fp32"], (a, err)


def test_device_version_log_matches_schedule():
    pol = D.make_diffusion_policy("tiny", dtype="bf16", weights=weights("tiny"))
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=4, fetch_offset=-1), pol, None, 10)
    for rec in res.trace[1:]:
        if rec["generation"]:
            assert int(res.device_versions[rec["frame"]]) == rec["generation"][0]["context_version"]


def test_graph_and_eager_paths_agree():
    w = weights("tiny")
    cfg = PipelineConfig(pp_perception=1, pp_generation=2, fetch_offset=0)
    a = run_pipelined(cfg, D.make_diffusion_policy("tiny", dtype="bf16", weights=w, use_graph=True), None, 6)
    b = run_pipelined(cfg, D.make_diffusion_policy("tiny", dtype="bf16", weights=w, use_graph=False), None, 6)
    assert np.array_equal(np.array([x.values for x in a.actions]), np.array([x.values for x in b.actions]))


def test_pusht_bf16_matches_oracle():
    """BASELINE configs[1] shape (512/1024/2048 UNet, 100-step DDPM), 2 emitted actions."""
    w = weights("pusht")
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=w)
    cfg = dict(pp_perception=1, pp_generation=2, fetch_offset=0)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 3)
    ref = oracle_run(pol, cfg, 3)
    err = rel_err(res.actions, ref.actions)
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("agents", [1, 3])
def test_disaggregated_path_matches_colocated(agents):
    """Disaggregated variant (perception GPU -> P2P slot copy -> system-scope
    release into the generation GPU's ring), run with both roles on GPU 0
    (every run here has one GPU): same actions bit for bit, same versions,
    and within tolerance of the oracle."""
    w = weights("tiny")
    cfg = dict(pp_perception=1, pp_generation=3, fetch_offset=-1)
    kw = dict(dtype="fp32", weights=w, agents=agents)
    a = run_pipelined(PipelineConfig(**cfg), D.make_diffusion_policy("tiny", **kw), None, 9, agents=agents)
    b = run_pipelined(PipelineConfig(**cfg), D.make_diffusion_policy("tiny", perception_device=0, **kw),
                      None, 9, agents=agents)
    for x, y in zip(a.agent_actions, b.agent_actions):
        assert np.array_equal(np.array([r.values for r in x]), np.array([r.values for r in y]))
    assert [r.context_versions for r in a.requests] == [r.context_versions for r in b.requests]
    assert np.array_equal(a.device_versions, b.device_versions)
    ref = oracle_run(D.make_diffusion_policy("tiny", **kw), cfg, 9)
    assert rel_err(b.agent_actions[0], ref.actions) <= TOL["fp32"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_disaggregated_two_gpus():
    w = weights("tiny")
    cfg = dict(pp_perception=1, pp_generation=2, fetch_offset=0)
    pol = D.make_diffusion_policy("tiny", dtype="fp32", weights=w, perception_device=1)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 8, clock="device")
    ref = oracle_run(pol, cfg, 8)
    assert [r.context_versions for r in res.requests] == [r.context_versions for r in ref.requests]
    assert rel_err(res.actions, ref.actions) <= TOL["fp32"]


_ORC = {}


@pytest.mark.parametrize("variant", ["64", "128"])
def test_cluster_kernel_variants_match_oracle(variant, monkeypatch):
    """Both cluster-kernel variants (64 / 128 columns per tile task; the per-S
    autotune may pick either) forced on the pusht shape with 8 lock-stepped
    agents at depth 2, so one denoise launch runs S = 16 samples over all of
    the frame's iterations: agents 0 and 7 within the bf16 tolerance of their
    oracle runs, same context versions."""
    monkeypatch.setenv("AURAS_MEGA_KERNEL", "cluster")
    monkeypatch.setenv("AURAS_CL_VARIANT", variant)
    w = weights("pusht")
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=w, agents=8)
    cfg = dict(pp_perception=1, pp_generation=2, fetch_offset=0)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 3, agents=8)
    for a in (0, 7):
        if a not in _ORC:
            _ORC[a] = oracle_run(pol, cfg, 3, agent=a)
        ref = _ORC[a]
        err = rel_err(res.agent_actions[a], ref.actions)
        assert err <= TOL["bf16"], (variant, a, err)


@pytest.mark.parametrize("mode", ["par", "dec"])
def test_tiny_par_dec_match_oracle(mode):
    """PAR / DEC baselines with the Diffusion Policy
    plugin vs the oracle driving the CPU network through the restated
    schedules: same context versions, fp32 actions within 1e-3."""
    pol = D.make_diffusion_policy("tiny", dtype="fp32", weights=weights("tiny"))
    gen = pol.generation
    orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol.perception.layer_costs, gen.step_cost)
    interval = pol.sequential_cost / 4.0
    if mode == "par":
        res = run_parallel(pol, None, 3, 10, interval)
        ref = osched.run_parallel(orc, None, 3, 10, interval)
    else:
        res = run_decoupled(pol, None, 10, interval)
        ref = osched.run_decoupled(orc, None, 10, interval)
    assert len(res.actions) == len(ref.actions) > 0
    assert [r.context_versions for r in res.requests] == [r.context_versions for r in ref.requests]
    assert rel_err(res.actions, ref.actions) <= TOL["fp32"]
