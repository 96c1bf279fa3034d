"""Tight parity of the benchmarked bf16 tensor-core denoise path.

The oracle is oracle/dp_model.py in its bf16-faithful mode
(`OracleDP(..., numerics="bf16")`, `bf16_weights` + a bf16 store at every
point the device stores an activation, fp32 accumulation, GroupNorm
statistics, FiLM rows and scheduler update).  It differs from the device only
in summation order and the rounding flips that order causes, so the bars here
are an order of magnitude tighter than the bf16-vs-fp32 tolerance
(tests/test_gpu_dp.py):

  one batched denoise launch (every sample at its own timestep, unequal
  iteration counts inside the launch)      : max|dx| <= 5e-3 * max|x_ref|
  pipelined actions, exact BENCH config    : <= 1e-2 vs the bf16 oracle,
                                             <= 6e-2 vs the fp32 oracle
  context versions                         : identical

Reference semantics: each request's stage j runs plan[j-1] iterations on the
frame's single fetched context (fp/executor.py:318-349, split_generation at
fp/partition.py:101-123); the step is GenerationModel.step
(fp/policy.py:217-228) with a neural generator.
"""

import numpy as np
import pytest
import torch

from oracle import dp_model
from oracle import schedule as osched
from paper_2509_09560_b200 import PipelineConfig, run_pipelined
from paper_2509_09560_b200 import diffusion as D

pytestmark = pytest.mark.gpu

STEP_TOL = 5e-3
PIPE_TOL_BF16 = 1e-2
PIPE_TOL_FP32 = 6e-2

from dp_harness import norm_err, run_denoise_launch, weights


@pytest.mark.parametrize("S", [1, 3, 5, 8, 16, 64])
def test_denoise_launch_matches_bf16_oracle(S):
    """The headline kernel (autotuned per S: the cluster megakernel wins every
    S measured) on S samples, each at its own diffusion timestep with 1-3
    iterations in the same launch."""
    got, want, x0, kernel = run_denoise_launch("pusht", S)
    err = norm_err(got, want)
    print(f"S={S} kernel={kernel} err={err:.2e}")
    assert kernel in (1, 2)
    assert np.abs(got - x0).max() > 1e-2          # the samples moved
    assert err <= STEP_TOL, err


@pytest.mark.parametrize("kernel,variant", [("cluster", "64"), ("cluster", "128"), ("l2", None)])
def test_denoise_launch_every_engine(kernel, variant, monkeypatch):
    """Each persistent engine forced (cluster 64- / 128-column variants, L2
    split-K megakernel) at S = 16 with 2 agents x 8 lanes."""
    monkeypatch.setenv("AURAS_MEGA_KERNEL", kernel)
    if variant:
        monkeypatch.setenv("AURAS_CL_VARIANT", variant)
    got, want, _, k = run_denoise_launch("pusht", 16, agents=2)
    err = norm_err(got, want)
    print(f"{kernel}/{variant} kernel={k} err={err:.2e}")
    assert k == (2 if kernel == "cluster" else 1)
    assert err <= STEP_TOL, err


def test_large_prenorm_partials_are_range_safe():
    """Split-K partials travel between the cluster's CTAs as fp16.  Scaling the
    weights of GroupNorm'd convs by 1e6 makes their pre-norm values ~1e5-1e6,
    so 1/8-K partial sums pass fp16's 65504: unscaled they would become inf and
    NaN through GroupNorm.  The kernel sends such rows as fp16(x 2^-e) with the
    exponent on the side, and GroupNorm makes the block's output scale-free, so
    the launch must still match the bf16 oracle at the usual bar."""
    w = dict(weights("pusht"))
    for name in ("unet.down1.0.c1.w", "unet.mid.0.c2.w", "unet.up1.1.c1.w"):
        w[name] = w[name] * 1e6
    got, want, _, kernel = run_denoise_launch("pusht", 8, w=w)
    err = norm_err(got, want)
    print(f"pre-norm x1e6: kernel={kernel} err={err:.2e}")
    assert kernel == 2
    assert np.isfinite(got).all()
    assert err <= STEP_TOL, err


def test_layer_by_layer_path_matches_bf16_oracle(monkeypatch):
    """The stand-alone tcgen05 GEMM + epilogue path (no persistent kernel)."""
    monkeypatch.setenv("AURAS_NO_MEGA", "1")
    got, want, _, k = run_denoise_launch("pusht", 5)
    assert k == 0
    assert norm_err(got, want) <= STEP_TOL


# ---------------------------------------------------------------- pipelines

_ORC_CACHE = {}


def oracle_pipe(cfg_name, numerics, cfg_dict, duration, alpha=0.0):
    key = (cfg_name, numerics, tuple(sorted(cfg_dict.items())), duration)
    if key not in _ORC_CACHE:
        cfg = D.PRESETS[cfg_name]
        pol = D.make_diffusion_policy(cfg_name, dtype="bf16", weights=weights(cfg_name))
        orc = dp_model.OracleDP(weights(cfg_name), cfg, 0, 0, pol.perception.layer_costs,
                                pol.generation.step_cost, numerics=numerics)
        _ORC_CACHE[key] = osched.run_pipelined(cfg_dict, orc, None, duration)
    return _ORC_CACHE[key]


def actions_err(got, want):
    g = np.array([a.values for a in got])
    w = np.array([a.values for a in want])
    assert g.shape == w.shape, (g.shape, w.shape)
    return float(np.abs(g - w).max() / np.abs(w).max())


def test_bench_config_matches_oracles():
    """The exact BENCH config: pusht, bf16, pp = (1, 8), offset 0, alpha 0 --
    split_generation(100, 8) = [13, 12, 13, 12, 13, 12, 13, 12], so the S = 8
    launch of every steady-state frame mixes 13- and 12-iteration samples --
    for 11 emitted actions."""
    cfg = dict(pp_perception=1, pp_generation=8, fetch_offset=0)
    duration = 18
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=weights("pusht"))
    res = run_pipelined(PipelineConfig(**cfg), pol, None, duration)
    assert len(res.actions) >= 10
    ref16 = oracle_pipe("pusht", "bf16", cfg, duration)
    ref32 = oracle_pipe("pusht", "fp32", cfg, duration)
    assert [r.context_versions for r in res.requests] == [r.context_versions for r in ref16.requests]
    e16, e32 = actions_err(res.actions, ref16.actions), actions_err(res.actions, ref32.actions)
    print(f"bench config: vs bf16 oracle {e16:.2e}, vs fp32 oracle {e32:.2e}")
    assert e16 <= PIPE_TOL_BF16, e16
    assert e32 <= PIPE_TOL_FP32, e32


def test_alpha_half_plan_matches_bf16_oracle():
    """alpha = 0.5 at pp = (1, 4): split_generation(100, 4, 0.5) = [10, 17, 27,
    46] (fp/partition.py:101-123, t/test_partition.py:12-22): four unequal
    stage shares inside each frame's launch, offset -1."""
    from paper_2509_09560_b200 import split_generation
    assert split_generation(100, 4, 0.5) == [10, 17, 27, 46]
    cfg = dict(pp_perception=1, pp_generation=4, fetch_offset=-1, alpha=0.5)
    duration = 9
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=weights("pusht"))
    res = run_pipelined(PipelineConfig(**cfg), pol, None, duration)
    ref = oracle_pipe("pusht", "bf16", cfg, duration)
    assert len(res.actions) >= 4
    assert [r.context_versions for r in res.requests] == [r.context_versions for r in ref.requests]
    err = actions_err(res.actions, ref.actions)
    print(f"alpha 0.5: {err:.2e}")
    assert err <= PIPE_TOL_BF16, err


def test_pusht_fp32_matches_oracle():
    """fp32 reference-precision path on the full pusht shape: 1e-3 relative
    (north_star)."""
    cfg = dict(pp_perception=1, pp_generation=2, fetch_offset=0)
    duration = 4
    pol = D.make_diffusion_policy("pusht", dtype="fp32", weights=weights("pusht"))
    res = run_pipelined(PipelineConfig(**cfg), pol, None, duration)
    ref = oracle_pipe("pusht", "fp32", cfg, duration)
    err = actions_err(res.actions, ref.actions)
    print(f"pusht fp32: {err:.2e}")
    assert err <= 1e-3, err


# ---------------------------------------------------------------- closed loop

class _PosEnv:
    """Deterministic closed-loop environment for the image policy: the camera
    frame is the synthetic frame of (seed, frame); the low-dim state (agent
    position, part of the global conditioning) integrates every applied
    action.  A stale or missing action changes every later observation."""

    success_threshold = None

    def __init__(self, cfg):
        self.cfg = cfg
        self.pos = np.array([0.25, -0.5])
        self.applied = []
        self.last_error = 0.0

    def observe(self, frame):
        from paper_2509_09560_b200 import Observation
        img = D.synthetic_frame(self.cfg, 0, 0, frame).image
        return Observation(frame=frame, vector=self.pos.astype(np.float32), image=img)

    def apply_action(self, action):
        a = np.asarray(action, dtype=np.float64).reshape(-1)
        if a.size != self.cfg.action_dim:           # the oracle hands over the whole horizon
            a = a.reshape(self.cfg.horizon, self.cfg.action_dim)[self.cfg.n_obs_steps - 1]
            n = float(np.linalg.norm(a))
            if n > self.cfg.max_action:
                a = a * (self.cfg.max_action / n)
        self.applied.append(a.copy())
        self.pos = self.pos + a

    def advance_frame(self):
        self.last_error = float(np.linalg.norm(self.pos))


def test_closed_loop_applies_the_emitted_actions():
    """fp/executor.py:165-178, 386: the action emitted in frame t lands at
    t + 1, before frame t + 1 is observed.  The device writes the action row on
    the generation stream; the host must not read it before the finish kernel
    ran (a read racing it lands zeros or a stale row and the trajectories
    diverge)."""
    cfg = D.PRESETS["pusht"]
    pcfg = dict(pp_perception=1, pp_generation=4, fetch_offset=0)
    duration = 10
    env_dev, env_orc = _PosEnv(cfg), _PosEnv(cfg)
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=weights("pusht"))
    run_pipelined(PipelineConfig(**pcfg), pol, env_dev, duration)
    orc = dp_model.OracleDP(weights("pusht"), cfg, 0, 0, pol.perception.layer_costs,
                            pol.generation.step_cost, numerics="bf16")
    osched.run_pipelined(pcfg, orc, env_orc, duration)
    got, want = np.array(env_dev.applied), np.array(env_orc.applied)
    assert got.shape == want.shape and len(got) >= 5, (got.shape, want.shape)
    assert np.abs(got).min() > 0.0                  # never a zero (unwritten) row
    err = float(np.abs(got - want).max() / np.abs(want).max())
    print(f"closed loop: {len(got)} actions, err {err:.2e}")
    assert err <= PIPE_TOL_BF16, err
