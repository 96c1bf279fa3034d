"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Test infrastructure only (see oracle/__init__.py).  Run in the build container,
where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

It imports `framepipe` read-only and records, for a fixed list of cases:

* partition goldens: `split_generation` / `split_perception` outputs
  (fp/partition.py:57-123), including the seeded fuzz sets the reference tests
  use (t/test_partition.py:42-82);
* schedule goldens: complete schema-1 traces and RequestRecords of
  `run_pipelined` (fp/executor.py:200-399) and `run_sequential`
  (fp/executor.py:406-461) with the toy refinement policy
  (fp/policy.py:279-297).  Closed-loop cases also record every observation
  vector the TrackingEnv produced (fp/envsim.py:89-95) and every sealed error,
  so the GPU box (which has no /root/reference) can replay them open-loop: if
  the device engine's actions are bit-identical, the closed loop would have
  produced the same observations.

Nothing here is imported by the product package.
"""

from __future__ import annotations

import gzip
import json
import math
import os
import random
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from framepipe.envsim import CirclePath, TrackingEnv  # noqa: E402
from framepipe.executor import (PipelineConfig, run_decoupled, run_parallel, run_pipelined,  # noqa: E402
                                run_sequential)
from framepipe.metrics import compare, summarize  # noqa: E402
from framepipe.partition import split_generation, split_perception  # noqa: E402
from framepipe.policy import make_autoregressive_policy, make_conditioning_policy  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


class RecordingEnv:
    """Wraps a reference TrackingEnv and records what the executor saw."""

    def __init__(self, env):
        self.env = env
        self.success_threshold = env.success_threshold
        self.observations = {}
        self.errors = []
        self.applied = []

    def observe(self, frame):
        obs = self.env.observe(frame)
        self.observations[frame] = [float(v) for v in obs.vector]
        return obs

    def apply_action(self, action):
        self.applied.append([float(v) for v in np.asarray(action, dtype=np.float64)])
        self.env.apply_action(action)

    def advance_frame(self):
        self.env.advance_frame()

    @property
    def last_error(self):
        err = self.env.last_error
        self.errors.append(float(err))
        return err


def tracking_env(seed, frames=300, omega_deg=15.0, sigma=0.02):
    return TrackingEnv(path=CirclePath(radius=1.0, omega=math.radians(omega_deg)),
                       noise_sigma=sigma, max_step=0.8, episode_frames=frames, seed=seed)


def _jsonable(x):
    if isinstance(x, dict):
        return {k: _jsonable(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_jsonable(v) for v in x]
    if isinstance(x, (np.floating,)):
        return float(x)
    if isinstance(x, (np.integer,)):
        return int(x)
    return x


def _metrics_or_error(trace):
    try:
        return json.loads(summarize(trace).to_json())
    except Exception as e:                           # noqa: BLE001 -- EmptyTrace on 0-frame runs
        return {"error": type(e).__name__}


def record_case(name, mode, policy_kw, duration, cfg_kw=None, env_seed=None,
                seq_interval=None, env_kw=None, workers=None, capacity=1.0):
    kw = dict(policy_kw)
    factory = make_autoregressive_policy if kw.pop("autoregressive", False) else make_conditioning_policy
    policy = factory(**kw)
    env = None
    if env_seed is not None:
        env = RecordingEnv(tracking_env(env_seed, **(env_kw or {})))
    if mode == "pipe":
        cfg = PipelineConfig(**cfg_kw)
        result = run_pipelined(cfg, policy, env, duration)
    elif mode == "par":
        result = run_parallel(policy, env, workers, duration, frame_interval=seq_interval, capacity=capacity)
    elif mode == "dec":
        result = run_decoupled(policy, env, duration, frame_interval=seq_interval)
    else:
        result = run_sequential(policy, env, duration, frame_interval=seq_interval)
    case = {
        "name": name,
        "mode": mode,
        "policy": policy_kw,
        "duration": duration,
        "pipeline": cfg_kw,
        "seq_interval": seq_interval,
        "workers": workers,
        "capacity": capacity,
        "trace": _jsonable(result.trace),
        "requests": [_jsonable(vars(r)) for r in result.requests],
        "actions": [[float(v) for v in a.values] for a in result.actions],
        "staleness_profiles": [list(a.staleness_profile) for a in result.actions],
        "metrics": _metrics_or_error(result.trace),
        "env": None,
    }
    if env is not None:
        case["env"] = {
            "seed": env_seed,
            "kw": env_kw or {},
            "success_threshold": env.success_threshold,
            "observations": [env.observations[t] for t in sorted(env.observations)],
            "errors": env.errors,
            "applied": env.applied,
        }
    return case


SIX = dict(layer_costs=(1.0, 1.0), n_iterations=4, step_cost=1.0)
CAL = dict(layer_costs=(14.0, 14.0), n_iterations=100, step_cost=1.0, eta=0.08, max_action=0.8)
STALE = dict(layer_costs=(1.0,), n_iterations=100, step_cost=0.01)
NOISY16 = dict(layer_costs=(14.0, 14.0), n_iterations=16, step_cost=1.0, noise_init=True)
NOISY100 = dict(layer_costs=(14.0, 14.0), n_iterations=100, step_cost=1.0, noise_init=True)
SKEW = dict(layer_costs=(128.0, 128.0), n_iterations=100, step_cost=1.0, max_action=0.8)
MULTI = dict(layer_costs=(3.0, 5.0, 2.0, 4.0), n_iterations=30, step_cost=1.0, noise_init=True)


def schedule_cases():
    pc = PipelineConfig
    cases = []
    # t/test_executor.py:52-59 throughput law, :67-74 steady emission, :94-108
    for pp in ((2, 4), (1, 2), (1, 1)):
        cases.append(record_case(f"six_pipe_{pp[0]}{pp[1]}_m1", "pipe", SIX, 48,
                                 dict(pp_perception=pp[0], pp_generation=pp[1], fetch_offset=-1)))
    cases.append(record_case("six_pipe_24_m1_interval1", "pipe", SIX, 40,
                             dict(pp_perception=2, pp_generation=4, fetch_offset=-1, frame_interval=1.0)))
    cases.append(record_case("six_pipe_24_off0", "pipe", SIX, 48,
                             dict(pp_perception=2, pp_generation=4, fetch_offset=0)))
    cases.append(record_case("six_seq", "seq", SIX, 48))
    # t/test_executor.py:76-92 staleness profile and final age
    cases.append(record_case("stale_14_m1", "pipe", STALE, 30,
                             dict(pp_perception=1, pp_generation=4, fetch_offset=-1, frame_interval=1.0)))
    cases.append(record_case("stale_14_off0_i2", "pipe", STALE, 30,
                             dict(pp_perception=1, pp_generation=4, fetch_offset=0, frame_interval=2.0)))
    # :127-135 offset -2 with K = 4
    cases.append(record_case("stale_12_m2_k4", "pipe", STALE, 30,
                             dict(pp_perception=1, pp_generation=2, fetch_offset=-2,
                                  store_capacity=4, frame_interval=2.0)))
    # :110-125 mode equivalence (closed loop, env seed 11)
    cases.append(record_case("cal_seq_env11", "seq", CAL, 200, env_seed=11, seq_interval=128.0))
    cases.append(record_case("cal_pipe_11_off0_env11", "pipe", CAL, 200,
                             dict(pp_perception=1, pp_generation=1, fetch_offset=0, frame_interval=128.0),
                             env_seed=11))
    # :137-167 snapshot / live, closed loop
    for mode in ("snapshot", "live"):
        cases.append(record_case(f"cal_pipe_12_m1_{mode}_env4", "pipe", CAL, 120,
                                 dict(pp_perception=1, pp_generation=2, fetch_offset=-1,
                                      frame_interval=64.0, read_policy=mode), env_seed=4))
    # seq with dropped observations (:42-48)
    cases.append(record_case("cal_seq_i64", "seq", CAL, 20, seq_interval=64.0))
    # :178-199 overrun stretch / drop
    for pol in ("stretch", "drop"):
        cases.append(record_case(f"six_pipe_11_m1_{pol}", "pipe", SIX, 21,
                                 dict(pp_perception=1, pp_generation=1, fetch_offset=-1,
                                      frame_interval=3.0, overrun_policy=pol)))
    # SURVEY appendix A dumps: noise-initialised 16-step policy
    for pp, off in (((1, 2), 0), ((1, 2), -1), ((1, 4), 0), ((1, 4), -1)):
        cases.append(record_case(f"noisy16_pipe_{pp[0]}{pp[1]}_off{off}", "pipe", NOISY16, 40,
                                 dict(pp_perception=pp[0], pp_generation=pp[1], fetch_offset=off)))
    cases.append(record_case("noisy16_seq", "seq", NOISY16, 40))
    # skewed partitions (t/test_partition.py:15-19; t/test_acceptance.py:180-201)
    cases.append(record_case("noisy100_pipe_14_a05", "pipe", NOISY100, 40,
                             dict(pp_perception=1, pp_generation=4, fetch_offset=0, alpha=0.5)))
    cases.append(record_case("skew_pipe_15_a1_env2", "pipe", SKEW, 80,
                             dict(pp_perception=1, pp_generation=5, fetch_offset=0, alpha=1.0),
                             env_seed=2, env_kw=dict(omega_deg=24.0)))
    # depth sweep at n = 100 (SURVEY appendix A virtual k-sweep), both offsets
    for k in (3, 5, 8):
        for off in (0, -1):
            cases.append(record_case(f"noisy100_pipe_1{k}_off{off}", "pipe", NOISY100, 30,
                                     dict(pp_perception=1, pp_generation=k, fetch_offset=off)))
    cases.append(record_case("noisy100_seq", "seq", NOISY100, 30))
    # multi-stage perception (pp_p > 1) and deeper offsets
    cases.append(record_case("multi_pipe_23_m1", "pipe", MULTI, 36,
                             dict(pp_perception=2, pp_generation=3, fetch_offset=-1)))
    cases.append(record_case("multi_pipe_32_m2_k3", "pipe", MULTI, 36,
                             dict(pp_perception=3, pp_generation=2, fetch_offset=-2, store_capacity=3)))
    cases.append(record_case("multi_pipe_42_off0_live", "pipe", MULTI, 36,
                             dict(pp_perception=4, pp_generation=2, fetch_offset=0, read_policy="live")))
    return cases


def baseline_cases():
    """PAR (fp/executor.py:477-576) and DEC (:583-701), the paper's baselines
    (SURVEY.md §8(f) row 1), with the same toy policies."""
    cases = []
    for w in (1, 2, 4):
        cases.append(record_case(f"six_par_w{w}", "par", SIX, 40, workers=w))
    cases.append(record_case("six_par_w3_i2", "par", SIX, 40, workers=3, seq_interval=2.0))
    cases.append(record_case("six_par_w2_cap2_i3", "par", SIX, 40, workers=2, seq_interval=3.0, capacity=2.0))
    cases.append(record_case("noisy16_par_w4_i8", "par", NOISY16, 40, workers=4, seq_interval=8.0))
    cases.append(record_case("noisy100_par_w8_i16", "par", NOISY100, 40, workers=8, seq_interval=16.0))
    cases.append(record_case("cal_par_w2_i64_env3", "par", CAL, 120, workers=2, seq_interval=64.0, env_seed=3))
    cases.append(record_case("six_dec", "dec", SIX, 40))
    cases.append(record_case("six_dec_i1", "dec", SIX, 40, seq_interval=1.0))
    cases.append(record_case("noisy16_dec_i8", "dec", NOISY16, 40, seq_interval=8.0))
    cases.append(record_case("noisy100_dec_i16", "dec", NOISY100, 40, seq_interval=16.0))
    cases.append(record_case("multi_dec_i5", "dec", MULTI, 40, seq_interval=5.0))
    cases.append(record_case("cal_dec_i64_env5", "dec", CAL, 120, seq_interval=64.0, env_seed=5))
    return cases


TUNE_POLICY = dict(layer_costs=(4.0, 4.0), n_iterations=12, step_cost=1.0, eta=0.3, max_action=0.8)
TUNE_REQUEST = dict(throughput_requirement=0.06, l_max=4, alpha_grid=(0.0, 0.5), seeds=(0, 1),
                    throughput_frames=24, accuracy_frames=40)


def tuner_golden():
    """fp/tuner.py grid_search + finetune_alpha on a small request (toy policy,
    TrackingEnv rollouts), and an infeasible request's evaluation log."""
    from framepipe.errors import NoFeasibleConfig
    from framepipe.tuner import TuneRequest, finetune_alpha, grid_search
    pol = make_conditioning_policy(**TUNE_POLICY)
    req = TuneRequest(**TUNE_REQUEST)
    factory = lambda seed: tracking_env(seed, frames=60)  # noqa: E731
    g = grid_search(pol, factory, req)
    f = finetune_alpha(pol, factory, g.chosen, req)
    bad = TuneRequest(**dict(TUNE_REQUEST, throughput_requirement=5.0))
    try:
        grid_search(pol, factory, bad)
        infeasible = None
    except NoFeasibleConfig as exc:
        infeasible = {"message": str(exc), "result": exc.result.to_dict()}
    return {"policy": TUNE_POLICY, "request": {k: list(v) if isinstance(v, tuple) else v
                                               for k, v in TUNE_REQUEST.items()},
            "env_frames": 60, "grid": g.to_dict(), "alpha": f.to_dict(), "infeasible": infeasible}


def partition_goldens():
    out = {"generation": [], "perception": []}
    fixed = [(100, 4, 0.0), (100, 4, 0.5), (100, 5, 1.0), (100, 5, 0.0), (7, 1, 0.0),
             (3, 5, 1.5), (100, 5, -1.0), (16, 2, 0.0), (100, 8, 0.0), (100, 3, 0.0),
             (100, 7, 0.0), (40, 6, 0.25), (100, 5, 2.0), (1, 1, 0.0)]
    for alpha in (0.0, 0.25, 0.5, 0.75, 1.0, 1.5, 2.0):
        fixed.append((100, 5, alpha))
    rng = random.Random(20240817)  # same seed as t/test_partition.py:43
    for _ in range(600):
        n = rng.randint(1, 10_000)
        s = rng.randint(1, 16)
        alpha = rng.uniform(-2.0, 2.0)
        if alpha == 0.0 and n < s:
            continue
        fixed.append((n, s, alpha))
    rng = random.Random(7)  # t/test_partition.py:55
    for _ in range(200):
        s = rng.randint(1, 16)
        n = rng.randint(s, 5000)
        fixed.append((n, s, 0.0))
    for n, s, a in fixed:
        out["generation"].append({"n": n, "stages": s, "alpha": a,
                                  "counts": split_generation(n, s, a)})
    rng = random.Random(5)  # t/test_partition.py:117
    pcases = [([1.0, 1.0, 1.0, 1.0], 2), ([3.0, 1.0, 1.0, 1.0], 2), ([2.0, 5.0, 1.0], 1)]
    for _ in range(200):
        n = rng.randint(1, 9)
        costs = [float(rng.randint(1, 20)) for _ in range(n)]
        pcases.append((costs, rng.randint(1, n)))
    for costs, st in pcases:
        out["perception"].append({"costs": costs, "stages": st,
                                  "ranges": [list(r) for r in split_perception(costs, st)]})
    # fault-hook golden (t/test_partition.py:96-99)
    os.environ["FRAMEPIPE_ROUNDING_FAULT"] = "truncate"
    try:
        out["fault_truncate"] = {"n": 100, "stages": 4, "alpha": 0.5,
                                 "counts": split_generation(100, 4, 0.5)}
    finally:
        del os.environ["FRAMEPIPE_ROUNDING_FAULT"]
    return out


def transformer_goldens():
    """Hidden states, logits and greedy tokens of the reference's float64
    CausalTransformer (fp/transformer.py:69-211) for the cases its own tests
    exercise (t/test_transformer.py:34-192, t/test_acceptance.py:61-90):
    prefills of random token strings over several seeds and shapes, a
    prefill + decode chain, a merged prefill over an [X_V; X_L; X_A] context."""
    from framepipe.context import ContextKind, PublicContext
    from framepipe.transformer import CausalTransformer, TransformerConfig
    out = {"configs": [], "prefill": [], "decode": [], "merged": []}
    shapes = [dict(), dict(seed=3), dict(d_model=32, n_heads=2, n_layers=2, vocab_size=50, max_len=64, seed=5),
              dict(d_model=48, n_heads=4, n_layers=3, vocab_size=40, max_len=96, seed=6)]
    rng = np.random.default_rng(20240911)
    for ci, kw in enumerate(shapes):
        cfg = TransformerConfig(**kw)
        model = CausalTransformer(cfg)
        out["configs"].append(kw)
        for n in (1, 2, 7, 24, 40):
            n = min(n, cfg.max_len)
            toks = rng.integers(0, cfg.vocab_size, n)
            h, cache = model.prefill(toks)
            out["prefill"].append({"config": ci, "tokens": [int(t) for t in toks], "hidden": h.tolist(),
                                   "logits_last": model.logits(h[-1]).tolist(),
                                   "greedy": [model.greedy_token(r) for r in h],
                                   "k_layer0_last": cache.keys[0][-1].ravel().tolist()})
        toks = rng.integers(0, cfg.vocab_size, 16)
        _, cache = model.prefill(toks[:-7])
        chain = []
        for t in toks[-7:]:
            hd, cache = model.decode(int(t), cache)
            chain.append(hd.tolist())
        out["decode"].append({"config": ci, "tokens": [int(t) for t in toks], "prefix": 9, "hidden": chain})
        d = cfg.d_model
        vision = rng.normal(0.0, 0.05, (16, d))
        language = rng.normal(0.0, 0.05, (8, d))
        atoks = tuple(int(x) for x in rng.integers(0, cfg.vocab_size, 5))
        ctx = PublicContext(kind=ContextKind.AUTOREGRESSIVE, vision_tokens=vision, language_tokens=language,
                            action_tokens=atoks, source_observation_id=0, produced_frame=0)
        pos = [24, 26, 28]
        mg = model.merged_generate(ctx, pos)
        out["merged"].append({"config": ci, "vision": vision.tolist(), "language": language.tolist(),
                              "action_tokens": list(atoks), "positions": pos,
                              "hidden": {str(p): mg[p].tolist() for p in pos}})
    return out


def edge_goldens():
    """Boundary runs the reference's tests touch (empty and one-frame runs in
    every mode, live reads, drop on overrun, alpha outside [0, 1]) and the
    configuration errors PipelineConfig.validate raises (fp/executor.py:72-92)."""
    cases = []
    for d in (0, 1, 2):
        cases.append(record_case(f"six_pipe_22_d{d}", "pipe", SIX, d, dict(pp_perception=2, pp_generation=2)))
        cases.append(record_case(f"six_seq_d{d}", "seq", SIX, d))
        cases.append(record_case(f"six_par_w2_d{d}", "par", SIX, d, workers=2))
        cases.append(record_case(f"six_dec_d{d}", "dec", SIX, d))
        cases.append(record_case(f"ar7_pipe_14_d{d}", "pipe", AR, d, dict(pp_perception=1, pp_generation=4)))
    cases.append(record_case("noisy16_pipe_14_live_m1", "pipe", NOISY16, 30,
                             dict(pp_perception=1, pp_generation=4, fetch_offset=-1, read_policy="live")))
    cases.append(record_case("noisy16_pipe_22_live_m2_k3", "pipe", NOISY16, 30,
                             dict(pp_perception=2, pp_generation=2, fetch_offset=-2, read_policy="live",
                                  store_capacity=3)))
    cases.append(record_case("multi_pipe_33_drop_i12", "pipe", MULTI, 40,
                             dict(pp_perception=3, pp_generation=3, frame_interval=12.0, overrun_policy="drop")))
    cases.append(record_case("multi_pipe_33_stretch_i12", "pipe", MULTI, 40,
                             dict(pp_perception=3, pp_generation=3, frame_interval=12.0)))
    cases.append(record_case("six_pipe_12_alpha1.5", "pipe", SIX, 20, dict(pp_perception=1, pp_generation=2, alpha=1.5)))
    cases.append(record_case("noisy16_pipe_14_alpha-0.5", "pipe", NOISY16, 30,
                             dict(pp_perception=1, pp_generation=4, alpha=-0.5)))
    errors = []
    for kw in (dict(pp_perception=1, pp_generation=2, fetch_offset=-2),
               dict(pp_perception=3, pp_generation=2),
               dict(pp_perception=1, pp_generation=5),
               dict(pp_perception=1, pp_generation=2, fetch_offset=1),
               dict(pp_perception=0, pp_generation=2),
               dict(pp_perception=1, pp_generation=0),
               dict(pp_perception=1, pp_generation=2, overrun_policy="skip"),
               dict(pp_perception=1, pp_generation=2, frame_interval=-1.0),
               dict(pp_perception=1, pp_generation=2, frame_interval=0.0),
               dict(pp_perception=1, pp_generation=2, store_capacity=1),
               dict(pp_perception=1, pp_generation=2, read_policy="bogus"),
               dict(pp_perception=1, pp_generation=2, fetch_offset=-3, store_capacity=3)):
        try:
            run_pipelined(PipelineConfig(**kw), make_conditioning_policy(**SIX), None, 4)
            errors.append({"pipeline": kw, "error": None})
        except Exception as e:                       # noqa: BLE001 -- recording the class
            errors.append({"pipeline": kw, "error": type(e).__name__})
    return {"cases": cases, "errors": errors}


AR = dict(autoregressive=True, layer_costs=(14.0, 14.0), l_a=7, prefill_cost=10.0, decode_cost=1.0)


def autoregressive_cases():
    """Token policy (fp/policy.py:300-327) through the merged-prefill schedule
    (fp/executor.py:321-348), sequential (:447-449), PAR and DEC (:670-672):
    SURVEY.md §8(f) row 3.  Mirrors t/test_executor.py:214-260 and
    t/test_acceptance.py:230-260, plus closed-loop runs."""
    cases = []
    for merge in (True, False):
        m = "m" if merge else "u"
        for l_a in (7, 14, 28):
            kw = dict(AR, l_a=l_a)
            cases.append(record_case(f"ar{l_a}_pipe_14_{m}", "pipe", kw, 40,
                                     dict(pp_perception=1, pp_generation=4, fetch_offset=-1,
                                          merge_autoregressive=merge)))
        cases.append(record_case(f"ar7_pipe_24_{m}", "pipe", AR, 40,
                                 dict(pp_perception=2, pp_generation=4, fetch_offset=-1,
                                      merge_autoregressive=merge)))
        cases.append(record_case(f"ar14_pipe_13_off0_{m}", "pipe", dict(AR, l_a=14), 40,
                                 dict(pp_perception=1, pp_generation=3, fetch_offset=0,
                                      merge_autoregressive=merge)))
    cases.append(record_case("ar7_pipe_12_snapshot", "pipe", AR, 40,
                             dict(pp_perception=1, pp_generation=2, fetch_offset=-2, read_policy="snapshot",
                                  store_capacity=4)))
    for l_a in (7, 14, 28):
        cases.append(record_case(f"ar{l_a}_seq", "seq", dict(AR, l_a=l_a), 30))
    cases.append(record_case("ar7_seq_i16", "seq", AR, 30, seq_interval=16.0))
    cases.append(record_case("ar7_pipe_14_m_env3", "pipe", AR, 120,
                             dict(pp_perception=1, pp_generation=4, fetch_offset=-1, merge_autoregressive=True),
                             env_seed=3))
    cases.append(record_case("ar7_seq_env3", "seq", AR, 60, env_seed=3))
    cases.append(record_case("ar7_par_w2_i8", "par", AR, 40, workers=2, seq_interval=8.0))
    cases.append(record_case("ar7_dec_i8", "dec", AR, 40, seq_interval=8.0))
    cases.append(record_case("ar7_dec_i32_env5", "dec", AR, 80, seq_interval=32.0, env_seed=5))
    return cases


def main():
    os.makedirs(OUT, exist_ok=True)
    with gzip.open(os.path.join(OUT, "transformer.json.gz"), "wt") as fh:
        json.dump({"generator": "oracle/make_golden.py", "reference": REF_SRC,
                   "numpy": np.__version__, **transformer_goldens()}, fh)
    print("wrote the transformer goldens")
    with gzip.open(os.path.join(OUT, "edge.json.gz"), "wt") as fh:
        json.dump({"generator": "oracle/make_golden.py", "reference": REF_SRC,
                   "numpy": np.__version__, **edge_goldens()}, fh)
    print("wrote the edge-case goldens")
    ar = autoregressive_cases()
    with gzip.open(os.path.join(OUT, "autoregressive.json.gz"), "wt") as fh:
        json.dump({"generator": "oracle/make_golden.py", "reference": REF_SRC,
                   "numpy": np.__version__, "cases": ar}, fh)
    print(f"wrote {len(ar)} autoregressive cases to {OUT}")
    with gzip.open(os.path.join(OUT, "partition.json.gz"), "wt") as fh:
        json.dump(partition_goldens(), fh)
    cases = schedule_cases()
    with gzip.open(os.path.join(OUT, "schedules.json.gz"), "wt") as fh:
        json.dump({"generator": "oracle/make_golden.py", "reference": REF_SRC,
                   "numpy": np.__version__, "cases": cases}, fh)
    print(f"wrote {len(cases)} schedule cases to {OUT}")
    base = baseline_cases()
    # comparison tables of the reference (fp/metrics.py:181-215) over recorded runs
    by = {c["name"]: c for c in cases + base}
    tables = []
    for names, bl in ((["six_seq", "six_pipe_24_m1", "six_par_w2", "six_dec"], 0),
                      (["noisy100_seq", "noisy100_pipe_18_off0", "noisy100_par_w8_i16", "noisy100_dec_i16"], 1),
                      (["cal_seq_env11", "cal_pipe_11_off0_env11"], 0)):
        from framepipe.metrics import RolloutMetrics
        runs = [RolloutMetrics.from_dict(by[n]["metrics"]) for n in names]
        t = compare(runs, names=names, baseline=bl)
        tables.append({"names": names, "baseline": bl, "json": t.to_json(), "csv": t.to_csv(),
                       "text": t.to_text()})
    with gzip.open(os.path.join(OUT, "baselines.json.gz"), "wt") as fh:
        json.dump({"generator": "oracle/make_golden.py", "reference": REF_SRC,
                   "numpy": np.__version__, "cases": base, "compare_tables": tables}, fh)
    print(f"wrote {len(base)} PAR/DEC cases to {OUT}")
    with gzip.open(os.path.join(OUT, "tuner.json.gz"), "wt") as fh:
        json.dump(tuner_golden(), fh)
    print("wrote the tuner golden")


if __name__ == "__main__":
    main()
