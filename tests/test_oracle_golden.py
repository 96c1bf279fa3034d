"""Pin the CPU oracle against the reference-recorded goldens (no GPU).

The oracle (oracle/schedule.py, oracle/toy.py) must reproduce every schema-1
trace the unmodified reference produced -- frame times, stage activations,
context versions, staleness, emitted fp64 actions -- bit for bit.
"""

import json
import os

import numpy as np
import pytest

from golden_util import ReplayEnv, baseline_cases, load, schedule_cases
from oracle import schedule as osched
from oracle import toy


def _jsonify(x):
    return json.loads(json.dumps(x))


CASES = schedule_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_reproduces_reference_trace(case):
    pol = toy.ToyPolicy(**case["policy"])
    env = ReplayEnv(case["env"], toy.Obs) if case["env"] else None
    if case["mode"] == "pipe":
        res = osched.run_pipelined(case["pipeline"], pol, env, case["duration"])
    else:
        res = osched.run_sequential(pol, env, case["duration"], case["seq_interval"])
    assert _jsonify(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_jsonify(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches


BASE = baseline_cases()


@pytest.mark.parametrize("case", BASE, ids=[c["name"] for c in BASE])
def test_oracle_reproduces_reference_par_dec(case):
    """PAR and DEC baselines restated in the oracle."""
    pol = toy.ToyPolicy(**case["policy"])
    env = ReplayEnv(case["env"], toy.Obs) if case["env"] else None
    if case["mode"] == "par":
        res = osched.run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"],
                                  case["capacity"])
    else:
        res = osched.run_decoupled(pol, env, case["duration"], case["seq_interval"])
    assert _jsonify(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_jsonify(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches


def test_oracle_partition_goldens(monkeypatch):
    g = load("partition")
    for c in g["generation"]:
        assert osched.split_generation(c["n"], c["stages"], c["alpha"]) == c["counts"]
    for c in g["perception"]:
        assert [list(r) for r in osched.split_perception(c["costs"], c["stages"])] == c["ranges"]
    f = g["fault_truncate"]
    monkeypatch.setenv("FRAMEPIPE_ROUNDING_FAULT", "truncate")
    assert osched.split_generation(f["n"], f["stages"], f["alpha"]) == f["counts"]


def test_toy_closed_forms():
    # t/test_policy.py:62-94 closed forms, restated against the oracle toy
    eta, n, k = 0.08, 100, 30
    beta = 1.0 - eta
    pol = toy.ToyPolicy(eta=eta, n_iterations=n, max_action=10.0)
    c1, c2 = np.array([1.0, 0.5]), np.array([-0.3, 0.8])
    s = pol.generation.initial_state()
    for _ in range(k):
        s = pol.generation.step(s, toy.Ctx(c1, 0))
    for _ in range(n - k):
        s = pol.generation.step(s, toy.Ctx(c2, 1))
    want = c2 + beta ** (n - k) * ((1.0 - beta ** k) * c1 - c2)
    assert np.allclose(s.vector, want, rtol=1e-12)



CLOSED = [c for c in CASES + BASE if c["env"]]


@pytest.mark.parametrize("case", CLOSED, ids=[c["name"] for c in CLOSED])
def test_oracle_env_closes_the_loop_like_the_reference(case):
    """oracle/envsim.py restates fp/envsim.py: running the oracle schedule in
    a real closed loop with it (not a replay) reproduces the reference's
    recorded trace, observations and sealed errors bit for bit."""
    from oracle import envsim
    rec = case["env"]
    env = envsim.tracking_env(rec["seed"], **rec["kw"])
    assert env.success_threshold == rec["success_threshold"]
    pol = toy.ToyPolicy(**case["policy"])
    if case["mode"] == "pipe":
        res = osched.run_pipelined(case["pipeline"], pol, env, case["duration"])
    elif case["mode"] == "seq":
        res = osched.run_sequential(pol, env, case["duration"], case["seq_interval"])
    elif case["mode"] == "par":
        res = osched.run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"],
                                  case["capacity"])
    else:
        res = osched.run_decoupled(pol, env, case["duration"], case["seq_interval"])
    assert _jsonify(res.trace) == case["trace"]
    assert env.errors == rec["errors"]


from golden_util import autoregressive_cases, policy_kwargs  # noqa: E402

AR_CASES = autoregressive_cases()


@pytest.mark.parametrize("case", AR_CASES, ids=[c["name"] for c in AR_CASES])
def test_oracle_reproduces_reference_autoregressive(case):
    """Token policy through the merged / per-stage prefill schedule, the
    per-frame token update, sequential, PAR and DEC."""
    ar, kw = policy_kwargs(case)
    assert ar
    pol = toy.TokenPolicy(**kw)
    env = ReplayEnv(case["env"], toy.Obs) if case["env"] else None
    if case["mode"] == "pipe":
        res = osched.run_pipelined(case["pipeline"], pol, env, case["duration"])
    elif case["mode"] == "par":
        res = osched.run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"],
                                  case["capacity"])
    elif case["mode"] == "dec":
        res = osched.run_decoupled(pol, env, case["duration"], case["seq_interval"])
    else:
        res = osched.run_sequential(pol, env, case["duration"], case["seq_interval"])
    assert _jsonify(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_jsonify(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches


def test_token_schema_matches_reference_examples():
    """t/test_policy.py:150-205: encode / decode round trip within a bucket."""
    enc = toy.encode_action_tokens((0.25, -0.1), 0.8)
    assert len(enc) == 7 and enc[6] == 0 and enc[0] == 1 and enc[3] == 2
    back = toy.decode_action_tokens(enc, 0.8)
    assert np.allclose(back, [0.25, -0.1], atol=0.8 / 63)
    assert np.allclose(toy.decode_action_tokens(toy.encode_action_tokens((5.0, -5.0), 0.8), 0.8), [0.8, -0.8])
    assert toy.encode_action_tokens((0.0, 0.0), 0.8) == (0,) * 7
    assert toy.encode_action_tokens((0.3, 0.3), 0.8, 14)[7:] == toy.encode_action_tokens((0.3, 0.3), 0.8)


from golden_util import edge_goldens  # noqa: E402

EDGE = edge_goldens()


def _oracle_run(case):
    ar, kw = policy_kwargs(case)
    pol = toy.TokenPolicy(**kw) if ar else toy.ToyPolicy(**kw)
    env = ReplayEnv(case["env"], toy.Obs) if case["env"] else None
    if case["mode"] == "pipe":
        return osched.run_pipelined(case["pipeline"], pol, env, case["duration"]), env
    if case["mode"] == "par":
        return osched.run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"],
                                   case["capacity"]), env
    if case["mode"] == "dec":
        return osched.run_decoupled(pol, env, case["duration"], case["seq_interval"]), env
    return osched.run_sequential(pol, env, case["duration"], case["seq_interval"]), env


@pytest.mark.parametrize("case", EDGE["cases"], ids=[c["name"] for c in EDGE["cases"]])
def test_oracle_edge_cases(case):
    res, env = _oracle_run(case)
    assert _jsonify(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [_jsonify(vars(r)) for r in res.requests] == case["requests"]


@pytest.mark.parametrize("case", EDGE["cases"], ids=[c["name"] for c in EDGE["cases"]])
def test_summarize_edge_cases(case):
    """summarize on the reference's own traces, incl. EmptyTrace on 0-frame runs."""
    from paper_2509_09560_b200 import summarize
    from paper_2509_09560_b200.errors import EmptyTrace
    if "error" in case["metrics"]:
        assert case["metrics"]["error"] == "EmptyTrace"
        with pytest.raises(EmptyTrace):
            summarize(case["trace"])
    else:
        got = json.loads(summarize(case["trace"]).to_json())
        for k, v in case["metrics"].items():
            assert got[k] == v, k


@pytest.mark.parametrize("err", EDGE["errors"], ids=[str(i) for i in range(len(EDGE["errors"]))])
def test_config_errors_match_reference(err):
    """PipelineConfig.validate + the partitioner raise the reference's error
    class (fp/executor.py:72-92, fp/partition.py); the store-capacity
    ValueError comes from the device ring and is checked on the GPU."""
    from paper_2509_09560_b200 import PipelineConfig, errors, make_conditioning_policy, plan_stages
    if err["pipeline"].get("store_capacity") == 1:
        pytest.skip("raised by the device ContextStore (tests/test_gpu_edge.py)")
    pol = make_conditioning_policy(layer_costs=(1.0, 1.0), n_iterations=4, step_cost=1.0)
    cls = getattr(errors, err["error"])
    with pytest.raises(cls):
        cfg = PipelineConfig(**err["pipeline"])
        cfg.validate(pol)
        plan_stages(pol.perception.layer_costs, cfg.pp_perception, pol.generation.n_iterations,
                    cfg.pp_generation, cfg.alpha)
