"""Autoregressive token policy on the device engine.

Every case in tests/golden/autoregressive.json.gz was recorded from the
unmodified reference (oracle/make_golden.py): merged and per-stage prefill
(fp/executor.py:321-348), the per-frame token update of the public context
(:345-348), sequential, PAR and DEC, open- and closed-loop.  The B200 engine
must reproduce schedule, versions, prefill/decode accounting and the tokens
its kernels computed bit for bit.
"""

import json

import pytest

from golden_util import ReplayEnv, autoregressive_cases, policy_kwargs
from paper_2509_09560_b200 import (PipelineConfig, make_autoregressive_policy, run_decoupled,
                                   run_parallel, run_pipelined, run_sequential, summarize)
from paper_2509_09560_b200.policy import Observation

pytestmark = pytest.mark.gpu
CASES = autoregressive_cases()


def _j(x):
    return json.loads(json.dumps(x))


def _strip(trace):
    out = _j(trace)
    for k in ("device", "clock"):
        out[0].pop(k, None)
    return out


def _run(case, clock="virtual"):
    ar, kw = policy_kwargs(case)
    assert ar
    pol = make_autoregressive_policy(**kw)
    env = ReplayEnv(case["env"], lambda f, v: Observation(frame=f, vector=v)) if case["env"] else None
    if case["mode"] == "pipe":
        res = run_pipelined(PipelineConfig(**case["pipeline"]), pol, env, case["duration"], clock=clock)
    elif case["mode"] == "par":
        res = run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"],
                           case["capacity"], clock=clock)
    elif case["mode"] == "dec":
        res = run_decoupled(pol, env, case["duration"], case["seq_interval"], clock=clock)
    else:
        res = run_sequential(pol, env, case["duration"], case["seq_interval"], clock=clock)
    return res, env


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_ar_trace_bit_exact_vs_reference(case):
    res, env = _run(case)
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches
    assert json.loads(summarize(res.trace).to_json())["mean_interval"] == case["metrics"]["mean_interval"]


def test_ar_device_clock_same_tokens():
    case = next(c for c in CASES if c["name"] == "ar7_pipe_14_m_env3")
    res, env = _run(case, clock="device")
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert not env.mismatches


def test_ar_tokens_are_integers_in_schema():
    case = next(c for c in CASES if c["name"] == "ar7_seq_env3")
    res, _ = _run(case)
    for a in res.actions:
        v = list(a.values)
        assert all(isinstance(x, int) for x in v)
        assert v[0] in (0, 1, 2) and v[3] in (0, 1, 2) and v[6] == 0
        assert all(0 <= x <= 7 for x in (v[1], v[2], v[4], v[5]))
