"""Reference-style duck-typed policies under the B200 engine.

A user of the reference brings a Policy whose perception model has start /
apply_layers / finalize and whose generation model has initial_state / step /
finish (fp/policy.py:46-272).  run_pipelined / run_sequential accept such an
object (executor._require_plugin wraps it in policy.HostPolicy): the engine's
schedule, ring bookkeeping and stream ordering are unchanged and the policy's
callbacks run on the host.  The duck-typed objects here are the oracle's
restatement of the reference's toy policy (oracle/toy.py, pinned against the
reference in tests/test_oracle_golden.py), and every reference trace must come
out bit for bit, as for the device plugin (tests/test_gpu_toy.py)."""

import json

import pytest

from golden_util import ReplayEnv, autoregressive_cases, policy_kwargs, schedule_cases
from oracle import toy
from paper_2509_09560_b200 import (ConfigInvalid, PipelineConfig, run_decoupled, run_parallel, run_pipelined,
                                   run_sequential)
from paper_2509_09560_b200.policy import HostPolicy, Observation, is_reference_plugin

pytestmark = pytest.mark.gpu
CASES = schedule_cases()
AR_CASES = autoregressive_cases()


def _j(x):
    return json.loads(json.dumps(x))


def _strip(trace):
    out = _j(trace)
    for k in ("device", "clock"):
        out[0].pop(k, None)
    return out


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reference_style_policy_reproduces_reference_traces(case):
    pol = toy.ToyPolicy(**case["policy"])
    assert is_reference_plugin(pol) and not hasattr(pol, "open_session")
    env = ReplayEnv(case["env"], lambda f, v: Observation(frame=f, vector=v)) if case["env"] else None
    if case["mode"] == "pipe":
        res = run_pipelined(PipelineConfig(**case["pipeline"]), pol, env, case["duration"])
    else:
        res = run_sequential(pol, env, case["duration"], case["seq_interval"])
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches


@pytest.mark.parametrize("case", AR_CASES, ids=[c["name"] for c in AR_CASES])
def test_reference_style_token_policy_reproduces_reference_traces(case):
    # merged / per-stage prefill, the per-frame token update of the context, PAR and DEC
    _, kw = policy_kwargs(case)
    pol = toy.TokenPolicy(**kw)
    env = ReplayEnv(case["env"], lambda f, v: Observation(frame=f, vector=v)) if case["env"] else None
    if case["mode"] == "pipe":
        res = run_pipelined(PipelineConfig(**case["pipeline"]), pol, env, case["duration"])
    elif case["mode"] == "par":
        res = run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"], case["capacity"])
    elif case["mode"] == "dec":
        res = run_decoupled(pol, env, case["duration"], case["seq_interval"])
    else:
        res = run_sequential(pol, env, case["duration"], case["seq_interval"])
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]


def test_non_plugin_is_rejected():
    with pytest.raises(ConfigInvalid):
        run_pipelined(PipelineConfig(pp_perception=1, pp_generation=2), object(), None, 4)


def test_kind_is_normalised():
    class Kind:                       # an enum of another module (the reference's ContextKind)
        value = "conditioning"
    pol = toy.ToyPolicy()
    pol.kind = Kind()
    assert HostPolicy(pol).kind.value == "conditioning"
