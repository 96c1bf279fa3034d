"""Boundary runs on the device engine against the reference (tests/golden/edge.json.gz):
empty and one-frame runs in every mode, live reads, drop on overrun, alpha
outside [0, 1], and the reference's configuration errors."""

import json

import pytest

from golden_util import edge_goldens, policy_kwargs
from paper_2509_09560_b200 import (PipelineConfig, errors, make_autoregressive_policy, make_conditioning_policy,
                                   run_decoupled, run_parallel, run_pipelined, run_sequential)

pytestmark = pytest.mark.gpu
EDGE = edge_goldens()


def _j(x):
    return json.loads(json.dumps(x))


def _strip(trace):
    out = _j(trace)
    for k in ("device", "clock"):
        out[0].pop(k, None)
    return out


@pytest.mark.parametrize("case", EDGE["cases"], ids=[c["name"] for c in EDGE["cases"]])
def test_edge_cases_bit_exact(case):
    ar, kw = policy_kwargs(case)
    pol = make_autoregressive_policy(**kw) if ar else make_conditioning_policy(**kw)
    if case["mode"] == "pipe":
        res = run_pipelined(PipelineConfig(**case["pipeline"]), pol, None, case["duration"])
    elif case["mode"] == "par":
        res = run_parallel(pol, None, case["workers"], case["duration"], case["seq_interval"], case["capacity"])
    elif case["mode"] == "dec":
        res = run_decoupled(pol, None, case["duration"], case["seq_interval"])
    else:
        res = run_sequential(pol, None, case["duration"], case["seq_interval"])
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]


@pytest.mark.parametrize("err", EDGE["errors"], ids=[str(i) for i in range(len(EDGE["errors"]))])
def test_config_errors_match_reference(err):
    pol = make_conditioning_policy(layer_costs=(1.0, 1.0), n_iterations=4, step_cost=1.0)
    cls = ValueError if err["error"] == "ValueError" else getattr(errors, err["error"])
    with pytest.raises(cls):
        run_pipelined(PipelineConfig(**err["pipeline"]), pol, None, 4)
