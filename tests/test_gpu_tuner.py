"""Configuration search (fp/tuner.py) on the B200 engine.

Virtual clock: the engine's traces are bit-exact, so grid_search and
finetune_alpha with the toy policy and closed-loop tracking rollouts must
return the reference's recorded TuneResult exactly (tests/golden/tuner.json.gz,
oracle/make_golden.py); the rollouts use oracle/envsim.py, the restated
reference environment (pinned in tests/test_oracle_golden.py).
Device clock: the same search with throughput measured on the GPU."""

import json

import numpy as np
import pytest

from golden_util import load
from oracle import envsim
from paper_2509_09560_b200 import (NoFeasibleConfig, TuneRequest, finetune_alpha, grid_search,
                                   make_conditioning_policy)
from paper_2509_09560_b200.policy import Observation

pytestmark = pytest.mark.gpu


def _factory(frames):
    return lambda seed: envsim.tracking_env(seed, frames=frames, obs_factory=lambda f, v: Observation(frame=f, vector=v))


def _req(d, **kw):
    d = dict(d, **kw)
    for k in ("alpha_grid", "seeds"):
        d[k] = tuple(d[k])
    return TuneRequest(**d)


def _j(x):
    return json.loads(json.dumps(x))


def test_tuner_matches_reference_exactly():
    g = load("tuner")
    pol = make_conditioning_policy(**g["policy"])
    req = _req(g["request"])
    res = grid_search(pol, _factory(g["env_frames"]), req)
    assert _j(res.to_dict()) == g["grid"]
    fin = finetune_alpha(pol, _factory(g["env_frames"]), res.chosen, req)
    assert _j(fin.to_dict()) == g["alpha"]
    with pytest.raises(NoFeasibleConfig) as exc:
        grid_search(pol, _factory(g["env_frames"]), _req(g["request"], throughput_requirement=5.0))
    assert str(exc.value) == g["infeasible"]["message"]
    assert _j(exc.value.result.to_dict()) == g["infeasible"]["result"]


def test_tuner_on_measured_device_throughput():
    """clock="device": each grid point's throughput is actions/s of the real
    kernels.  The grid points of the toy policy run within ~10% of each other,
    so the requirement is set clear of timing noise on both sides: below every
    measured point (all feasible, ranked by tracking error) and above every
    point (NoFeasibleConfig carrying the measured result)."""
    g = load("tuner")
    pol = make_conditioning_policy(**g["policy"])
    probe = grid_search(pol, _factory(g["env_frames"]), _req(g["request"], throughput_requirement=1e-9),
                        clock="device")
    thr = sorted(p.throughput for p in probe.evaluated)
    assert thr[0] > 0
    req = _req(g["request"], throughput_requirement=0.5 * thr[0])
    res = grid_search(pol, _factory(g["env_frames"]), req, clock="device")
    assert 0 < len(res.ranked) <= len(res.evaluated)
    assert all(p.throughput >= req.throughput_requirement for p in res.ranked)
    errs = [p.mean_error for p in res.ranked]
    assert errs == sorted(errs)
    with pytest.raises(NoFeasibleConfig) as exc:
        grid_search(pol, _factory(g["env_frames"]), _req(g["request"], throughput_requirement=3.0 * thr[-1]),
                    clock="device")
    assert len(exc.value.result.evaluated) == len(probe.evaluated)
