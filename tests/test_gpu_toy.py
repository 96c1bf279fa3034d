"""Device engine + fp64 refinement policy vs the reference's golden traces.

Every case in tests/golden/schedules.json.gz was recorded from the unmodified
reference (oracle/make_golden.py).  The B200 engine must reproduce each trace
-- schedule, versions, ages, virtual times, and the fp64 actions computed by
the device kernels -- bit for bit, and the versions the device read in-kernel
must equal the versions the host schedule assigned.
"""

import collections
import json

import numpy as np
import pytest

from golden_util import ReplayEnv, schedule_cases
from paper_2509_09560_b200 import (ContextKind, ContextStore, KindMismatch, NotYetPublished, OffsetOutOfRange,
                                   PipelineConfig, PublicContext, StaleWrite,
                                   make_conditioning_policy, run_pipelined, run_sequential,
                                   summarize)
from paper_2509_09560_b200.policy import Observation

pytestmark = pytest.mark.gpu
CASES = schedule_cases()


def _j(x):
    return json.loads(json.dumps(x))


def _strip(trace):
    out = _j(trace)
    for k in ("device", "clock"):
        out[0].pop(k, None)
    return out


def _run(case, clock="virtual"):
    pol = make_conditioning_policy(**case["policy"])
    env = ReplayEnv(case["env"], lambda f, v: Observation(frame=f, vector=v)) if case["env"] else None
    if case["mode"] == "pipe":
        res = run_pipelined(PipelineConfig(**case["pipeline"]), pol, env, case["duration"], clock=clock)
    else:
        res = run_sequential(pol, env, case["duration"], case["seq_interval"], clock=clock)
    return res, env


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_trace_bit_exact_vs_reference(case):
    res, env = _run(case)
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches
    # the device read, in-kernel, exactly the versions the schedule assigned
    if case["mode"] == "pipe":
        for rec in case["trace"][1:]:
            if rec["generation"]:
                assert int(res.device_versions[rec["frame"]]) == rec["generation"][0]["context_version"]


def test_device_clock_keeps_schedule():
    case = next(c for c in CASES if c["name"] == "noisy100_pipe_15_off0")
    res, _ = _run(case, clock="device")
    got = [[(g["request"], g["stage"], g["iterations"], g["context_version"]) for g in r["generation"]]
           for r in res.trace[1:]]
    want = [[(g["request"], g["stage"], g["iterations"], g["context_version"]) for g in r["generation"]]
            for r in case["trace"][1:]]
    assert got == want
    assert [list(a.values) for a in res.actions] == case["actions"]
    m = summarize(res.trace)
    assert m.throughput > 0 and all(j > 0 for j in m.jct)
    ends = [r["end"] for r in res.trace[1:]]
    assert ends == sorted(ends)


def test_staleness_profile_offset_minus_one():
    # t/test_executor.py:76-83
    pol = make_conditioning_policy(layer_costs=(1.0,), n_iterations=100, step_cost=0.01)
    cfg = PipelineConfig(pp_perception=1, pp_generation=4, fetch_offset=-1, frame_interval=1.0)
    res = run_pipelined(cfg, pol, None, 30)
    prof = collections.Counter(res.actions[-1].staleness_profile)
    assert prof == {4.0: 25, 3.0: 25, 2.0: 25, 1.0: 25}


def test_throughput_law():
    # t/test_acceptance.py:95-116
    pol = make_conditioning_policy(layer_costs=(1.0, 1.0), n_iterations=4, step_cost=1.0)
    seq = summarize(run_sequential(pol, None, 60).trace)
    for pp_p, pp_g in ((2, 4), (1, 2)):
        m = summarize(run_pipelined(PipelineConfig(pp_perception=pp_p, pp_generation=pp_g,
                                                   fetch_offset=-1), pol, None, 60).trace)
        assert seq.mean_interval / m.mean_interval == float(pp_p + pp_g)
        assert m.pipeline_fill_frames == pp_p + pp_g - 1


class TestDeviceContextStore:
    """t/test_context_store.py:51-144 against the HBM ring."""

    @staticmethod
    def ctx(frame, value=1.0):
        return PublicContext(kind=ContextKind.CONDITIONING, source_observation_id=frame,
                             produced_frame=frame, conditioning=np.array([value, -value]))

    def test_first_publish_is_version_one(self):
        assert ContextStore().publish(self.ctx(0), 0) == 1

    def test_ring_semantics_and_payload(self):
        st = ContextStore(capacity=2)
        for f in range(3):
            st.publish(self.ctx(f, float(f)), f)
        got = st.fetch(2, -1)
        assert got.produced_frame == 1 and list(got.conditioning) == [1.0, -1.0]
        assert got.verify_checksum()

    def test_errors(self):
        st = ContextStore(capacity=2)
        with pytest.raises(NotYetPublished):
            st.fetch(0, 0)
        st.publish(self.ctx(5), 5)
        with pytest.raises(OffsetOutOfRange):
            st.fetch(5, -2)
        with pytest.raises(OffsetOutOfRange):
            st.fetch(5, 1)
        with pytest.raises(NotYetPublished):
            st.fetch(6, 0)
        with pytest.raises(StaleWrite):
            st.publish(self.ctx(4), 4)

    def test_same_frame_republish_supersedes(self):
        st = ContextStore()
        v1 = st.publish(self.ctx(0, 1.0), 0)
        v2 = st.publish(self.ctx(0, 2.0), 0)
        assert v2 > v1 and st.fetch(0, 0).conditioning[0] == 2.0

    def test_versions_strictly_increase_and_device_agrees(self):
        st = ContextStore(capacity=4)
        vs = [st.publish(self.ctx(f), f) for f in range(10)]
        assert vs == list(range(1, 11))
        assert st.device_state() == (10, 9, 10, 0)
        for off in (0, -1, -2, -3):
            assert st.fetch(9, off).produced_frame == 9 + off

    def test_update_action_tokens(self):
        """t/test_context_store.py token-update cases (fp/context.py:166-175)."""
        st = ContextStore(capacity=2)
        with pytest.raises(NotYetPublished):
            st.update_action_tokens(0, [1])
        st.publish(self.ctx(0), 0)
        with pytest.raises(KindMismatch):
            st.update_action_tokens(0, [1])
        vis = np.zeros((4, 8))
        vis[0, :2] = [0.25, -0.5]
        ar = PublicContext(kind=ContextKind.AUTOREGRESSIVE, source_observation_id=1, produced_frame=1,
                           vision_tokens=vis, language_tokens=np.zeros((2, 8)))
        v1 = st.publish(ar, 1)
        v2 = st.update_action_tokens(2, [3, 4, 5])
        assert v2 == v1 + 1
        got = st.fetch(2, 0)
        assert got.kind == ContextKind.AUTOREGRESSIVE and got.action_tokens == (3, 4, 5)
        assert got.produced_frame == 2 and got.source_observation_id == 1
        assert list(st.payload[0, st.slot_of(2)].cpu().numpy()) == [0.25, -0.5]
        assert st.fetch(2, -1).action_tokens == ()
        assert st.device_state()[:3] == (v2, 2, 3)
        with pytest.raises(StaleWrite):
            st.update_action_tokens(1, [1])


# ---------------------------------------------------------------- PAR / DEC baselines

from golden_util import baseline_cases  # noqa: E402
from paper_2509_09560_b200 import run_decoupled, run_parallel  # noqa: E402

BASE = baseline_cases()


@pytest.mark.parametrize("case", BASE, ids=[c["name"] for c in BASE])
def test_par_dec_bit_exact_vs_reference(case):
    """PAR and DEC (fp/executor.py:477-701) on the device engine: schedule,
    versions, ages, virtual times and the device-computed fp64 actions equal
    the reference's traces bit for bit (closed-loop cases replayed)."""
    pol = make_conditioning_policy(**case["policy"])
    env = ReplayEnv(case["env"], lambda f, v: Observation(frame=f, vector=v)) if case["env"] else None
    if case["mode"] == "par":
        res = run_parallel(pol, env, case["workers"], case["duration"], case["seq_interval"], case["capacity"])
    else:
        res = run_decoupled(pol, env, case["duration"], case["seq_interval"])
    assert _strip(res.trace) == case["trace"]
    assert [list(a.values) for a in res.actions] == case["actions"]
    assert [list(a.staleness_profile) for a in res.actions] == case["staleness_profiles"]
    assert [_j(vars(r)) for r in res.requests] == case["requests"]
    if env is not None:
        assert not env.mismatches
    if case["mode"] == "dec":
        got = [int(v) for v in res.device_versions[:len(res.requests)]]
        assert got == [r["context_versions"][0] for r in case["requests"]][:len(got)]


def test_par_dec_device_clock_runs():
    case = next(c for c in BASE if c["name"] == "noisy16_par_w4_i8")
    pol = make_conditioning_policy(**case["policy"])
    res = run_parallel(pol, None, case["workers"], case["duration"], case["seq_interval"], clock="device")
    assert [list(a.values) for a in res.actions] == case["actions"]
    case = next(c for c in BASE if c["name"] == "noisy16_dec_i8")
    res = run_decoupled(make_conditioning_policy(**case["policy"]), None, case["duration"], case["seq_interval"],
                        clock="device")
    assert [list(a.values) for a in res.actions] == case["actions"]
