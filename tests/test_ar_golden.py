"""CPU checks on the reference-recorded autoregressive goldens: the merged
prefill properties the reference's own tests assert
(t/test_executor.py:214-260, t/test_acceptance.py:230-260) hold in the
fixtures the GPU tests replay, and the host-side token schema decodes them
exactly as fp/policy.py:135-148 does."""

import numpy as np

from golden_util import autoregressive_cases
from paper_2509_09560_b200.policy import ACTION_TOKEN_COUNT, decode_action_tokens

BY = {c["name"]: c for c in autoregressive_cases()}


def _steady(case, stages):
    return [f for f in case["trace"][1:] if len(f["generation"]) == stages]


def test_merged_frames_charge_one_prefill():
    for l_a in (7, 14, 28):
        st = _steady(BY[f"ar{l_a}_pipe_14_m"], 4)
        assert st and all(f["prefill_calls"] == 1 and f["generation_cost"] == 10.0 for f in st)
        st = _steady(BY[f"ar{l_a}_pipe_14_u"], 4)
        assert st and all(f["prefill_calls"] == 4 and f["decode_calls"] == l_a - 4 for f in st)


def test_merged_interval_invariant_and_sequential_affine():
    iv = [BY[f"ar{l}_pipe_14_m"]["metrics"]["mean_interval"] for l in (7, 14, 28)]
    assert iv[0] == iv[1] == iv[2]
    sq = {l: BY[f"ar{l}_seq"]["metrics"]["mean_interval"] for l in (7, 14, 28)}
    assert sq[14] - sq[7] == 7.0 and sq[28] - sq[14] == 14.0


def test_applied_actions_decode_from_tokens():
    case = BY["ar7_seq_env3"]
    for toks, applied in zip(case["actions"], case["env"]["applied"]):
        vec = decode_action_tokens([int(t) for t in toks[:ACTION_TOKEN_COUNT]], 0.8)
        n = float(np.linalg.norm(vec))
        if n > 0.8:
            vec = vec * (0.8 / n)
        assert [float(x) for x in vec] == applied
