"""The numpy transformer oracle against hidden states recorded from the
reference (fp/transformer.py; tests/golden/transformer.json.gz)."""

import numpy as np
import pytest

from golden_util import load
from oracle import transformer as tfo

G = load("transformer")
TOL = 1e-12    # same fp64 math, numpy both sides: only BLAS blocking may differ


def _model(ci):
    return tfo.init_weights(**G["configs"][ci])


@pytest.mark.parametrize("i", range(len(G["prefill"])))
def test_prefill_matches_reference(i):
    case = G["prefill"][i]
    w = _model(case["config"])
    h, kv = tfo.prefill(w, case["tokens"])
    assert np.max(np.abs(h - np.array(case["hidden"]))) <= TOL
    assert np.max(np.abs(kv[0][0][-1].ravel() - np.array(case["k_layer0_last"]))) <= TOL
    assert np.max(np.abs(tfo.logits(w, h[-1]) - np.array(case["logits_last"]))) <= TOL
    assert [int(np.argmax(tfo.logits(w, r))) for r in h] == case["greedy"]


def test_decode_chain_is_prefill_tail():
    for case in G["decode"]:
        w = _model(case["config"])
        h, _ = tfo.prefill(w, case["tokens"])
        assert np.max(np.abs(h[case["prefix"]:] - np.array(case["hidden"]))) <= 1e-10


def test_merged_matches_reference():
    for case in G["merged"]:
        w = _model(case["config"])
        emb = np.concatenate([np.array(case["vision"]), np.array(case["language"]),
                              w["tok"][case["action_tokens"]]])
        h, _ = tfo.forward(w, emb)
        for p, want in case["hidden"].items():
            assert np.max(np.abs(h[int(p)] - np.array(want))) <= TOL
