"""Device causal transformer (csrc/transformer.cu) vs the reference.

Golden hidden states / KV rows / logits / greedy tokens recorded from the
reference's float64 CausalTransformer (tests/golden/transformer.json.gz) and
the numpy oracle (oracle/transformer.py, pinned to those goldens) on random
inputs.  Tolerance: 1e-11 absolute on O(1) fp64 hidden states (the device
sums in another order than numpy's BLAS); the reference's own bar is 1e-5
relative (t/test_transformer.py:8).  The merge / prefix / decode / isolation
properties the reference checks within tolerance hold bit-exactly here and
are asserted with array_equal.
"""

import numpy as np
import pytest

from golden_util import load
from oracle import transformer as tfo
from paper_2509_09560_b200 import (CausalTransformer, ContextKind, KindMismatch, KvCache, LengthExceeded,
                                   PublicContext, TransformerConfig)

pytestmark = pytest.mark.gpu
G = load("transformer")
TOL = 1e-11
_MODELS = {}


def model(ci=0, **kw):
    key = (ci, tuple(sorted(kw.items())))
    if key not in _MODELS:
        cfg = TransformerConfig(**(G["configs"][ci] if ci is not None else kw))
        _MODELS[key] = CausalTransformer(cfg)
    return _MODELS[key]


def close(a, b, tol=TOL):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) <= tol


@pytest.mark.parametrize("i", range(len(G["prefill"])))
def test_prefill_matches_reference_golden(i):
    case = G["prefill"][i]
    m = model(case["config"])
    h, cache = m.prefill(case["tokens"])
    assert close(h, case["hidden"])
    assert cache.length == len(case["tokens"])
    assert close(cache.keys[0][-1].ravel(), case["k_layer0_last"])
    assert close(m.logits(h[-1]), case["logits_last"])
    lg = np.array([m.logits(r) for r in h])
    for row, want in zip(lg, case["greedy"]):
        top = np.sort(row)[-2:]
        if top[1] - top[0] > 1e-9:
            assert int(np.argmax(row)) == want
    assert [m.greedy_token(r) for r in h] == [int(np.argmax(r)) for r in lg]


def test_decode_chain_matches_reference_golden():
    for case in G["decode"]:
        m = model(case["config"])
        toks = case["tokens"]
        _, cache = m.prefill(toks[:case["prefix"]])
        for t, want in zip(toks[case["prefix"]:], case["hidden"]):
            h, cache = m.decode(t, cache)
            assert close(h, want)


def test_merged_generate_matches_reference_golden():
    for case in G["merged"]:
        m = model(case["config"])
        ctx = PublicContext(kind=ContextKind.AUTOREGRESSIVE, vision_tokens=np.array(case["vision"]),
                            language_tokens=np.array(case["language"]),
                            action_tokens=tuple(case["action_tokens"]), source_observation_id=0,
                            produced_frame=0)
        got = m.merged_generate(ctx, case["positions"])
        for p, want in case["hidden"].items():
            assert close(got[int(p)], want)
        # merged == separate shorter prefills, bit for bit
        emb = m.context_embeddings(ctx)
        for p in case["positions"]:
            sep, _ = m.prefill_embedded(emb[:p + 1])
            assert np.array_equal(sep[-1], got[p])


def test_randomized_vs_oracle_and_exact_merge():
    """t/test_acceptance.py:61-90 on the device: 100 (model, tokens, cut)
    triples; device vs oracle within TOL, merged vs separate exact."""
    rng = np.random.default_rng(20240911)
    w = {s: tfo.init_weights(seed=s) for s in range(5)}
    ms = {s: model(None, seed=s) for s in range(5)}
    for _ in range(100):
        s = int(rng.integers(0, 5))
        n = int(rng.integers(2, 40))
        toks = rng.integers(0, 64, n)
        cut = int(rng.integers(1, n))
        merged, _ = ms[s].prefill(toks)
        separate, _ = ms[s].prefill(toks[:cut])
        assert np.array_equal(merged[:cut], separate)
        want, _ = tfo.prefill(w[s], toks)
        assert close(merged, want)


def test_long_sequences_to_max_len():
    m = model(0)
    w = tfo.init_weights()
    toks = np.random.default_rng(1).integers(0, 64, 256)
    h, cache = m.prefill(toks)
    want, kv = tfo.prefill(w, toks)
    assert close(h, want)
    assert close(cache.values[3], kv[3][1])
    with pytest.raises(LengthExceeded):
        m.decode(1, cache)


def test_causal_isolation_exact():
    m = model(0)
    toks = np.random.default_rng(5).integers(0, 64, 20)
    base, _ = m.prefill(toks)
    for q in (10, 15, 19):
        mut = toks.copy()
        mut[q] = (mut[q] + 13) % 64
        changed, _ = m.prefill(mut)
        assert np.array_equal(base[:q], changed[:q])
        assert not np.array_equal(base[q], changed[q])


def test_decode_equals_longer_prefill_exactly_and_old_caches_stay_valid():
    m = model(0)
    toks = np.random.default_rng(3).integers(0, 64, 16)
    full, _ = m.prefill(toks)
    _, cache = m.prefill(toks[:-7])
    c0 = cache
    for i, t in enumerate(toks[-7:]):
        h, cache = m.decode(int(t), cache)
        assert np.array_equal(h, full[9 + i])
        assert cache.length == 10 + i
    # a second decode from an old view copies instead of clobbering the newer one
    h_alt, alt = m.decode(int((toks[9] + 1) % 64), c0)
    h_again, _ = m.decode(int(toks[10]), alt)
    h_ref, _ = m.decode(int(toks[-1]), KvCache(cache._buf, 15, 4))
    assert np.array_equal(h_ref, full[15])
    alt_full, _ = m.prefill(np.concatenate([toks[:9], [(toks[9] + 1) % 64, toks[10]]]))
    assert np.array_equal(h_alt, alt_full[9]) and np.array_equal(h_again, alt_full[10])


def test_determinism_and_seeds():
    a = CausalTransformer(TransformerConfig(seed=7))
    b = CausalTransformer(TransformerConfig(seed=7))
    c = CausalTransformer(TransformerConfig(seed=8))
    t = np.arange(10) % 64
    assert np.array_equal(a.prefill(t)[0], b.prefill(t)[0])
    assert not np.array_equal(a.prefill(t)[0], c.prefill(t)[0])


def test_errors():
    m = model(0)
    with pytest.raises(ValueError):
        m.prefill([])
    with pytest.raises(LengthExceeded):
        m.prefill(np.zeros(257, dtype=int))
    with pytest.raises(ValueError):
        m.prefill([64])
    with pytest.raises(ValueError):
        m.decode(3, KvCache())
    small = CausalTransformer(TransformerConfig(max_len=4))
    _, cache = small.prefill([1, 2, 3, 4])
    with pytest.raises(LengthExceeded):
        small.decode(5, cache)
    with pytest.raises(KindMismatch):
        m.merged_generate(PublicContext(kind=ContextKind.CONDITIONING, conditioning=np.zeros(2),
                                        source_observation_id=0, produced_frame=0), [0])
    ctx = PublicContext(kind=ContextKind.AUTOREGRESSIVE, vision_tokens=np.zeros((3, 64)),
                        language_tokens=np.zeros((2, 64)), action_tokens=(1, 2),
                        source_observation_id=0, produced_frame=0)
    with pytest.raises(ValueError):
        m.merged_generate(ctx, [0])
    with pytest.raises(ValueError):
        TransformerConfig(d_model=65, n_heads=4)
