"""numpy restatement of the reference's causal transformer (fp/transformer.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker for
paper_2509_09560_b200.transformer on inputs the golden fixtures do not hold.
Pinned against tests/golden/transformer.json.gz (tests/test_oracle_transformer.py).
"""

from __future__ import annotations

import numpy as np


def init_weights(d_model=64, n_heads=4, n_layers=4, vocab_size=64, max_len=256, seed=0):
    """Seeded initializer, fp/transformer.py:72-95 (same draw order)."""
    rng = np.random.default_rng(seed)
    s, d = 0.08, d_model
    w = {"tok": rng.normal(0.0, s, (vocab_size, d)), "pos": rng.normal(0.0, s, (max_len, d)),
         "h": n_heads, "layers": []}
    for _ in range(n_layers):
        layer = {k: rng.normal(0.0, s, (d, d)) for k in ("wq", "wk", "wv", "wo")}
        layer["w1"] = rng.normal(0.0, s, (d, 4 * d))
        layer["w2"] = rng.normal(0.0, s, (4 * d, d))
        w["layers"].append(layer)
    return w


def _ln(x):
    """fp/transformer.py:59-62 with unit gain / zero bias (the initializer's)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-5)


def _gelu(x):
    return 0.5 * x * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (x + 0.044715 * x ** 3)))


def forward(w, emb):
    """Hidden states and per-layer (k, v) of a full sequence (fp/transformer.py:115-143)."""
    x = np.asarray(emb, dtype=np.float64)
    m, d = x.shape
    h = w["h"]
    dh = d // h
    x = x + w["pos"][:m]
    mask = np.tril(np.ones((m, m), dtype=bool))
    kv = []
    for p in w["layers"]:
        a = _ln(x)
        q, k, v = ((a @ p[n]).reshape(m, h, dh) for n in ("wq", "wk", "wv"))
        kv.append((k, v))
        sc = np.einsum("qhd,khd->hqk", q, k) / np.sqrt(dh)
        sc = np.where(mask[None], sc, -np.inf)
        sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
        sc = sc / sc.sum(axis=-1, keepdims=True)
        x = x + np.einsum("hqk,khd->qhd", sc, v).reshape(m, d) @ p["wo"]
        x = x + _gelu(_ln(x) @ p["w1"]) @ p["w2"]
    return _ln(x), kv


def prefill(w, tokens):
    return forward(w, w["tok"][np.asarray(tokens, dtype=np.int64)])


def logits(w, hidden):
    return np.asarray(hidden) @ w["tok"].T
