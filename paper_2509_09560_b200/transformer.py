"""Causal pre-norm transformer with a KV cache in HBM (fp/transformer.py:1-211).

Same API as the reference's `CausalTransformer`: `prefill`, `prefill_embedded`,
`decode`, `merged_generate`, `context_embeddings`, `logits`, `greedy_token`,
with the same errors.  Every forward runs in `auras_tf_forward`
(csrc/transformer.cu): fp64 LayerNorm / causal attention / GELU MLP on the
device, the KV cache a [layers, 2, max_len, d] fp64 buffer that never leaves
HBM.  Weights come from the reference's seeded initializer (numpy
default_rng, same draw order), so a given seed is the same model.

A cache is a view `(buffer, length)`.  `decode` appends one row in place when
the cache is the buffer's newest view and copies the buffer first otherwise,
so old caches stay valid as in the reference's functional `decode`.

Row arithmetic is independent of the prefill length and of which launch
computes the row, so `merged_generate` equals separate shorter prefills bit
for bit (the reference guarantees 1e-5 relative).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .context import ContextKind, PublicContext
from .errors import DeviceError, KindMismatch, LengthExceeded


@dataclass(frozen=True)
class TransformerConfig:
    """fp/transformer.py:27-44."""

    d_model: int = 64
    n_heads: int = 4
    n_layers: int = 4
    vocab_size: int = 64
    max_len: int = 256
    seed: int = 0

    def __post_init__(self):
        if min(self.d_model, self.n_heads, self.n_layers, self.vocab_size, self.max_len) <= 0:
            raise ValueError("all transformer dimensions must be positive")
        if self.d_model % self.n_heads:
            raise ValueError("d_model must be divisible by n_heads")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


class _KvBuffer:
    def __init__(self, tensor):
        self.tensor = tensor     # [layers, 2, max_len, d] fp64 on the device
        self.tip = 0             # length of the newest cache view


class KvCache:
    """Keys / values of positions [0, length) (fp/transformer.py:47-56)."""

    def __init__(self, buffer: _KvBuffer | None = None, length: int = 0, n_heads: int = 1):
        self._buf = buffer
        self._length = length
        self._h = n_heads

    @property
    def length(self) -> int:
        return self._length

    def _host(self, which):
        if self._buf is None or self._length == 0:
            return []
        t = self._buf.tensor[:, which, :self._length].double().cpu().numpy()
        L, m, d = t.shape
        return [t[i].reshape(m, self._h, d // self._h) for i in range(L)]

    @property
    def keys(self) -> list:
        """Host copies, [m, H, hd] per layer."""
        return self._host(0)

    @property
    def values(self) -> list:
        return self._host(1)


class CausalTransformer:
    """fp/transformer.py:69-211 on the B200."""

    def __init__(self, config: TransformerConfig | None = None, device=None):
        import torch
        self.config = config or TransformerConfig()
        cfg = self.config
        # the reference initializer (fp/transformer.py:72-95), same draw order
        rng = np.random.default_rng(cfg.seed)
        s = 0.08
        d = cfg.d_model
        self.tok_emb = rng.normal(0.0, s, (cfg.vocab_size, d))
        self.pos_emb = rng.normal(0.0, s, (cfg.max_len, d))
        parts = [self.tok_emb.ravel(), self.pos_emb.ravel()]
        for _ in range(cfg.n_layers):
            wq, wk, wv, wo = (rng.normal(0.0, s, (d, d)) for _ in range(4))
            w1 = rng.normal(0.0, s, (d, 4 * d))
            w2 = rng.normal(0.0, s, (4 * d, d))
            parts += [np.ones(d), np.zeros(d), wq.ravel(), wk.ravel(), wv.ravel(), wo.ravel(),
                      np.ones(d), np.zeros(d), w1.ravel(), np.zeros(4 * d), w2.ravel(), np.zeros(d)]
        parts += [np.ones(d), np.zeros(d)]
        blob = np.concatenate(parts)
        self.lib = _lib.load()
        want = self.lib.auras_tf_param_count(d, cfg.n_heads, cfg.n_layers, cfg.vocab_size, cfg.max_len)
        if want != blob.size:
            raise DeviceError(f"parameter blob holds {blob.size} values, the kernel expects {want}")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.params = torch.from_numpy(blob).to(self.device)
        self.launches = 0

    # -- device forward -------------------------------------------------------

    def _dims(self):
        c = self.config
        return (c.d_model, c.n_heads, c.n_layers, c.vocab_size, c.max_len)

    def _forward(self, buf: _KvBuffer, start: int, ids=None, emb=None):
        """Rows [start, start + n) into `buf`; returns the device hidden states."""
        import torch
        n = int(ids.shape[0] if ids is not None else emb.shape[0])
        d = self.config.d_model
        resid = torch.empty(n, d, dtype=torch.float64, device=self.device)
        qbuf = torch.empty_like(resid)
        hidden = torch.empty_like(resid)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.auras_tf_forward(
            self.params.data_ptr(), *self._dims(),
            ids.data_ptr() if ids is not None else None,
            emb.data_ptr() if emb is not None else None,
            start, n, buf.tensor.data_ptr(), resid.data_ptr(), qbuf.data_ptr(), hidden.data_ptr(), stream),
            "tf_forward")
        self.launches += self.config.n_layers + 1
        buf.tip = start + n
        return hidden

    def _new_buffer(self):
        import torch
        c = self.config
        return _KvBuffer(torch.empty(c.n_layers, 2, c.max_len, c.d_model, dtype=torch.float64,
                                     device=self.device))

    def _check_len(self, m):
        if m < 1:
            raise ValueError("prefill requires at least one token")
        if m > self.config.max_len:
            raise LengthExceeded(f"sequence length {m} > max {self.config.max_len}")

    def prefill_device(self, token_ids=None, embeddings=None):
        """Device-resident prefill: (hidden [m, d] fp64 tensor, KvCache)."""
        import torch
        buf = self._new_buffer()
        if token_ids is not None:
            ids = torch.as_tensor(token_ids, dtype=torch.int32).to(self.device)
            self._check_len(int(ids.shape[0]))
            hidden = self._forward(buf, 0, ids=ids)
        else:
            emb = torch.as_tensor(embeddings, dtype=torch.float64).to(self.device).contiguous()
            self._check_len(int(emb.shape[0]))
            if emb.dim() != 2 or emb.shape[1] != self.config.d_model:
                raise ValueError("embedding width must equal d_model")
            hidden = self._forward(buf, 0, emb=emb)
        return hidden, KvCache(buf, buf.tip, self.config.n_heads)

    # -- reference API ----------------------------------------------------------

    def embed_tokens(self, token_ids) -> np.ndarray:
        ids = np.asarray(token_ids, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= self.config.vocab_size):
            raise ValueError("token id outside vocabulary")
        return self.tok_emb[ids]

    def prefill(self, token_ids):
        ids = np.asarray(token_ids, dtype=np.int64).reshape(-1)
        self._check_len(ids.size)
        self.embed_tokens(ids)
        hidden, cache = self.prefill_device(token_ids=ids)
        return hidden.cpu().numpy(), cache

    def prefill_embedded(self, embeddings):
        x = np.asarray(embeddings, dtype=np.float64)
        m = x.shape[0]
        self._check_len(m)
        if x.ndim != 2 or x.shape[1] != self.config.d_model:
            raise ValueError("embedding width must equal d_model")
        hidden, cache = self.prefill_device(embeddings=x)
        return hidden.cpu().numpy(), cache

    def decode(self, token_id: int, cache: KvCache):
        """fp/transformer.py:147-173; the old cache stays valid."""
        import torch
        if cache is None or cache.length == 0:
            raise ValueError("decode requires a cache produced by prefill")
        m = cache.length
        if m + 1 > self.config.max_len:
            raise LengthExceeded(f"cache full at max length {self.config.max_len}")
        self.embed_tokens([token_id])
        buf = cache._buf
        if buf.tip != m:           # someone already extended this view: copy on write
            nb = self._new_buffer()
            nb.tensor[:, :, :m].copy_(buf.tensor[:, :, :m])
            buf = nb
        ids = torch.tensor([int(token_id)], dtype=torch.int32, device=self.device)
        hidden = self._forward(buf, m, ids=ids)
        return hidden[0].cpu().numpy(), KvCache(buf, m + 1, self.config.n_heads)

    def context_embeddings(self, ctx: PublicContext) -> np.ndarray:
        """[X_V; X_L; embed(X_A)] (fp/transformer.py:195-203)."""
        if ctx.kind != ContextKind.AUTOREGRESSIVE:
            raise KindMismatch("token embeddings only exist on autoregressive contexts")
        parts = [np.asarray(ctx.vision_tokens, dtype=np.float64),
                 np.asarray(ctx.language_tokens, dtype=np.float64)]
        if ctx.action_tokens:
            parts.append(self.embed_tokens(list(ctx.action_tokens)))
        return np.concatenate(parts, axis=0)

    def merged_generate(self, ctx: PublicContext, positions) -> dict:
        """One device prefill over the whole public context serving every
        requested action position (fp/transformer.py:175-193)."""
        if ctx.kind != ContextKind.AUTOREGRESSIVE:
            raise KindMismatch("merged generation requires an autoregressive context")
        emb = self.context_embeddings(ctx)
        l = emb.shape[0] - len(ctx.action_tokens)
        total = emb.shape[0]
        positions = sorted(set(int(p) for p in positions))
        for p in positions:
            if not (l <= p < total):
                raise ValueError(f"position {p} outside action region [{l}, {total})")
        hidden, _ = self.prefill_embedded(emb)
        return {p: hidden[p] for p in positions}

    def _logits_device(self, hidden):
        import torch
        h = torch.as_tensor(np.asarray(hidden, dtype=np.float64)).to(self.device)
        squeeze = h.dim() == 1
        h = h.reshape(-1, self.config.d_model).contiguous()
        n = h.shape[0]
        out = torch.empty(n, self.config.vocab_size, dtype=torch.float64, device=self.device)
        best = torch.empty(n, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.auras_tf_logits(self.params.data_ptr(), self.config.d_model, self.config.vocab_size,
                                            h.data_ptr(), n, out.data_ptr(), best.data_ptr(),
                                            torch.cuda.current_stream(self.device).cuda_stream), "tf_logits")
        self.launches += 1
        return out, best, squeeze

    def logits(self, hidden) -> np.ndarray:
        out, _, squeeze = self._logits_device(hidden)
        out = out.cpu().numpy()
        return out[0] if squeeze else out

    def greedy_token(self, hidden) -> int:
        _, best, _ = self._logits_device(hidden)
        return int(best[0].item())
