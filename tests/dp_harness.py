"""Device harness shared by the parity tests and __graft_entry__.smoke():
one DPSession.generate call (the frame's batched denoise launch) on chosen
inputs, and the same samples through the bf16-faithful oracle
(oracle/dp_model.py, test infrastructure)."""

import numpy as np
import torch

from oracle import dp_model
from paper_2509_09560_b200 import diffusion as D

_W = {}


def weights(name, seed=0):
    if (name, seed) not in _W:
        _W[(name, seed)] = D.init_weights(D.PRESETS[name], seed, device="cpu")
    return _W[(name, seed)]


def _plan(S, n_steps, rng):
    """S (start, count) pairs: distinct starting steps spread over the whole
    schedule, counts 1..3 (unequal inside one launch), start + count <= n."""
    starts = rng.permutation(n_steps - 3)[:S] if S <= n_steps - 3 else rng.integers(0, n_steps - 3, S)
    counts = rng.integers(1, 4, S)
    return [(int(s), int(c)) for s, c in zip(starts, counts)]


def run_denoise_launch(cfg_name, S, agents=1, seed=0, w=None):
    """One DPSession.generate call (one denoise launch per iteration chain of
    the frame) over S samples on the device, and the same samples through the
    bf16-faithful oracle.  Returns (device x, oracle x, x_in, kernel id).
    `w`: weights to use instead of the seeded preset weights."""
    cfg = D.PRESETS[cfg_name]
    w = weights(cfg_name) if w is None else w
    pol = D.make_diffusion_policy(cfg_name, dtype="bf16", weights=w, agents=agents)
    lanes = -(-S // agents)
    P, G = torch.cuda.Stream(), torch.cuda.Stream()
    sess = pol.generation.open_session(pol, capacity=2, lanes=lanes, agents=agents, max_outputs=2,
                                       max_frames=2, p_stream=P, g_stream=G)
    try:
        obs = [D.synthetic_frame(cfg, 0, a, 0) for a in range(agents)]
        sess.ingest(0, 0, obs)
        sess.perceive(0, 0, len(pol.perception.layers))
        slot, version = sess.store.reserve(0)
        sess.publish(0, 0, slot, version)
        G.wait_stream(P)
        sess.fetch(0, 0)
        rng = np.random.default_rng(1000 + S)
        plan = _plan(lanes, cfg.num_inference_steps, rng)
        hr = cfg.horizon * cfg.action_dim
        x0 = rng.standard_normal((agents, lanes, hr)).astype(np.float32)
        z = rng.standard_normal((agents, lanes, cfg.num_inference_steps, hr)).astype(np.float32)
        with torch.cuda.stream(G):
            sess.x.copy_(torch.from_numpy(x0))
            if sess.noise is not None:
                sess.noise.copy_(torch.from_numpy(z))
        sess.generate([(lane, s0, n) for lane, (s0, n) in enumerate(plan)])
        G.synchronize()
        got = sess.x.cpu().numpy()
        gc = sess.store.payload[:, slot, :cfg.gc_dim].float().cpu()
        kernel = int(sess.lib.auras_unet_kernel_for(sess.plan, agents * lanes))
    finally:
        sess.close()
    orc = dp_model.OracleDP(w, cfg, 0, 0, (1.0,), 1.0, numerics="bf16")
    gen = orc.generation
    want = np.empty_like(got)
    for a in range(agents):
        for lane, (s0, n) in enumerate(plan):
            st = dp_model.State(torch.from_numpy(x0[a, lane].reshape(cfg.horizon, cfg.action_dim)),
                                torch.from_numpy(z[a, lane].reshape(cfg.num_inference_steps, cfg.horizon,
                                                                    cfg.action_dim)), s0)
            for _ in range(n):
                st = gen.step(st, dp_model.Ctx(gc[a], 0))
            want[a, lane] = st.x.numpy().reshape(-1)
    return got, want, x0, kernel


def norm_err(got, want):
    return float(np.abs(got - want).max() / np.abs(want).max())
