"""Policy plugins for the B200 engine.

A policy is the reference's duck type (fp/policy.py:259-272: `kind`,
`perception.layers/.layer_costs`, `generation.n_iterations/.step_cost/...`,
`sequential_cost`) plus one B200 hook, `open_session(...)`, returning a
device session whose methods enqueue kernels on the engine's perception (P)
and generation (G) streams:

  ingest(t, lane, observations)            P  request birth: upload the frame(s),
                                              initialise the request lane's state
  perceive(lane, lo, hi)                   P  perception layers [lo, hi) of a lane
  publish(lane, frame, slot, version)      P  finalize + write ring slot + commit
  fetch(target_frame, log_index)           G  in-kernel slot resolution (+ version log)
  generate(batch)                          G  batch = [(lane, start_step, iters)]
  finish(lane, out_index)                  G  action into the device output buffer
  read_actions(n) -> np.ndarray               D2H of the first n emitted actions

The engine owns the schedule; the session owns the arithmetic.  There is no
CPU implementation of any session method.

This module holds the reference's own refinement policy on the device
(`make_conditioning_policy`, fp/policy.py:279-297): fp64 kernels that are
bit-identical to numpy, used to prove the ring / stream / batching plumbing
against the reference's golden traces.  The Diffusion Policy CNN plugin is
in `diffusion.py`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .context import ContextKind, ContextStore
from .errors import ShapeMismatch


@dataclass(frozen=True)
class Observation:
    """One frame's observation (fp/policy.py:35-42).  `image` carries the
    uint8 CHW camera frame for image policies; `vector` the low-dim state."""

    frame: int
    vector: np.ndarray
    image: Optional[np.ndarray] = None

    @property
    def id(self) -> int:
        return self.frame


@dataclass(frozen=True)
class ActionOutput:
    kind: ContextKind
    values: tuple
    emitted_frame: int = -1
    staleness_profile: tuple = ()

    def as_vector(self) -> np.ndarray:
        return np.asarray(self.values, dtype=np.float64)


@dataclass(frozen=True)
class PerceptionSpec:
    """Host-side description of the perception layers (costs drive the
    partitioner and the virtual clock; fp/policy.py:55-74)."""

    layer_costs: tuple
    obs_width: int = 4

    @property
    def layers(self) -> tuple:
        return self.layer_costs

    @property
    def total_cost(self) -> float:
        return float(sum(self.layer_costs))


@dataclass(frozen=True)
class Policy:
    perception: object
    generation: object

    @property
    def kind(self) -> ContextKind:
        return self.generation.kind

    @property
    def sequential_cost(self) -> float:
        return self.perception.total_cost + self.generation.total_cost

    def open_session(self, **kw):
        return self.generation.open_session(self, **kw)


# ---------------------------------------------------------------- toy policy

@dataclass(frozen=True)
class RefinementGeneration:
    """x <- x + eta (H - x) on the device in fp64 (fp/policy.py:167-256)."""

    n_iterations: int
    step_cost: float
    eta: float = 0.08
    max_action: float = 0.8
    noise_init: bool = False
    init_sigma: float = 1.0
    state_dim: int = 2
    kind: ContextKind = ContextKind.CONDITIONING

    def __post_init__(self):
        if self.n_iterations < 1:
            raise ValueError("n_iterations must be positive")
        if self.step_cost <= 0:
            raise ValueError("step_cost must be strictly positive")
        if not (0.0 < self.eta < 1.0):
            raise ValueError("eta must lie in (0, 1)")

    @property
    def total_cost(self) -> float:
        return self.n_iterations * self.step_cost

    def initial_noise(self, seed: Optional[int]) -> np.ndarray:
        """Host-drawn initial state (fp/policy.py:203-211): the random draw is
        numpy's, by design, so device runs replay the reference's noise."""
        if self.noise_init:
            rng = np.random.default_rng(0 if seed is None else seed)
            return rng.normal(0.0, self.init_sigma, self.state_dim)
        return np.zeros(self.state_dim)

    def decode_action(self, action: ActionOutput) -> np.ndarray:
        return action.as_vector()

    def open_session(self, policy, **kw):
        return RefinementSession(policy, **kw)


class RefinementSession:
    """Device state of the toy policy: fp64 lanes, an fp64 ring, fp64 outputs."""

    def __init__(self, policy, *, capacity, lanes, agents, max_outputs, max_frames,
                 p_stream, g_stream, pp_perception=1):
        import torch
        if agents != 1:
            raise ValueError("the refinement toy policy runs one agent per session")
        self.lib = _lib.load()
        self.gen = policy.generation
        self.p, self.g = p_stream, g_stream
        dev = torch.device("cuda", torch.cuda.current_device())
        self.store = ContextStore(capacity, slot_elems=2, agents=1, dtype=torch.float64, device=dev)
        self.latent = torch.zeros(lanes, 4, dtype=torch.float64, device=dev)
        self.x = torch.zeros(lanes, 2, dtype=torch.float64, device=dev)
        self.out = torch.zeros(max(1, max_outputs), 2, dtype=torch.float64, device=dev)
        self.fetched = torch.zeros(3, dtype=torch.int64, device=dev)
        self.version_log = torch.zeros(max(1, max_frames), dtype=torch.int64, device=dev)
        self.obs_width = policy.perception.obs_width

    def ingest(self, t, lane, observations):
        obs = observations[0]
        vec = np.asarray(obs.vector, dtype=np.float64)
        if vec.shape != (self.obs_width,):
            raise ShapeMismatch(f"observation width {vec.shape} != ({self.obs_width},)")
        x0 = np.ascontiguousarray(self.gen.initial_noise(t), dtype=np.float64)
        o = np.ascontiguousarray(vec)
        _lib.check(self.lib.auras_toy_ingest(
            self.latent.data_ptr(), lane, o.ctypes.data_as(_lib.C.POINTER(_lib.f64)),
            self.x.data_ptr(), x0.ctypes.data_as(_lib.C.POINTER(_lib.f64)), self.p.cuda_stream),
            "toy_ingest")

    def perceive(self, lane, lo, hi):
        return None     # identity layers (fp/policy.py:275-276): nothing to launch

    def publish(self, lane, frame, slot, version):
        st = self.store
        _lib.check(self.lib.auras_toy_publish(self.latent.data_ptr(), lane, st.payload.data_ptr(),
                                              st.meta.data_ptr(), st.state.data_ptr(), st.capacity,
                                              frame, version, self.p.cuda_stream), "toy_publish")

    def fetch(self, target, log_index):
        self.store.device_fetch(target, self.fetched, self.version_log, log_index, self.g)

    def generate(self, batch):
        lanes = _lib.int_array([b[0] for b in batch])
        iters = _lib.int_array([b[2] for b in batch])
        _lib.check(self.lib.auras_toy_generate(self.x.data_ptr(), lanes, iters, len(batch),
                                               self.gen.eta, self.store.payload.data_ptr(),
                                               self.fetched.data_ptr(), self.g.cuda_stream),
                   "toy_generate")

    def finish(self, lane, out_index):
        _lib.check(self.lib.auras_toy_finish(self.x.data_ptr(), lane, self.gen.max_action,
                                             self.out[out_index].data_ptr(), self.g.cuda_stream),
                   "toy_finish")

    def read_actions(self, n):
        return self.out[:n].cpu().numpy()[:, None, :]      # [n, agents=1, 2]

    def read_action(self, i):
        return self.out[i].cpu().numpy()[None, :]

    def read_version_log(self, n):
        return self.version_log[:n].cpu().numpy()

    def action_values(self, row):
        return tuple(float(v) for v in row)

    def close(self):
        pass


def make_conditioning_policy(layer_costs=(14.0, 14.0), n_iterations: int = 100,
                             step_cost: float = 1.0, eta: float = 0.08, max_action: float = 0.8,
                             noise_init: bool = False) -> Policy:
    """Same signature and semantics as fp/policy.py:279-297, running on the B200."""
    costs = tuple(float(c) for c in layer_costs)
    if not costs:
        raise ValueError("perception needs at least one layer")
    if any(c <= 0 for c in costs):
        raise ValueError("layer cost must be strictly positive")
    return Policy(perception=PerceptionSpec(costs, obs_width=4),
                  generation=RefinementGeneration(n_iterations=n_iterations, step_cost=step_cost,
                                                  eta=eta, max_action=max_action,
                                                  noise_init=noise_init))


# ---------------------------------------------------------------- scripted token policy

ACTION_TOKEN_COUNT = 7
_MAG_LEVELS = 63


def decode_action_tokens(tokens, max_action: float) -> np.ndarray:
    """fp/policy.py:135-148: the 7-token schema back to a planar displacement."""
    toks = [int(t) for t in tokens]
    if len(toks) < ACTION_TOKEN_COUNT:
        raise ValueError(f"need {ACTION_TOKEN_COUNT} tokens, got {len(toks)}")
    width = max_action / _MAG_LEVELS
    out = []
    for axis in range(2):
        sign, hi, lo = toks[3 * axis: 3 * axis + 3]
        s = 0.0 if sign == 0 else (1.0 if sign == 1 else -1.0)
        out.append(s * (hi * 8 + lo) * width)
    return np.array(out)


@dataclass(frozen=True)
class TokenGeneration:
    """Token-sequential generation (fp/policy.py:167-256, autoregressive
    branch): one token per iteration from the scripted policy, costs a flat
    prefill per call plus one decode per further token."""

    n_iterations: int
    step_cost: float
    prefill_cost: float = 10.0
    decode_cost: float = 1.0
    max_action: float = 0.8
    kind: ContextKind = ContextKind.AUTOREGRESSIVE

    def __post_init__(self):
        if self.n_iterations < 1:
            raise ValueError("n_iterations must be positive")
        if self.step_cost <= 0:
            raise ValueError("step_cost must be strictly positive")

    @property
    def total_cost(self) -> float:
        return self.prefill_cost + (self.n_iterations - 1) * self.decode_cost

    def initial_noise(self, seed: Optional[int]) -> np.ndarray:
        return np.zeros(2)                      # token states start empty

    def decode_action(self, action: ActionOutput) -> np.ndarray:
        vec = decode_action_tokens(action.values, self.max_action)
        norm = float(np.linalg.norm(vec))
        if norm > self.max_action:
            vec = vec * (self.max_action / norm)
        return vec

    def open_session(self, policy, **kw):
        return TokenSession(policy, **kw)


class TokenSession(RefinementSession):
    """Device state of the scripted token policy: the toy ring (the context's
    displacement, fp64), int32 token lanes, fp64 token outputs."""

    def __init__(self, policy, **kw):
        import torch
        max_outputs = kw.get("max_outputs", 1)
        super().__init__(policy, **kw)
        dev = self.x.device
        self.l_a = policy.generation.n_iterations
        self.tokens = torch.zeros(self.x.shape[0], self.l_a, dtype=torch.int32, device=dev)
        self.out = torch.zeros(max(1, max_outputs), self.l_a, dtype=torch.float64, device=dev)

    def generate(self, batch):
        lanes = _lib.int_array([b[0] for b in batch])
        starts = _lib.int_array([b[1] for b in batch])
        counts = _lib.int_array([b[2] for b in batch])
        _lib.check(self.lib.auras_ar_generate(self.tokens.data_ptr(), self.l_a, lanes, starts, counts,
                                              len(batch), self.store.payload.data_ptr(),
                                              self.fetched.data_ptr(), self.gen.max_action, self.g.cuda_stream),
                   "ar_generate")

    def finish(self, lane, out_index):
        _lib.check(self.lib.auras_ar_finish(self.tokens.data_ptr(), lane, self.l_a,
                                            self.out[out_index].data_ptr(), self.g.cuda_stream), "ar_finish")

    def republish(self, src_slot, slot, frame, version):
        """Device half of an action-token context update (P stream)."""
        st = self.store
        _lib.check(self.lib.auras_ring_copy_slot(st.payload.data_ptr(), st.slot_elems, src_slot, slot,
                                                 self.p.cuda_stream), "ring_copy_slot")
        st.commit(frame, version, self.p)

    def action_values(self, row):
        return tuple(int(v) for v in row)


def make_autoregressive_policy(layer_costs=(14.0, 14.0), l_a: int = ACTION_TOKEN_COUNT,
                               prefill_cost: float = 10.0, decode_cost: float = 1.0,
                               max_action: float = 0.8, vision_len: int = 96, language_len: int = 32,
                               latent_width: int = 64) -> Policy:
    """Same signature and semantics as fp/policy.py:300-327 (the scripted token
    policy whose context mirrors the X_V / X_L / X_A layout), on the B200.  The
    token policy reads only the displacement in vision row 0, which is what
    the device ring carries; the long X_V / X_L rows exist in the reference to
    size the merged prefill and do not change any token."""
    costs = tuple(float(c) for c in layer_costs)
    if not costs or any(c <= 0 for c in costs):
        raise ValueError("layer costs must be positive")
    return Policy(perception=PerceptionSpec(costs, obs_width=4),
                  generation=TokenGeneration(n_iterations=l_a, step_cost=decode_cost,
                                             prefill_cost=prefill_cost, decode_cost=decode_cost,
                                             max_action=max_action))


# ---------------------------------------------------------------- reference-style plugins

def is_reference_plugin(policy) -> bool:
    """The reference's duck-typed plugin protocol (fp/policy.py:46-272): a
    perception model with start / apply_layers / finalize and a generation
    model with initial_state / step / finish."""
    p, g = getattr(policy, "perception", None), getattr(policy, "generation", None)
    return (p is not None and g is not None
            and all(callable(getattr(p, m, None)) for m in ("start", "apply_layers", "finalize"))
            and all(callable(getattr(g, m, None)) for m in ("initial_state", "step", "finish")))


class HostPolicy:
    """A reference-style policy object under the B200 engine.  The engine's
    schedule, context ring bookkeeping, versions, streams and events are the
    same as for the device plugins; the policy's own callbacks run on the host
    in stream order (they are arbitrary Python: nothing here can move them onto
    the GPU).  Use make_conditioning_policy / make_diffusion_policy /
    make_autoregressive_policy for the device kernels."""

    def __init__(self, policy):
        self.ref = policy
        self.perception = policy.perception
        self.generation = policy.generation
        kind = getattr(policy, "kind", ContextKind.CONDITIONING)
        self.kind = ContextKind(getattr(kind, "value", kind))
        # (no synthetic_observation: without an environment the executor makes the
        #  reference's zero observation, fp/executor.py:142-143)

    @property
    def sequential_cost(self) -> float:
        sc = getattr(self.ref, "sequential_cost", None)
        if sc is not None:
            return float(sc)
        return float(self.perception.total_cost) + float(self.generation.total_cost)

    def open_session(self, **kw):
        return HostPluginSession(self, **kw)


class HostPluginSession:
    """The session protocol of the device plugins (ingest / perceive / publish /
    fetch / generate / finish, fp/executor.py:256-380) over a reference-style
    policy's callbacks.  Each call runs once the stream it is ordered on has
    drained, so the host work observes the same ordering the device work
    would.  Contexts live in a host ring indexed like the device ring."""

    def __init__(self, policy, *, capacity, lanes, agents, max_outputs, max_frames,
                 p_stream, g_stream, pp_perception=1):
        import torch
        if agents != 1:
            raise ValueError("a reference-style policy runs one agent per session")
        self.pol = policy
        self.per, self.gen = policy.perception, policy.generation
        self.p, self.g = p_stream, g_stream
        dev = torch.device("cuda", torch.cuda.current_device())
        # the executor's host mirror (reserve / resolve) of the ring; the payload stays unused
        self.store = ContextStore(capacity, slot_elems=1, agents=1, dtype=torch.float64, device=dev)
        self.obs = [None] * lanes
        self.latent = [None] * lanes
        self.state = [None] * lanes
        self.slots = [None] * capacity           # (frame, version, context)
        self.ctx = None
        self.out = [None] * max(1, max_outputs)
        self.version_log = np.zeros(max(1, max_frames), dtype=np.int64)

    def ingest(self, t, lane, observations):
        self.p.synchronize()
        obs = observations[0]
        self.obs[lane] = obs
        self.latent[lane] = self.per.start(obs)
        self.state[lane] = self.gen.initial_state(seed=t)

    def perceive(self, lane, lo, hi):
        self.p.synchronize()
        self.latent[lane] = self.per.apply_layers(self.latent[lane], lo, hi)

    def publish(self, lane, frame, slot, version):
        self.p.synchronize()
        ctx = self.per.finalize(self.latent[lane], self.obs[lane])
        # fp/context.py:129-143 stamps the produced frame
        if getattr(ctx, "produced_frame", frame) != frame and hasattr(ctx, "with_produced_frame"):
            ctx = ctx.with_produced_frame(frame)
        self.slots[slot] = (frame, version, ctx)

    def republish(self, src_slot, slot, frame, version):
        self.p.synchronize()
        _, _, ctx = self.slots[src_slot]
        self.slots[slot] = (frame, version, ctx)

    def fetch(self, target, log_index):
        self.g.synchronize()
        entry = self.slots[target % len(self.slots)]
        if entry is None or entry[0] != target:
            from .errors import NotYetPublished
            raise NotYetPublished(f"no context published for frame {target}")
        self.version_log[log_index] = entry[1]
        self.ctx = entry[2]

    def generate(self, batch):
        self.g.synchronize()
        for lane, _start, iters in batch:
            for _ in range(iters):
                self.state[lane] = self.gen.step(self.state[lane], self.ctx)

    def finish(self, lane, out_index):
        self.g.synchronize()
        self.out[out_index] = tuple(self.gen.finish(self.state[lane]).values)

    def read_actions(self, n):
        return [[self.out[i]] for i in range(n)]

    def read_action(self, i):
        return [self.out[i]]

    def read_version_log(self, n):
        return self.version_log[:n].copy()

    def action_values(self, row):
        return tuple(row)

    def close(self):
        pass
