"""fp64 restatement of the reference's toy policies.

TEST ORACLE.  Follows fp/policy.py:55-93 (staged perception), :203-246
(initial state, step, finish), :279-297 (make_conditioning_policy) and, for
the scripted token policy, :116-165 (token schema, scripted next token) and
:300-327 (make_autoregressive_policy).  Every
floating-point operation is the numpy operation the reference performs, so
results are bit-identical to the reference on the same host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Obs:
    frame: int
    vector: np.ndarray

    @property
    def id(self):
        return self.frame


@dataclass(frozen=True)
class Ctx:
    payload: np.ndarray
    produced_frame: int


@dataclass
class State:
    vector: np.ndarray
    steps: int = 0


@dataclass(frozen=True)
class Action:
    values: tuple
    emitted_frame: int = -1
    staleness_profile: tuple = ()


class ToyPerception:
    def __init__(self, layer_costs):
        self.layer_costs = tuple(float(c) for c in layer_costs)
        self.layers = self.layer_costs

    @property
    def total_cost(self):
        return float(sum(self.layer_costs))

    def start(self, obs):
        v = np.asarray(obs.vector, dtype=np.float64)
        assert v.shape == (4,)
        return v

    def apply_layers(self, latent, lo, hi):     # identity layers, fp/policy.py:275-276
        return latent

    def finalize(self, latent, obs):            # fp/policy.py:285-290
        return Ctx(latent[:2] - latent[2:4], obs.frame)

    def perceive(self, obs):
        return self.finalize(self.apply_layers(self.start(obs), 0, len(self.layers)), obs)


class ToyGeneration:
    def __init__(self, n_iterations, step_cost, eta, max_action, noise_init, init_sigma=1.0):
        self.n_iterations, self.step_cost = n_iterations, step_cost
        self.eta, self.max_action = eta, max_action
        self.noise_init, self.init_sigma = noise_init, init_sigma

    @property
    def total_cost(self):
        return self.n_iterations * self.step_cost

    def initial_state(self, seed=None):          # fp/policy.py:203-211
        if self.noise_init:
            rng = np.random.default_rng(0 if seed is None else seed)
            return State(rng.normal(0.0, self.init_sigma, 2))
        return State(np.zeros(2))

    def step(self, state, ctx):                 # fp/policy.py:224
        h = np.asarray(ctx.payload, dtype=np.float64)
        return State(state.vector + self.eta * (h - state.vector), state.steps + 1)

    def finish(self, state, emitted_frame=-1, staleness_profile=()):   # :230-246
        assert state.steps >= self.n_iterations
        vec = np.asarray(state.vector, dtype=np.float64)
        norm = float(np.linalg.norm(vec))
        if norm > self.max_action:
            vec = vec * (self.max_action / norm)
        return Action(tuple(float(v) for v in vec), emitted_frame, tuple(staleness_profile))

    def decode_action(self, action):
        return np.asarray(action.values, dtype=np.float64)


class ToyPolicy:
    kind = "conditioning"

    def __init__(self, layer_costs=(14.0, 14.0), n_iterations=100, step_cost=1.0,
                 eta=0.08, max_action=0.8, noise_init=False):
        self.perception = ToyPerception(layer_costs)
        self.generation = ToyGeneration(n_iterations, step_cost, eta, max_action, noise_init)

    @property
    def sequential_cost(self):
        return self.perception.total_cost + self.generation.total_cost

    @staticmethod
    def synthetic_observation(frame):           # fp/executor.py:142-143
        return Obs(frame, np.zeros(4))


# ---------------------------------------------------------------- token policy

ACTION_TOKEN_COUNT, MAG_LEVELS, STOP_TOKEN = 7, 63, 0


def encode_action_tokens(displacement, max_action, l_a=ACTION_TOKEN_COUNT):
    """fp/policy.py:120-134: per axis (sign, mag // 8, mag % 8), then STOP;
    repeated cyclically past 7 tokens."""
    width = max_action / MAG_LEVELS
    block = []
    for raw in np.asarray(displacement, dtype=np.float64)[:2]:
        v = float(min(max(raw, -max_action), max_action))
        mag = min(int(np.floor(abs(v) / width + 0.5)), MAG_LEVELS)
        sign = 0 if mag == 0 else (1 if v > 0 else 2)
        block.extend((sign, mag // 8, mag % 8))
    block.append(STOP_TOKEN)
    return tuple(block[i % ACTION_TOKEN_COUNT] for i in range(l_a))


def decode_action_tokens(tokens, max_action):
    """fp/policy.py:136-148."""
    width = max_action / MAG_LEVELS
    out = []
    for axis in range(2):
        sign, hi, lo = list(tokens)[3 * axis: 3 * axis + 3]
        s = 0.0 if sign == 0 else (1.0 if sign == 1 else -1.0)
        out.append(s * (hi * 8 + lo) * width)
    return np.array(out)


@dataclass
class TokenState:
    tokens: list
    steps: int = 0


class TokenGeneration:
    """fp/policy.py:167-256, autoregressive branches: one scripted token per
    step (the request's own prefix picks the position), a flat prefill per
    call plus one decode per further token."""

    def __init__(self, l_a, prefill_cost, decode_cost, max_action):
        self.n_iterations, self.step_cost = l_a, decode_cost
        self.prefill_cost, self.decode_cost, self.max_action = prefill_cost, decode_cost, max_action

    @property
    def total_cost(self):
        return self.prefill_cost + (self.n_iterations - 1) * self.decode_cost

    def stage_cost(self, iterations):                # fp/executor.py:227-229
        return self.prefill_cost + max(iterations - 1, 0) * self.decode_cost

    def initial_state(self, seed=None):
        return TokenState([])

    def step(self, state, ctx):                     # fp/policy.py:226-228, :151-165
        tok = encode_action_tokens(ctx.payload, self.max_action, self.n_iterations)[len(state.tokens)]
        return TokenState(state.tokens + [tok], state.steps + 1)

    def finish(self, state, emitted_frame=-1, staleness_profile=()):
        assert state.steps >= self.n_iterations
        return Action(tuple(state.tokens), emitted_frame, tuple(staleness_profile))

    def decode_action(self, action):                # fp/policy.py:248-255
        vec = decode_action_tokens(action.values, self.max_action)
        norm = float(np.linalg.norm(vec))
        if norm > self.max_action:
            vec = vec * (self.max_action / norm)
        return vec


class TokenPolicy:
    """make_autoregressive_policy (fp/policy.py:300-327): the context's
    vision row 0 carries the displacement, which is all the scripted policy
    reads, so the oracle context is that displacement."""
    kind = "autoregressive"

    def __init__(self, layer_costs=(14.0, 14.0), l_a=ACTION_TOKEN_COUNT, prefill_cost=10.0,
                 decode_cost=1.0, max_action=0.8, **_ignored):
        self.perception = ToyPerception(layer_costs)
        self.generation = TokenGeneration(l_a, prefill_cost, decode_cost, max_action)

    @property
    def sequential_cost(self):
        return self.perception.total_cost + self.generation.total_cost

    @staticmethod
    def synthetic_observation(frame):
        return Obs(frame, np.zeros(4))
