"""fp64 restatement of the reference's refinement ("conditioning") toy policy.

TEST ORACLE.  Follows fp/policy.py:55-93 (staged perception), :203-246
(initial state, step, finish) and :279-297 (make_conditioning_policy).  Every
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
