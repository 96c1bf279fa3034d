"""CPU restatement of the reference's closed-loop tracking environment
(fp/envsim.py:24-128) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The tuner's accuracy ranking (fp/tuner.py:95-106) needs closed-loop
rollouts; the product takes an `env_factory` from its caller, and the tests
pass this one.  Pinned against the observations and sealed errors the
reference's TrackingEnv produced in the recorded closed-loop goldens
(tests/test_oracle_golden.py).  The frame protocol only: observe, apply_action,
advance_frame, last_error, success_threshold.
"""

from __future__ import annotations

import math

import numpy as np

from .toy import Obs


class CirclePath:
    """fp/envsim.py:24-33: constant angular velocity, omega in radians per frame."""

    def __init__(self, radius: float = 1.0, omega: float = math.pi / 12):
        self.radius, self.omega = radius, omega

    def position(self, frame: int) -> np.ndarray:
        a = self.omega * frame
        return self.radius * np.array([math.cos(a), math.sin(a)])


class TrackingEnv:
    """fp/envsim.py:51-128: the agent chases the path target under an action
    norm budget; observation noise is a pure function of (seed, frame)."""

    def __init__(self, path=None, noise_sigma: float = 0.02, max_step: float = 0.8,
                 success_threshold: float = 0.75, episode_frames: int = 300, seed: int = 0,
                 obs_factory=None):
        self.path = path if path is not None else CirclePath()
        self.noise_sigma, self.max_step = noise_sigma, max_step
        self.success_threshold, self.episode_frames, self.seed = success_threshold, episode_frames, seed
        self.obs_factory = obs_factory or (lambda f, v: Obs(f, v))
        self.agent = np.zeros(2)
        self.frame = 0
        self.errors = []

    def observe(self, frame: int):
        if frame >= self.episode_frames:
            raise IndexError(f"frame {frame} beyond the episode")
        if self.noise_sigma > 0:
            noise = np.random.default_rng((self.seed, frame)).normal(0.0, self.noise_sigma, 2)
        else:
            noise = np.zeros(2)
        return self.obs_factory(frame, np.concatenate([self.path.position(frame) + noise, self.agent]))

    def apply_action(self, action) -> None:
        v = np.asarray(action, dtype=np.float64)
        if float(np.linalg.norm(v)) > self.max_step * (1.0 + 1e-9) + 1e-12:
            raise ValueError("action norm above max_step")
        self.agent = self.agent + v

    def advance_frame(self) -> None:
        self.errors.append(float(np.linalg.norm(self.path.position(self.frame) - self.agent)))
        self.frame += 1

    @property
    def last_error(self) -> float:
        return self.errors[-1]


def tracking_env(seed, frames=300, omega_deg=15.0, sigma=0.02, obs_factory=None):
    """The env the goldens were recorded with (oracle/make_golden.py:tracking_env)."""
    return TrackingEnv(path=CirclePath(radius=1.0, omega=math.radians(omega_deg)), noise_sigma=sigma,
                       max_step=0.8, episode_frames=frames, seed=seed, obs_factory=obs_factory)
