"""Helpers that replay the reference-recorded golden fixtures (tests/golden/).

The fixtures come from oracle/make_golden.py run against the unmodified
reference.  Closed-loop cases are replayed open-loop through `ReplayEnv`: it
returns the observation vectors the reference's TrackingEnv produced
(fp/envsim.py:89-95) and the errors it sealed (fp/envsim.py:109-128), and it
checks that every action applied to it equals the action the reference
applied -- so a replay passes only if the engine under test drives the same
closed loop bit for bit.
"""

from __future__ import annotations

import gzip
import json
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def load(name):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as fh:
        return json.load(fh)


def schedule_cases():
    return load("schedules")["cases"]


def baseline_cases():
    """PAR / DEC traces (fp/executor.py:477-701) recorded from the reference."""
    return load("baselines")["cases"]


def case_by_name(name):
    for c in schedule_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


class ReplayEnv:
    def __init__(self, env_record, obs_factory):
        self.rec = env_record
        self.success_threshold = env_record["success_threshold"]
        self._obs_factory = obs_factory
        self._sealed = 0
        self._applied = 0
        self.mismatches = []

    def observe(self, frame):
        return self._obs_factory(frame, np.array(self.rec["observations"][frame], dtype=np.float64))

    def apply_action(self, action):
        got = [float(v) for v in np.asarray(action, dtype=np.float64)]
        want = self.rec["applied"][self._applied]
        if got != want:
            self.mismatches.append((self._applied, got, want))
        self._applied += 1

    def advance_frame(self):
        self._sealed += 1

    @property
    def last_error(self):
        return self.rec["errors"][self._sealed - 1]


def strip_none_keys(trace):
    return json.loads(json.dumps(trace))


def autoregressive_cases():
    """Token-policy traces (fp/policy.py:300-327, merged prefill
    fp/executor.py:321-348) recorded from the reference."""
    return load("autoregressive")["cases"]


def policy_kwargs(case):
    kw = dict(case["policy"])
    return kw.pop("autoregressive", False), kw


def edge_goldens():
    """Empty / one-frame runs, live reads, drop on overrun, alpha outside
    [0, 1], and PipelineConfig errors, recorded from the reference."""
    return load("edge")
