"""Stage planning for the frame pipeline.

Same contract as the reference partitioner (fp/partition.py:57-132):

* generation iterations are split over `stages` pipeline stages with weights
  w_i = exp((i+1) * alpha); cumulative boundaries are n * (running weight sum /
  fsum of weights), rounded half up, clamped to be monotone, with the final
  boundary pinned to n (fp/partition.py:101-123).  Reproduced bit for bit --
  the tests compare against the reference's goldens, including its seeded fuzz
  sets;
* perception layers are split into contiguous ranges minimising the largest
  stage cost (exact dynamic program, earliest-cut tie breaking, as
  fp/partition.py:57-98);
* the `FRAMEPIPE_ROUNDING_FAULT=truncate` fault hook (fp/partition.py:18-30)
  is honoured so the reference's fault-injection test still bites.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

from .errors import InvalidStageCount, TooManyStages

ROUNDING_FAULT_ENV = "FRAMEPIPE_ROUNDING_FAULT"


def round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def _boundary_rounding():
    if os.environ.get(ROUNDING_FAULT_ENV) == "truncate":
        return lambda x: int(math.floor(x))
    return round_half_up


@dataclass(frozen=True)
class StagePlan:
    """Layer ranges per perception stage and iteration counts per generation stage."""

    perception_stages: tuple
    generation_stages: tuple
    alpha: float = 0.0

    @property
    def pp_perception(self) -> int:
        return len(self.perception_stages)

    @property
    def pp_generation(self) -> int:
        return len(self.generation_stages)

    def stage_starts(self) -> tuple:
        """Inference-step index at which each generation stage begins."""
        starts, acc = [], 0
        for c in self.generation_stages:
            starts.append(acc)
            acc += c
        return tuple(starts)

    def to_dict(self) -> dict:
        return {"perception_stages": [list(r) for r in self.perception_stages],
                "generation_stages": list(self.generation_stages),
                "alpha": self.alpha}


def split_generation(n: int, stages: int, alpha: float = 0.0) -> list:
    if n < 1 or stages < 1:
        raise InvalidStageCount(f"need n >= 1 and stages >= 1 (n={n}, stages={stages})")
    if alpha == 0.0 and n < stages:
        raise InvalidStageCount(f"a uniform split needs n >= stages (n={n}, stages={stages})")
    rnd = _boundary_rounding()
    weights = [math.exp((i + 1) * alpha) for i in range(stages)]
    total = math.fsum(weights)
    counts, prev, running = [], 0, 0.0
    for i, w in enumerate(weights):
        running += w
        edge = n if i + 1 == stages else rnd(n * (running / total))
        edge = min(max(edge, prev), n)
        counts.append(edge - prev)
        prev = edge
    return counts


def split_perception(costs, stages: int) -> list:
    c = [float(x) for x in costs]
    n = len(c)
    if stages < 1:
        raise TooManyStages("need at least one perception stage")
    if stages > n:
        raise TooManyStages(f"{stages} stages for {n} layers")
    if any(x <= 0 for x in c):
        raise ValueError("layer costs must be strictly positive")
    prefix = [0.0]
    for x in c:
        prefix.append(prefix[-1] + x)
    inf = float("inf")
    cost = {(0, 0): 0.0}
    cut = {}
    for s in range(1, stages + 1):
        for i in range(s, n + 1):
            best, arg = inf, 0
            for j in range(s - 1, i):
                prev = cost.get((j, s - 1), inf)
                cand = max(prev, prefix[i] - prefix[j])
                if cand < best:
                    best, arg = cand, j
            cost[(i, s)], cut[(i, s)] = best, arg
    ranges, i = [], n
    for s in range(stages, 0, -1):
        j = cut[(i, s)]
        ranges.append((j, i))
        i = j
    return ranges[::-1]


def plan_stages(layer_costs, pp_perception: int, n_iterations: int, pp_generation: int,
                alpha: float = 0.0) -> StagePlan:
    return StagePlan(tuple(split_perception(layer_costs, pp_perception)),
                     tuple(split_generation(n_iterations, pp_generation, alpha)), alpha)
