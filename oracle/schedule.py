"""Virtual-time restatement of the reference frame executor (TEST ORACLE).

Restates, for conditioning (iterative-refinement) policies only:

* `split_generation`  -- fp/partition.py:101-123 (weights e^{(i+1)a}, fsum
  total, running-sum cumulative fractions, round-half-up boundaries, last
  boundary forced to n, FRAMEPIPE_ROUNDING_FAULT hook fp/partition.py:18-30);
* `split_perception`  -- fp/partition.py:57-98 (exact min-max contiguous
  split; ties resolved towards the earliest cut, as the reference's strict
  `<` comparison does);
* `Ring`              -- fp/context.py:98-164 (K slots, version counter,
  StaleWrite / NotYetPublished / OffsetOutOfRange semantics);
* `run_pipelined`     -- fp/executor.py:200-399;
* `run_sequential`    -- fp/executor.py:406-461.

The arithmetic of every float that reaches the trace (stage costs, frame
durations, the clock, JCT, staleness means) is performed with the same
operations in the same order as the reference, so traces compare equal with
`==`.  The model arithmetic is delegated to a policy object with the
reference's duck type (fp/executor.py:216-330).
"""

from __future__ import annotations

import dataclasses
import math
import os
from dataclasses import dataclass, field

import numpy as np


class OracleError(Exception):
    pass


class NotYetPublished(OracleError):
    pass


class OffsetOutOfRange(OracleError):
    pass


class StaleWrite(OracleError):
    pass


class DeadlockDetected(OracleError):
    pass


# ---------------------------------------------------------------- partition

def _half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def split_generation(n: int, stages: int, alpha: float = 0.0) -> list[int]:
    """fp/partition.py:101-123."""
    if n < 1 or stages < 1 or (alpha == 0.0 and n < stages):
        raise OracleError("invalid stage count")
    rounding = (lambda v: int(math.floor(v))) \
        if os.environ.get("FRAMEPIPE_ROUNDING_FAULT") == "truncate" else _half_up
    w = [math.exp(alpha * (i + 1)) for i in range(stages)]
    denom = math.fsum(w)
    bounds, running = [], 0.0
    for i, wi in enumerate(w):
        running += wi
        bounds.append(n if i == stages - 1 else rounding(n * (running / denom)))
    out, prev = [], 0
    for b in bounds:
        b = min(max(b, prev), n)
        out.append(b - prev)
        prev = b
    return out


def split_perception(costs, stages: int) -> list[tuple[int, int]]:
    """fp/partition.py:57-98: minimise the largest contiguous stage cost."""
    costs = [float(c) for c in costs]
    n = len(costs)
    if stages < 1 or stages > n:
        raise OracleError("too many stages")
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + c)
    inf = float("inf")
    # best[s][i]: optimal max-cost splitting the first i layers into s stages
    best = [[inf] * (n + 1) for _ in range(stages + 1)]
    arg = [[0] * (n + 1) for _ in range(stages + 1)]
    best[0][0] = 0.0
    for s in range(1, stages + 1):
        for i in range(s, n + 1):
            for j in range(s - 1, i):
                v = max(best[s - 1][j], pre[i] - pre[j])
                if v < best[s][i]:
                    best[s][i], arg[s][i] = v, j
    cuts, i = [], n
    for s in range(stages, 0, -1):
        cuts.append((arg[s][i], i))
        i = arg[s][i]
    return cuts[::-1]


# ---------------------------------------------------------------- ring store

@dataclass
class Ring:
    """fp/context.py:98-164 without the threading (the oracle is serial)."""

    capacity: int = 2
    version: int = 0
    last_frame: int | None = None
    slots: list = field(default_factory=list)

    def __post_init__(self):
        self.slots = [None] * self.capacity

    def publish(self, payload, frame: int) -> int:
        if self.last_frame is not None and frame < self.last_frame:
            raise StaleWrite(frame)
        self.version += 1
        self.slots[frame % self.capacity] = (frame, self.version, payload)
        self.last_frame = frame
        return self.version

    def fetch_entry(self, frame: int, offset: int):
        if offset > 0 or -offset >= self.capacity:
            raise OffsetOutOfRange(offset)
        want = frame + offset
        slot = self.slots[want % self.capacity]
        if slot is None or slot[0] != want:
            raise NotYetPublished(want)
        return slot[1], slot[0], slot[2]

    def latest_entry(self):
        if self.last_frame is None:
            raise NotYetPublished("empty")
        slot = self.slots[self.last_frame % self.capacity]
        return slot[1], slot[0], slot[2]


# ---------------------------------------------------------------- executor

@dataclass
class Request:
    observation_id: int
    birth_frame: int
    birth_time: float
    completion_frame: int = -1
    completion_time: float = -1.0
    jct: float = -1.0
    context_versions: list = field(default_factory=list)


@dataclass
class OracleResult:
    actions: list
    trace: list
    requests: list


class _Landing:
    """Boundary protocol of fp/executor.py:146-184 (land newest, then observe)."""

    def __init__(self, env, policy):
        self.env, self.policy, self.queue = env, policy, []
        self.last_superseded = 0

    def boundary(self, frame):
        due = [q for q in self.queue if q[0] == frame]
        self.last_superseded = 0
        if due:
            self.queue = [q for q in self.queue if q[0] != frame]
            chosen = max(due, key=lambda q: q[1])
            self.last_superseded = len(due) - 1
            if self.env is not None:
                self.env.apply_action(self.policy.generation.decode_action(chosen[2]))
        if self.env is None:
            return self.policy.synthetic_observation(frame)
        return self.env.observe(frame)

    def seal(self):
        if self.env is None:
            return None
        self.env.advance_frame()
        return self.env.last_error


def _frame_record(t, now):
    return {"type": "frame", "frame": t, "start": now, "perception": [], "generation": [],
            "publishes": [], "emissions": [], "prefill_calls": 0, "decode_calls": 0,
            "generation_cost": 0.0, "dropped_observations": 0}


def _emission(req_frame, time, t, land, jct, values, ages):
    return {"request": req_frame, "time": time, "emission_frame": t, "land_frame": land,
            "jct": jct, "action": list(values), "staleness_min": min(ages),
            "staleness_mean": float(np.mean(ages)), "staleness_max": max(ages),
            "staleness_final": ages[-1]}


def run_pipelined(cfg: dict, policy, env, duration: int) -> OracleResult:
    """fp/executor.py:200-399 for conditioning policies.

    `cfg` is the PipelineConfig field dict (fp/executor.py:48-60)."""
    pp_p, pp_g = cfg.get("pp_perception", 1), cfg.get("pp_generation", 1)
    ar = getattr(policy, "kind", "conditioning") == "autoregressive"
    off = cfg.get("fetch_offset")
    off = (-1 if ar else 0) if off is None else off          # fp/executor.py:61-65
    m_cfg = cfg.get("merge_autoregressive")
    merge = (m_cfg and ar) if m_cfg is not None else ar      # fp/executor.py:66-70
    alpha = cfg.get("alpha", 0.0)
    interval = cfg.get("frame_interval")
    cap = cfg.get("store_capacity", 2)
    read_policy = cfg.get("read_policy", "snapshot")
    overrun = cfg.get("overrun_policy", "stretch")
    perc, gen = policy.perception, policy.generation

    ranges = split_perception(perc.layer_costs, pp_p)
    counts = split_generation(gen.n_iterations, pp_g, alpha)
    shift = pp_p - 1 - off            # birth -> first generation stage
    span = shift + pp_g               # birth -> emission, inclusive
    p_cost = [sum(perc.layer_costs[a:b]) for a, b in ranges]
    full_cfg = {"pp_perception": pp_p, "pp_generation": pp_g,
                "fetch_offset": cfg.get("fetch_offset"), "alpha": alpha,
                "frame_interval": interval,
                "merge_autoregressive": cfg.get("merge_autoregressive"),
                "store_capacity": cap, "read_policy": read_policy,
                "overrun_policy": overrun}
    trace = [{"type": "header", "schema": 1, "mode": "pipe", "engine": "virtual",
              "frame_interval": interval, "duration": duration,
              "config": {"pipeline": full_cfg,
                         "plan": {"perception_stages": [list(r) for r in ranges],
                                  "generation_stages": list(counts), "alpha": alpha},
                         "fetch_offset": off, "merged": bool(merge)},
              "success_threshold": getattr(env, "success_threshold", None)}]

    ring = Ring(cap)
    port = _Landing(env, policy)
    live: dict[int, dict] = {}    # birth frame -> request state
    requests, actions = [], []
    now, skip = 0.0, 0
    for t in range(duration):
        rec = _frame_record(t, now)
        obs = port.boundary(t)
        rec["superseded_actions"] = port.last_superseded
        if skip:
            skip -= 1
            rec["dropped_observations"] += 1
        else:
            r = Request(observation_id=obs.id, birth_frame=t, birth_time=now)
            live[t] = {"req": r, "obs": obs, "latent": perc.start(obs),
                       "state": gen.initial_state(seed=t), "ages": []}
            requests.append(r)

        early = None
        if off <= -1 and read_policy == "snapshot":
            try:
                early = ring.fetch_entry(t, off)
            except NotYetPublished:
                early = None

        side_costs, pub_cost, published = [], 0.0, False
        for s in range(1, pp_p + 1):
            item = live.get(t - s + 1)
            if item is None:
                continue
            lo, hi = ranges[s - 1]
            item["latent"] = perc.apply_layers(item["latent"], lo, hi)
            entry = {"request": t - s + 1, "stage": s, "cost": p_cost[s - 1],
                     "published_version": None}
            if s == pp_p:
                ctx = perc.finalize(item["latent"], item["obs"])
                v = ring.publish(ctx, t)
                entry["published_version"] = v
                rec["publishes"].append(v)
                pub_cost, published = p_cost[s - 1], True
            else:
                side_costs.append(p_cost[s - 1])
            rec["perception"].append(entry)

        active = [(j, t - shift - (j - 1)) for j in range(1, pp_g + 1)
                  if (t - shift - (j - 1)) in live]
        gen_costs = []
        if active:
            if early is not None:
                version, ctx_frame, ctx = early
            else:
                try:
                    version, ctx_frame, ctx = ring.fetch_entry(t, off)
                except NotYetPublished:
                    if t + off < pp_p - 1:
                        raise DeadlockDetected(t)
                    version, ctx_frame, ctx = ring.latest_entry()
            if merge and ar:                     # one merged prefill (fp/executor.py:321-324)
                rec["prefill_calls"] += 1
                rec["generation_cost"] += gen.prefill_cost
                gen_costs.append(gen.prefill_cost)
            for j, b in active:
                item = live[b]
                iters = counts[j - 1]
                age = float(b + span - 1 - ctx_frame)
                for _ in range(iters):
                    item["state"] = gen.step(item["state"], ctx)
                item["ages"].extend([age] * iters)
                item["req"].context_versions.append(version)
                if not (merge and ar):
                    c = gen.stage_cost(iters) if ar else iters * gen.step_cost
                    gen_costs.append(c)
                    rec["generation_cost"] += c
                    if ar:
                        rec["prefill_calls"] += 1
                        rec["decode_calls"] += max(iters - 1, 0)
                rec["generation"].append({"request": b, "stage": j, "iterations": iters,
                                          "context_version": version,
                                          "context_frame": ctx_frame,
                                          "context_age_at_emission": age})
            if ar:
                # the freshest token prefix back into the shared context: the
                # newest context re-published as this frame's, new version
                # (fp/executor.py:345-348, fp/context.py:166-175)
                _, _, newest = ring.latest_entry()
                ring.publish(newest, t)

        if off == 0 and gen_costs and published:
            busiest = max(side_costs + [pub_cost + max(gen_costs)])
        else:
            pool = side_costs + gen_costs + ([pub_cost] if published else [])
            busiest = max(pool) if pool else 0.0
        if interval is None:
            dur = busiest
        elif busiest <= interval:
            dur = interval
        elif overrun == "stretch":
            dur, rec["overrun"] = busiest, True
        else:
            q = math.ceil(busiest / interval)
            dur, rec["overrun"] = q * interval, True
            skip += q - 1
        now += dur
        rec["end"] = now

        done = live.pop(t - span + 1, None)
        if done is not None:
            a = gen.finish(done["state"], emitted_frame=t,
                           staleness_profile=tuple(done["ages"]))
            actions.append(a)
            r = done["req"]
            r.completion_frame, r.completion_time = t + 1, now
            r.jct = now - r.birth_time
            port.queue.append((t + 1, now, a))
            rec["emissions"].append(_emission(t - span + 1, now, t, t + 1, r.jct,
                                              a.values, done["ages"]))
        rec["env_error"] = port.seal()
        trace.append(rec)
    return OracleResult(actions, trace, requests)


def run_sequential(policy, env, duration: int, frame_interval=None) -> OracleResult:
    """fp/executor.py:406-461."""
    gen = policy.generation
    cost = policy.sequential_cost
    interval = frame_interval if frame_interval is not None else cost
    per_req = max(1, math.ceil(cost / interval - 1e-12))
    trace = [{"type": "header", "schema": 1, "mode": "seq", "engine": "virtual",
              "frame_interval": interval, "duration": duration,
              "config": {"request_cost": cost},
              "success_threshold": getattr(env, "success_threshold", None)}]
    port = _Landing(env, policy)
    actions, requests = [], []
    free_at = 0
    for t in range(duration):
        now = t * interval
        rec = _frame_record(t, now)
        rec["end"] = now + interval
        obs = port.boundary(t)
        rec["superseded_actions"] = port.last_superseded
        if t >= free_at:
            r = Request(observation_id=obs.id, birth_frame=t, birth_time=now)
            ctx = policy.perception.perceive(obs)
            state = gen.initial_state(seed=t)
            for _ in range(gen.n_iterations):
                state = gen.step(state, ctx)
            emit = t + per_req - 1
            age = float(emit - ctx.produced_frame)
            a = gen.finish(state, emitted_frame=emit,
                           staleness_profile=(age,) * gen.n_iterations)
            land = t + per_req
            r.completion_frame, r.completion_time, r.jct = land, now + cost, cost
            r.context_versions.append(1)
            requests.append(r)
            actions.append(a)
            port.queue.append((land, now + cost, a))
            free_at = land
            if getattr(policy, "kind", "") == "autoregressive":     # fp/executor.py:447-449
                rec["prefill_calls"] = 1
                rec["decode_calls"] = gen.n_iterations - 1
            rec["generation_cost"] = gen.total_cost
            rec["emissions"].append(_emission(t, now + cost, emit, land, cost, a.values,
                                              [age]))
        else:
            rec["dropped_observations"] = 1
        rec["env_error"] = port.seal()
        trace.append(rec)
    return OracleResult(actions, trace, requests)


def _mode_header(mode, interval, duration, config, env):
    return {"type": "header", "schema": 1, "mode": mode, "engine": "virtual",
            "frame_interval": interval, "duration": duration, "config": config,
            "success_threshold": getattr(env, "success_threshold", None)}


def run_parallel(policy, env, workers: int, duration: int, frame_interval=None,
                 capacity: float = 1.0) -> OracleResult:
    """fp/executor.py:477-576 (PAR): `workers` private requests share one unit of
    compute by processor sharing; a worker that finishes inside a frame takes
    that frame's observation again at once (just-in-fit), one that finishes on
    the boundary waits for the next frame's observation."""
    if workers < 1:
        raise ValueError("need at least one worker")
    gen = policy.generation
    cost = policy.sequential_cost
    interval = frame_interval if frame_interval is not None else cost
    trace = [_mode_header("par", interval, duration,
                          {"workers": workers, "capacity": capacity, "request_cost": cost}, env)]
    port = _Landing(env, policy)
    actions, requests = [], []
    running = []                        # [worker, obs, birth frame, birth time, work left] per job
    idle = list(range(workers))

    def complete(job, when, rec):
        worker, obs, birth, born_at, _ = job
        ctx = policy.perception.perceive(obs)
        state = gen.initial_state(seed=birth)
        for _ in range(gen.n_iterations):
            state = gen.step(state, ctx)
        land = int(math.ceil(when / interval - 1e-12))
        emit = land - 1
        age = float(emit - ctx.produced_frame)
        a = gen.finish(state, emitted_frame=emit, staleness_profile=(age,) * gen.n_iterations)
        r = Request(observation_id=obs.id, birth_frame=birth, birth_time=born_at,
                    completion_frame=land, completion_time=when, jct=when - born_at)
        r.context_versions.append(1)
        requests.append(r)
        actions.append(a)
        port.queue.append((land, when, a))
        rec["emissions"].append(_emission(birth, when, emit, land, r.jct, a.values, [age]))

    for t in range(duration):
        now = float(t) * interval
        end = now + interval
        rec = _frame_record(t, now)
        rec["end"] = end
        obs = port.boundary(t)
        rec["superseded_actions"] = port.last_superseded
        taken = False
        if idle:
            running.append([idle.pop(0), obs, t, now, cost])
            taken = True
        clock = now
        while running and clock < end - 1e-12:
            rate = capacity / len(running)
            first = min(running, key=lambda j: j[4])
            finish_at = clock + first[4] / rate
            if finish_at > end + 1e-12:             # nobody finishes in this frame
                for j in running:
                    j[4] -= (end - clock) * rate
                clock = end
                break
            for j in running:
                j[4] -= (finish_at - clock) * rate
            clock = finish_at
            for j in [j for j in running if j[4] <= 1e-9]:
                running.remove(j)
                complete(j, finish_at, rec)
                if finish_at >= end - 1e-9:
                    idle.append(j[0])
                else:
                    running.append([j[0], obs, t, finish_at, cost])
                    taken = True
        if not taken:
            rec["dropped_observations"] = 1
        rec["env_error"] = port.seal()
        trace.append(rec)
    return OracleResult(actions, trace, requests)


def run_decoupled(policy, env, duration: int, frame_interval=None) -> OracleResult:
    """fp/executor.py:583-701 (DEC): perception free-runs on its own worker,
    publishing into a 2-slot store; generation starts a full request from the
    newest context as soon as one derived from an unused observation exists.
    Event order inside a frame: publish < generation start < generation end."""
    gen = policy.generation
    p_cost = policy.perception.total_cost
    g_cost = gen.total_cost
    interval = frame_interval if frame_interval is not None else policy.sequential_cost
    trace = [_mode_header("dec", interval, duration,
                          {"perception_cost": p_cost, "generation_cost": g_cost}, env)]
    port = _Landing(env, policy)
    actions, requests = [], []
    version, n_pub, latest = 0, 0, None     # latest: (frame, version, ctx, source obs id)
    used_versions = set()
    p_start, p_obs = 0.0, None
    g_free, job = 0.0, None                  # job: (end, start, version, ctx, source, state)
    last_used_obs, fresh_at = -1, None
    order = {"publish": 0, "gen_start": 1, "gen_done": 2}
    for t in range(duration):
        now = float(t) * interval
        end = now + interval
        rec = _frame_record(t, now)
        rec["end"] = end
        newest_obs = port.boundary(t)
        rec["superseded_actions"] = port.last_superseded
        if p_obs is None:
            p_obs = newest_obs
        while True:
            cands = []
            pub_at = p_start + p_cost
            if pub_at < end - 1e-9:
                cands.append(("publish", pub_at))
            if job is None and fresh_at is not None:
                g_at = max(g_free, fresh_at)
                if g_at < end - 1e-9:
                    cands.append(("gen_start", g_at))
            if job is not None and job[0] <= end + 1e-9:
                cands.append(("gen_done", job[0]))
            if not cands:
                break
            what, when = min(cands, key=lambda c: (c[1], order[c[0]]))
            if what == "publish":
                ctx = policy.perception.perceive(p_obs)
                version += 1
                n_pub += 1
                if ctx.produced_frame != t:          # the store stamps the publishing frame
                    ctx = dataclasses.replace(ctx, produced_frame=t)
                latest = (t, version, ctx, p_obs.id)
                rec["publishes"].append(version)
                rec["perception"].append({"start": p_start, "end": when, "obs": p_obs.id, "version": version})
                if fresh_at is None and p_obs.id > last_used_obs:
                    fresh_at = when
                p_start, p_obs = when, newest_obs
            elif what == "gen_start":
                _, ver, ctx, src = latest
                state = gen.initial_state(seed=int(round(when)))
                for _ in range(gen.n_iterations):
                    state = gen.step(state, ctx)
                used_versions.add(ver)
                last_used_obs, fresh_at = src, None
                job = (when + g_cost, when, ver, ctx, src, state)
                g_free = when + g_cost
                if getattr(policy, "kind", "") == "autoregressive":     # fp/executor.py:670-672
                    rec["prefill_calls"] += 1
                    rec["decode_calls"] += gen.n_iterations - 1
                rec["generation_cost"] += g_cost
            else:
                fin, began, ver, ctx, src, state = job
                land = int(math.ceil(fin / interval - 1e-12))
                emit = land - 1
                age = float(emit - ctx.produced_frame)
                a = gen.finish(state, emitted_frame=emit, staleness_profile=(age,) * gen.n_iterations)
                actions.append(a)
                r = Request(observation_id=src, birth_frame=int(began // interval), birth_time=began,
                            completion_frame=land, completion_time=fin, jct=fin - began)
                r.context_versions.append(ver)
                requests.append(r)
                port.queue.append((land, fin, a))
                rec["emissions"].append(_emission(src, fin, emit, land, r.jct, a.values, [age]))
                job = None
        rec["published_total"] = n_pub
        rec["consumed_total"] = len(used_versions)
        rec["env_error"] = port.seal()
        trace.append(rec)
    return OracleResult(actions, trace, requests)
