"""Frame-clocked pipeline executor on two CUDA streams.

Drop-in for the reference's `run_pipelined` / `run_sequential`
(fp/executor.py:200-461): same signatures, same `PipelineConfig`, same
`RunResult` / `RequestRecord`, same trace schema 1.  What changes is where
the work happens:

* perception stages, the finalize and the ring publish run on a perception
  stream P; every generation stage active in a frame is folded into ONE
  batched denoise launch chain on a generation stream G (the reference loops
  over stages and iterations in Python, fp/executor.py:325-331);
* the handoff is event based: G waits on the event recorded after the
  publish of the context it reads (offset 0 serialises publish -> fetch inside
  the frame as the SPEC demands; offset -1 lets P(t) overlap G(t)); P waits on
  the last G read of a slot before overwriting it (the K = 2 ring-reuse hazard)
  and on the finish of a lane's previous request before re-using the lane;
* the slot/version a stage consumes is decided by the same host rules as the
  reference (so the schedule is bit-identical) and re-resolved on the device,
  which logs the version it actually read.

Two clocks are available.  `clock="virtual"` (the default, as in the
reference) computes frame times from the policy's cost units exactly as
fp/executor.py:350-374 does, so traces are comparable field for field with the
reference's.  `clock="device"` stamps frame starts, frame ends, emissions and
JCTs with CUDA events (seconds); it requires `frame_interval=None`
(as-fast-as-possible frames, per-dependency waits).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .context import ContextKind
from .errors import ConfigInvalid, DeadlockDetected, IncompleteGeneration, NotYetPublished
from .partition import StagePlan, plan_stages
from .policy import ActionOutput, Observation

TRACE_SCHEMA = 1


@dataclass(frozen=True)
class PipelineConfig:
    """Pipelined search point (fp/executor.py:48-103): degrees, offset, skew,
    frame policy.  Identical fields and validation rules."""

    pp_perception: int = 1
    pp_generation: int = 1
    fetch_offset: Optional[int] = None
    alpha: float = 0.0
    frame_interval: Optional[float] = None
    merge_autoregressive: Optional[bool] = None
    store_capacity: int = 2
    read_policy: str = "snapshot"
    overrun_policy: str = "stretch"

    def resolve_offset(self, kind) -> int:
        if self.fetch_offset is not None:
            return self.fetch_offset
        return -1 if kind == ContextKind.AUTOREGRESSIVE else 0

    def resolve_merge(self, kind) -> bool:
        if self.merge_autoregressive is not None:
            return bool(self.merge_autoregressive) and kind == ContextKind.AUTOREGRESSIVE
        return kind == ContextKind.AUTOREGRESSIVE

    def validate(self, policy) -> None:
        if self.pp_perception < 1 or self.pp_generation < 1:
            raise ConfigInvalid("pipeline degrees must be positive")
        if self.pp_perception + self.pp_generation < 2:
            raise ConfigInvalid("pipelined mode needs at least two stages")
        off = self.resolve_offset(policy.kind)
        if off > 0:
            raise ConfigInvalid("fetch_offset must be <= 0")
        if -off >= self.store_capacity:
            raise ConfigInvalid(f"|fetch_offset| = {-off} must be below store capacity "
                                f"{self.store_capacity}")
        if self.pp_perception > len(policy.perception.layers):
            raise ConfigInvalid("more perception stages than layers")
        if self.read_policy not in ("snapshot", "live"):
            raise ConfigInvalid(f"unknown read policy {self.read_policy!r}")
        if self.overrun_policy not in ("stretch", "drop"):
            raise ConfigInvalid(f"unknown overrun policy {self.overrun_policy!r}")
        if self.frame_interval is not None and self.frame_interval <= 0:
            raise ConfigInvalid("frame interval must be positive")

    def to_dict(self) -> dict:
        return {"pp_perception": self.pp_perception, "pp_generation": self.pp_generation,
                "fetch_offset": self.fetch_offset, "alpha": self.alpha,
                "frame_interval": self.frame_interval,
                "merge_autoregressive": self.merge_autoregressive,
                "store_capacity": self.store_capacity, "read_policy": self.read_policy,
                "overrun_policy": self.overrun_policy}


@dataclass
class RequestRecord:
    observation_id: int
    birth_frame: int
    birth_time: float
    completion_frame: int = -1
    completion_time: float = -1.0
    jct: float = -1.0
    context_versions: list = field(default_factory=list)


@dataclass
class RunResult:
    actions: list
    trace: list
    requests: list
    agent_actions: list = field(default_factory=list)   # per agent (agent 0 == actions)
    device_versions: Optional[np.ndarray] = None        # version read in-kernel, per frame
    frame_times: Optional[dict] = None                  # device clock: raw event seconds

    @property
    def header(self) -> dict:
        return self.trace[0]


# ---------------------------------------------------------------- helpers

def _header(mode, interval, duration, config, envs, clock):
    env0 = envs[0] if envs else None
    return {"type": "header", "schema": TRACE_SCHEMA, "mode": mode,
            "engine": "virtual" if clock == "virtual" else "b200",
            "device": "b200", "clock": clock, "frame_interval": interval,
            "duration": duration, "config": config,
            "success_threshold": getattr(env0, "success_threshold", None)}


def _frame(t, now):
    return {"type": "frame", "frame": t, "start": now, "perception": [], "generation": [],
            "publishes": [], "emissions": [], "prefill_calls": 0, "decode_calls": 0,
            "generation_cost": 0.0, "dropped_observations": 0}


class _Port:
    """Per-agent environment boundary (fp/executor.py:146-184): land the newest
    due action, then observe.  env None -> synthetic observation source."""

    def __init__(self, env, policy, agent, source):
        self.env, self.policy, self.agent, self.source = env, policy, agent, source
        self.pending = []           # (land_frame, order, emission)
        self.last_superseded = 0

    def schedule(self, land_frame, order, emission):
        self.pending.append((land_frame, order, emission))

    def boundary(self, frame, materialize):
        due = [p for p in self.pending if p[0] == frame]
        self.last_superseded = 0
        if due:
            self.pending = [p for p in self.pending if p[0] != frame]
            newest = max(due, key=lambda p: p[1])
            self.last_superseded = len(due) - 1
            if self.env is not None:
                action = materialize(newest[2], self.agent)
                self.env.apply_action(self.policy.generation.decode_action(action))
        if self.env is not None:
            return self.env.observe(frame)
        if self.source is not None:
            return self.source(self.agent, frame)
        synth = getattr(self.policy, "synthetic_observation", None)
        if synth is not None:
            return synth(self.agent, frame)
        return Observation(frame=frame, vector=np.zeros(4))     # fp/executor.py:142-143

    def seal(self):
        if self.env is None:
            return None
        self.env.advance_frame()
        return self.env.last_error


class _Device:
    """Streams, events and the policy session for one run."""

    def __init__(self, policy, *, capacity, lanes, agents, max_outputs, max_frames, clock,
                 pp_perception=1):
        import torch
        self.torch = torch
        self.clock = clock
        # generation gets the higher priority: the persistent denoise kernel needs
        # all of its CTAs resident, so its pending CTAs must win SMs over the
        # perception kernels that run concurrently on P
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
            else (0, -1)
        import os
        gprio = -1 if os.environ.get("AURAS_G_PRIORITY", "1") == "1" else 0
        # disaggregated policies put perception (P) on their own GPU; events carry
        # the cross-device ordering
        pd = getattr(policy, "perception_device", None)
        self.disagg = pd is not None
        self.P = torch.cuda.Stream(device=pd, priority=0) if self.disagg else torch.cuda.Stream(priority=0)
        self.G = torch.cuda.Stream(priority=gprio)
        self.session = policy.open_session(capacity=capacity, lanes=lanes, agents=agents,
                                           max_outputs=max_outputs, max_frames=max_frames,
                                           p_stream=self.P, g_stream=self.G,
                                           pp_perception=pp_perception)
        self.store = self.session.store
        self.pub_event = {}          # context frame -> event after its publish (P)
        self.ingest_event = {}       # request -> event after ingest (P)
        self.slot_read = {}          # slot -> last G event that read it
        self.lane_free = {}          # lane -> G event after the previous occupant's finish
        self.out_ready = {}          # out_index -> G event after the finish that wrote it
        self.t_start, self.t_end = {}, {}
        self.origin = None
        self.throttle = []
        # A policy whose denoise step is a whole-GPU persistent kernel asks for
        # interleaving: perception of frame t+1 is ordered after generation of
        # frame t (still two streams + events, but no SM contention).
        import os
        env = os.environ.get("AURAS_INTERLEAVE_PG")
        self.interleave = (env == "1") if env is not None else bool(getattr(self.session, "exclusive", False))
        self.last_gen_end = None

    def event(self, stream, timing=False):
        ev = self.torch.cuda.Event(enable_timing=timing)
        ev.record(stream)
        return ev

    def begin_frame(self, t, window):
        # bound how far the host runs ahead of the device (event/pinned-buffer lifetimes)
        if len(self.throttle) >= window:
            self.throttle.pop(0).synchronize()
        if self.interleave and self.last_gen_end is not None:
            self.P.wait_event(self.last_gen_end)
        if self.clock == "device":
            # frame clocks are G-device events when P lives on another GPU
            # (elapsed_time needs both events on one device)
            ev = self.event(self.G if self.disagg else self.P, timing=True)
            self.t_start[t] = ev
            if self.origin is None:
                self.origin = ev

    def end_frame(self, t):
        ev = self.event(self.G, timing=self.clock == "device")
        if self.clock == "device":
            self.t_end[t] = ev
        self.throttle.append(ev)
        self.last_gen_end = ev

    def ingest(self, t, lane, observations):
        ev = self.lane_free.pop(lane, None)
        if ev is not None:
            self.P.wait_event(ev)
        self.session.ingest(t, lane, observations)
        self.ingest_event[t] = self.event(self.P)

    def publish(self, lane, frame, slot, version):
        ev = self.slot_read.get(slot)
        if ev is not None:
            self.P.wait_event(ev)
        self.session.publish(lane, frame, slot, version)
        self.pub_event[frame] = self.event(self.P)
        for f in [f for f in self.pub_event if f < frame - 4 * self.store.capacity]:
            del self.pub_event[f]

    def generate(self, ctx_frame, slot, log_index, batch, first_use):
        self.G.wait_event(self.pub_event[ctx_frame])
        for b in first_use:
            ev = self.ingest_event.pop(b, None)
            if ev is not None:
                self.G.wait_event(ev)
        self.session.fetch(ctx_frame, log_index)
        self.session.generate(batch)
        self.slot_read[slot] = self.event(self.G)

    def finish(self, lane, out_index):
        self.session.finish(lane, out_index)
        ev = self.event(self.G)
        self.lane_free[lane] = ev
        # the action row is written on G (a non-blocking stream): a mid-run
        # host read must wait for this event, not just issue a D2H
        self.out_ready[out_index] = ev

    def wait_output(self, out_index):
        ev = self.out_ready.pop(out_index, None)
        if ev is not None:
            ev.synchronize()

    def republish(self, src_slot, slot, frame, version):
        """Token-prefix update of the shared context (autoregressive policies)."""
        ev = self.slot_read.get(slot)
        if ev is not None:
            self.P.wait_event(ev)
        self.session.republish(src_slot, slot, frame, version)
        self.pub_event[frame] = self.event(self.P)

    def seconds(self, ev):
        return self.origin.elapsed_time(ev) / 1e3

    def synchronize(self):
        self.P.synchronize()
        self.G.synchronize()
        self.out_ready.clear()


class _Emissions:
    """Emitted actions: device rows materialised lazily (one D2H at the end,
    or one per action when a closed loop needs it).  Session rows are
    [agents, ...] arrays; `session.action_values(row)` turns one agent's row
    into the ActionOutput values tuple."""

    def __init__(self, device, policy, agents):
        self.device, self.policy, self.agents = device, policy, agents
        self.items = []             # (out_index, emitted_frame, staleness_profile)
        self.cache = {}

    def add(self, out_index, emitted_frame, profile):
        self.items.append((out_index, emitted_frame, profile))
        return len(self.items) - 1

    def _make(self, k, rows):
        _, emitted, prof = self.items[k]
        sess = self.device.session
        return [ActionOutput(kind=self.policy.kind, values=sess.action_values(rows[a]),
                             emitted_frame=emitted, staleness_profile=prof)
                for a in range(self.agents)]

    def materialize(self, k, agent):
        if k not in self.cache:
            out_index = self.items[k][0]
            self.device.wait_output(out_index)      # the finish kernel on G has written the row
            self.cache[k] = self._make(k, self.device.session.read_action(out_index))
        return self.cache[k][agent]

    def all(self):
        n = len(self.items)
        per_agent = [[] for _ in range(self.agents)]
        if n == 0:
            return per_agent
        rows = self.device.session.read_actions(n)
        for k in range(n):
            if k not in self.cache:
                self.cache[k] = self._make(k, rows[k])
            for a in range(self.agents):
                per_agent[a].append(self.cache[k][a])
        return per_agent


def _agents_and_envs(policy, env, agents):
    if isinstance(env, (list, tuple)):
        envs = list(env)
    else:
        n = agents if agents is not None else getattr(policy, "agents", 1)
        envs = [env] * n if env is None else [env]
    if agents is not None and len(envs) != agents:
        raise ConfigInvalid(f"{len(envs)} environments for {agents} agents")
    return envs


def _require_plugin(policy):
    """The device plugins (open_session), or a reference-style duck-typed policy
    (fp/policy.py:46-272 protocol) wrapped to run its callbacks on the host."""
    if hasattr(policy, "open_session"):
        return policy
    from .policy import HostPolicy, is_reference_plugin
    if is_reference_plugin(policy):
        return HostPolicy(policy)
    raise ConfigInvalid("the B200 engine needs a policy plugin: make_conditioning_policy / "
                        "make_diffusion_policy / make_autoregressive_policy from paper_2509_09560_b200, "
                        "or an object with the reference's perception (start / apply_layers / finalize) "
                        "and generation (initial_state / step / finish) protocol")


# ---------------------------------------------------------------- pipelined mode

def run_pipelined(cfg: PipelineConfig, policy, env, duration: int, *, clock: str = "virtual",
                  agents: Optional[int] = None, frame_source=None, frame_hook=None) -> RunResult:
    """fp/executor.py:200-399 on the B200.  `env` may be one environment, a list
    (one per agent, batched into the same kernels), or None (synthetic
    observations from `frame_source(agent, frame)` when given)."""
    policy = _require_plugin(policy)
    cfg.validate(policy)
    if clock not in ("virtual", "device"):
        raise ConfigInvalid(f"unknown clock {clock!r}")
    if clock == "device" and cfg.frame_interval is not None:
        raise ConfigInvalid("clock='device' runs frames as fast as possible (frame_interval=None)")
    _lib.load()
    offset = cfg.resolve_offset(policy.kind)
    merge = cfg.resolve_merge(policy.kind)
    plan: StagePlan = plan_stages(policy.perception.layer_costs, cfg.pp_perception,
                                  policy.generation.n_iterations, cfg.pp_generation, cfg.alpha)
    pp_p, pp_g = cfg.pp_perception, cfg.pp_generation
    shift = pp_p - 1 - offset
    span = shift + pp_g
    starts = plan.stage_starts()
    gen = policy.generation
    envs = _agents_and_envs(policy, env, agents)
    A = len(envs)
    lanes = span + 2
    p_cost = [sum(policy.perception.layer_costs[a:b]) for a, b in plan.perception_stages]

    dev = _Device(policy, capacity=cfg.store_capacity, lanes=lanes, agents=A,
                  max_outputs=duration, max_frames=duration, clock=clock, pp_perception=pp_p)
    store = dev.store
    ports = [_Port(e, policy, a, frame_source) for a, e in enumerate(envs)]
    emis = _Emissions(dev, policy, A)
    trace = [_header("pipe", cfg.frame_interval, duration,
                     {"pipeline": cfg.to_dict(), "plan": plan.to_dict(), "fetch_offset": offset,
                      "merged": merge}, envs, clock)]
    live = {}
    records = []
    emitted_rows = []                 # (frame record, emission dict, request record)
    now, skip = 0.0, 0
    window = max(4, lanes)
    for t in range(duration):
        if frame_hook is not None:
            frame_hook(t, dev, emis)
        dev.begin_frame(t, window)
        rec = _frame(t, now)
        obs = [port.boundary(t, emis.materialize) for port in ports]
        rec["superseded_actions"] = ports[0].last_superseded
        if skip > 0:
            skip -= 1
            rec["dropped_observations"] += 1
        else:
            lane = t % lanes
            r = RequestRecord(observation_id=obs[0].id, birth_frame=t, birth_time=now)
            dev.ingest(t, lane, obs)
            live[t] = {"rec": r, "lane": lane, "ages": [], "steps": 0, "used": False,
                       "obs_id": obs[0].id}
            records.append(r)

        early = None
        if offset <= -1 and cfg.read_policy == "snapshot":
            try:
                early = store.resolve(t, offset)
            except NotYetPublished:
                early = None

        side, pub_cost, published = [], 0.0, False
        for s in range(1, pp_p + 1):
            b = t - s + 1
            item = live.get(b)
            if item is None:
                continue
            lo, hi = plan.perception_stages[s - 1]
            dev.session.perceive(item["lane"], lo, hi)
            entry = {"request": b, "stage": s, "cost": p_cost[s - 1], "published_version": None}
            if s == pp_p:
                slot, version = store.reserve(t, item["obs_id"])
                dev.publish(item["lane"], t, slot, version)
                entry["published_version"] = version
                rec["publishes"].append(version)
                pub_cost, published = p_cost[s - 1], True
            else:
                side.append(p_cost[s - 1])
            rec["perception"].append(entry)

        # optional mid-frame hook: the frame's observation and perception are queued,
        # its generation not yet (a serving loop blocks on the previous action here)
        mid = getattr(frame_hook, "mid", None)
        if mid is not None:
            mid(t, dev, emis)

        active = []
        for j in range(1, pp_g + 1):
            b = t - shift - (j - 1)
            if b in live:
                active.append((j, b, live[b]))
        gen_costs = []
        if active:
            if early is not None:
                version, ctx_frame, slot = early
            else:
                try:
                    version, ctx_frame, slot = store.resolve(t, offset)
                except NotYetPublished:
                    if t + offset < pp_p - 1:
                        raise DeadlockDetected(
                            f"frame {t}: context for frame {t + offset} can never exist")
                    version, ctx_frame, slot = store.resolve_latest()
            ar = policy.kind == ContextKind.AUTOREGRESSIVE
            if merge and ar:
                # one merged prefill over the shared context serves every stage (fp/executor.py:321-324)
                rec["prefill_calls"] += 1
                rec["generation_cost"] += gen.prefill_cost
                gen_costs.append(gen.prefill_cost)
            batch, first = [], []
            for j, b, item in active:
                iters = plan.generation_stages[j - 1]
                batch.append((item["lane"], starts[j - 1], iters))
                if not item["used"]:
                    first.append(b)
                    item["used"] = True
                age = float(b + span - 1 - ctx_frame)
                item["ages"].extend([age] * iters)
                item["steps"] += iters
                item["rec"].context_versions.append(version)
                if not (merge and ar):
                    c = gen.prefill_cost + max(iters - 1, 0) * gen.decode_cost if ar else iters * gen.step_cost
                    gen_costs.append(c)
                    rec["generation_cost"] += c
                    if ar:
                        rec["prefill_calls"] += 1
                        rec["decode_calls"] += max(iters - 1, 0)
                rec["generation"].append({"request": b, "stage": j, "iterations": iters,
                                          "context_version": version, "context_frame": ctx_frame,
                                          "context_age_at_emission": age})
            dev.generate(ctx_frame, slot, t, batch, first)
            if ar:
                # the freshest token prefix goes back into the shared context as a new
                # version of this frame's context (fp/executor.py:345-348)
                src, slot2, ver2 = store.reserve_token_update(t)
                dev.republish(src, slot2, t, ver2)

        # frame duration in cost units (fp/executor.py:350-374)
        if offset == 0 and gen_costs and published:
            busiest = max(side + [pub_cost + max(gen_costs)])
        else:
            pool = side + gen_costs + ([pub_cost] if published else [])
            busiest = max(pool) if pool else 0.0
        interval = cfg.frame_interval
        if interval is None:
            dur = busiest
        elif busiest <= interval:
            dur = interval
        elif cfg.overrun_policy == "stretch":
            dur = busiest
            rec["overrun"] = True
        else:
            q = math.ceil(busiest / interval)
            dur = q * interval
            skip += q - 1
            rec["overrun"] = True
        now += dur
        rec["end"] = now

        b_done = t - span + 1
        item = live.pop(b_done, None)
        if item is not None:
            if item["steps"] < gen.n_iterations:
                raise IncompleteGeneration(f"{item['steps']}/{gen.n_iterations} iterations applied")
            out_index = len(emis.items)
            dev.finish(item["lane"], out_index)
            k = emis.add(out_index, t, tuple(item["ages"]))
            r = item["rec"]
            r.completion_frame = t + 1
            r.completion_time = now
            r.jct = now - r.birth_time
            for port in ports:
                port.schedule(t + 1, k, k)
            ages = item["ages"]
            em = {"request": b_done, "time": now, "emission_frame": t, "land_frame": t + 1,
                  "jct": r.jct, "action": None, "staleness_min": min(ages),
                  "staleness_mean": float(np.mean(ages)), "staleness_max": max(ages),
                  "staleness_final": ages[-1]}
            rec["emissions"].append(em)
            emitted_rows.append((rec, em, r, k))
        rec["env_error"] = ports[0].seal()
        for port in ports[1:]:
            port.seal()
        dev.end_frame(t)
        trace.append(rec)

    if frame_hook is not None:
        frame_hook(duration, dev, emis)
    dev.synchronize()
    per_agent = emis.all()
    for rec_, em, r, k in emitted_rows:
        em["action"] = list(per_agent[0][k].values)
    if clock == "device":
        _apply_device_clock(dev, trace, records, emitted_rows)
    versions = dev.session.read_version_log(duration)
    dev.session.close()
    return RunResult(actions=per_agent[0], trace=trace, requests=records, agent_actions=per_agent,
                     device_versions=versions,
                     frame_times=_frame_times(dev) if clock == "device" else None)


def _frame_times(dev):
    return {"start": {t: dev.seconds(e) for t, e in dev.t_start.items()},
            "end": {t: dev.seconds(e) for t, e in dev.t_end.items()}}


def _apply_device_clock(dev, trace, records, emitted_rows):
    start = {t: dev.seconds(e) for t, e in dev.t_start.items()}
    end = {t: dev.seconds(e) for t, e in dev.t_end.items()}
    for rec in trace[1:]:
        rec["start"], rec["end"] = start[rec["frame"]], end[rec["frame"]]
    for r in records:
        r.birth_time = start[r.birth_frame]
    for rec, em, r, k in emitted_rows:
        done = end[rec["frame"]]
        r.completion_time = done
        r.jct = done - r.birth_time
        em["time"], em["jct"] = done, r.jct


# ---------------------------------------------------------------- sequential mode

def run_sequential(policy, env, duration: int, frame_interval: Optional[float] = None, *,
                   clock: str = "virtual", agents: Optional[int] = None,
                   frame_source=None, frame_hook=None) -> RunResult:
    """fp/executor.py:406-461 on the B200: one request at a time (depth 1);
    observations arriving while a request is in flight are dropped."""
    policy = _require_plugin(policy)
    if clock not in ("virtual", "device"):
        raise ConfigInvalid(f"unknown clock {clock!r}")
    _lib.load()
    gen = policy.generation
    cost = policy.sequential_cost
    interval = frame_interval if frame_interval is not None else cost
    per_request = max(1, math.ceil(cost / interval - 1e-12))
    envs = _agents_and_envs(policy, env, agents)
    A = len(envs)
    lanes = 2
    dev = _Device(policy, capacity=2, lanes=lanes, agents=A, max_outputs=duration,
                  max_frames=duration, clock=clock)
    store = dev.store
    ports = [_Port(e, policy, a, frame_source) for a, e in enumerate(envs)]
    emis = _Emissions(dev, policy, A)
    trace = [_header("seq", interval, duration, {"request_cost": cost}, envs, clock)]
    records, emitted_rows = [], []
    free_at = 0
    n_layers = len(policy.perception.layers)
    for t in range(duration):
        if frame_hook is not None:
            frame_hook(t, dev, emis)
        dev.begin_frame(t, 4)
        now = t * interval
        rec = _frame(t, now)
        rec["end"] = now + interval
        obs = [port.boundary(t, emis.materialize) for port in ports]
        rec["superseded_actions"] = ports[0].last_superseded
        if t >= free_at:
            lane = t % lanes
            r = RequestRecord(observation_id=obs[0].id, birth_frame=t, birth_time=now)
            dev.ingest(t, lane, obs)
            dev.session.perceive(lane, 0, n_layers)
            slot, version = store.reserve(t, obs[0].id)
            dev.publish(lane, t, slot, version)
            dev.generate(t, slot, t, [(lane, 0, gen.n_iterations)], [t])
            emit = t + per_request - 1
            age = float(emit - t)
            done = now + cost
            land = t + per_request
            r.completion_frame, r.completion_time, r.jct = land, done, cost
            r.context_versions.append(1)        # the reference reports version 1 (fp/executor.py:442)
            records.append(r)
            out_index = len(emis.items)
            dev.finish(lane, out_index)
            k = emis.add(out_index, emit, (age,) * gen.n_iterations)
            for port in ports:
                port.schedule(land, k, k)
            free_at = land
            rec["generation_cost"] = gen.total_cost
            if policy.kind == ContextKind.AUTOREGRESSIVE:
                rec["prefill_calls"] = 1
                rec["decode_calls"] = gen.n_iterations - 1
            em = {"request": t, "time": done, "emission_frame": emit, "land_frame": land,
                  "jct": cost, "action": None, "staleness_min": age, "staleness_mean": age,
                  "staleness_max": age, "staleness_final": age}
            rec["emissions"].append(em)
            emitted_rows.append((rec, em, r, k))
        else:
            rec["dropped_observations"] = 1
        rec["env_error"] = ports[0].seal()
        for port in ports[1:]:
            port.seal()
        dev.end_frame(t)
        trace.append(rec)
    if frame_hook is not None:
        frame_hook(duration, dev, emis)
    dev.synchronize()
    per_agent = emis.all()
    for rec_, em, r, k in emitted_rows:
        em["action"] = list(per_agent[0][k].values)
    if clock == "device":
        _apply_device_clock(dev, trace, records, emitted_rows)
    versions = dev.session.read_version_log(duration)
    dev.session.close()
    return RunResult(actions=per_agent[0], trace=trace, requests=records, agent_actions=per_agent,
                     device_versions=versions,
                     frame_times=_frame_times(dev) if clock == "device" else None)


# ---------------------------------------------------------------- PAR / DEC baselines

def _ingest_keyed(dev, key, seed, lane, observations):
    """dev.ingest with the request state seeded by `seed` but the ingest event
    filed under `key` (PAR jobs share dispatch frames; DEC seeds by time).
    key None: nothing consumes the event (DEC's perception lane: its publish
    is ordered by the publish event), so none is kept."""
    ev = dev.lane_free.pop(lane, None)
    if ev is not None:
        dev.P.wait_event(ev)
    dev.session.ingest(seed, lane, observations)
    if key is not None:
        dev.ingest_event[key] = dev.event(dev.P)


def run_parallel(policy, env, workers: int, duration: int, frame_interval: Optional[float] = None,
                 capacity: float = 1.0, *, clock: str = "virtual", agents: Optional[int] = None,
                 frame_source=None, frame_hook=None) -> RunResult:
    """fp/executor.py:477-576 (PAR) on the B200: `workers` private requests
    share one compute capacity by processor sharing; a worker finishing inside
    a frame regrabs that frame's observation (just-in-fit).  The schedule is
    the reference's own float event loop; every job's perception, context
    publish, n denoise iterations and finish run on the device when it is
    dispatched (its context in its own ring slot), so its action is ready by
    the frame it lands.  With capacity 1 the jobs' device work is sequential
    -- the processor-sharing model's total throughput."""
    policy = _require_plugin(policy)
    if workers < 1:
        raise ConfigInvalid("need at least one worker")
    if clock not in ("virtual", "device"):
        raise ConfigInvalid(f"unknown clock {clock!r}")
    _lib.load()
    gen = policy.generation
    cost = policy.sequential_cost
    interval = frame_interval if frame_interval is not None else cost
    envs = _agents_and_envs(policy, env, agents)
    A = len(envs)
    lanes = workers + 2
    max_jobs = duration * (workers + 1) + 8
    dev = _Device(policy, capacity=max(2, workers + 2), lanes=lanes, agents=A, max_outputs=max_jobs,
                  max_frames=max_jobs, clock=clock)
    store = dev.store
    ports = [_Port(e, policy, a, frame_source) for a, e in enumerate(envs)]
    emis = _Emissions(dev, policy, A)
    trace = [_header("par", interval, duration,
                     {"workers": workers, "capacity": capacity, "request_cost": cost}, envs, clock)]
    records, emitted_rows = [], []
    n_layers = len(policy.perception.layers)
    running = []                 # [worker, job id, obs list, birth frame, birth time, work left]
    idle = list(range(workers))
    n_jobs = [0]

    def dispatch(worker, obs, t, when):
        j = n_jobs[0]
        n_jobs[0] += 1
        lane = j % lanes
        _ingest_keyed(dev, j, t, lane, obs)
        dev.session.perceive(lane, 0, n_layers)
        slot, version = store.reserve(j, obs[0].id)
        dev.publish(lane, j, slot, version)
        dev.generate(j, slot, j, [(lane, 0, gen.n_iterations)], [j])
        running.append([worker, j, obs, t, when, cost])

    def complete(job, when, rec):
        _, j, obs, birth, born_at, _ = job
        land = int(math.ceil(when / interval - 1e-12))
        emit = land - 1
        age = float(emit - birth)                  # the context is produced from the dispatch frame
        r = RequestRecord(observation_id=obs[0].id, birth_frame=birth, birth_time=born_at,
                          completion_frame=land, completion_time=when, jct=when - born_at)
        r.context_versions.append(1)             # the reference reports version 1 (fp/executor.py:520)
        records.append(r)
        out_index = len(emis.items)
        dev.finish(j % lanes, out_index)
        k = emis.add(out_index, emit, (age,) * gen.n_iterations)
        for port in ports:
            port.schedule(land, k, k)
        em = {"request": birth, "time": when, "emission_frame": emit, "land_frame": land,
              "jct": r.jct, "action": None, "staleness_min": age, "staleness_mean": age,
              "staleness_max": age, "staleness_final": age}
        rec["emissions"].append(em)
        emitted_rows.append((rec, em, r, k))

    for t in range(duration):
        if frame_hook is not None:
            frame_hook(t, dev, emis)
        dev.begin_frame(t, 4)
        now = float(t) * interval
        end = now + interval
        rec = _frame(t, now)
        rec["end"] = end
        obs = [port.boundary(t, emis.materialize) for port in ports]
        rec["superseded_actions"] = ports[0].last_superseded
        taken = False
        if idle:
            dispatch(idle.pop(0), obs, t, now)
            taken = True
        clock_t = now
        while running and clock_t < end - 1e-12:
            rate = capacity / len(running)
            first = min(running, key=lambda jb: jb[5])
            finish_at = clock_t + first[5] / rate
            if finish_at > end + 1e-12:
                for jb in running:
                    jb[5] -= (end - clock_t) * rate
                clock_t = end
                break
            for jb in running:
                jb[5] -= (finish_at - clock_t) * rate
            clock_t = finish_at
            for jb in [jb for jb in running if jb[5] <= 1e-9]:
                running.remove(jb)
                complete(jb, finish_at, rec)
                if finish_at >= end - 1e-9:
                    idle.append(jb[0])
                else:
                    dispatch(jb[0], obs, t, finish_at)
                    taken = True
        if not taken:
            rec["dropped_observations"] = 1
        rec["env_error"] = ports[0].seal()
        for port in ports[1:]:
            port.seal()
        dev.end_frame(t)
        trace.append(rec)
    if frame_hook is not None:
        frame_hook(duration, dev, emis)
    dev.synchronize()
    per_agent = emis.all()
    for rec_, em, r, k in emitted_rows:
        em["action"] = list(per_agent[0][k].values)
    if clock == "device":
        _apply_device_clock(dev, trace, records, emitted_rows)
    versions = dev.session.read_version_log(n_jobs[0])
    dev.session.close()
    return RunResult(actions=per_agent[0], trace=trace, requests=records, agent_actions=per_agent,
                     device_versions=versions,
                     frame_times=_frame_times(dev) if clock == "device" else None)


def run_decoupled(policy, env, duration: int, frame_interval: Optional[float] = None, *,
                  clock: str = "virtual", agents: Optional[int] = None, frame_source=None,
                  frame_hook=None) -> RunResult:
    """fp/executor.py:583-701 (DEC) on the B200: perception free-runs on the P
    stream, publishing into a 2-slot HBM ring; each generation request (seeded
    by its start time, as in the reference) fetches the newest context and
    runs all n denoise iterations on G once a context derived from an unused
    observation exists.  The event order is the reference's (publish < start
    < finish at equal times)."""
    policy = _require_plugin(policy)
    if clock not in ("virtual", "device"):
        raise ConfigInvalid(f"unknown clock {clock!r}")
    _lib.load()
    gen = policy.generation
    p_cost = policy.perception.total_cost
    g_cost = gen.total_cost
    interval = frame_interval if frame_interval is not None else policy.sequential_cost
    envs = _agents_and_envs(policy, env, agents)
    A = len(envs)
    per_frame = int(math.ceil(interval / max(min(p_cost, g_cost), 1e-9))) + 2
    max_events = duration * per_frame + 8
    P_LANE, G_LANE = 0, 1
    dev = _Device(policy, capacity=2, lanes=2, agents=A, max_outputs=max_events, max_frames=max_events,
                  clock=clock)
    store = dev.store
    ports = [_Port(e, policy, a, frame_source) for a, e in enumerate(envs)]
    emis = _Emissions(dev, policy, A)
    trace = [_header("dec", interval, duration,
                     {"perception_cost": p_cost, "generation_cost": g_cost}, envs, clock)]
    records, emitted_rows = [], []
    n_layers = len(policy.perception.layers)
    latest = None                # (frame, version, slot, source observation id)
    used_versions = set()
    p_start, p_obs = 0.0, None
    g_free, job = 0.0, None      # job: (end, start, version, ctx frame, source obs id)
    last_used_obs, fresh_at = -1, None
    n_pub, n_gen, keys = 0, 0, 0
    order = {"publish": 0, "gen_start": 1, "gen_done": 2}
    for t in range(duration):
        if frame_hook is not None:
            frame_hook(t, dev, emis)
        dev.begin_frame(t, 4)
        now = float(t) * interval
        end = now + interval
        rec = _frame(t, now)
        rec["end"] = end
        newest = [port.boundary(t, emis.materialize) for port in ports]
        rec["superseded_actions"] = ports[0].last_superseded
        if p_obs is None:
            p_obs = newest
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
                keys += 1
                _ingest_keyed(dev, None, t, P_LANE, p_obs)
                dev.session.perceive(P_LANE, 0, n_layers)
                slot, version = store.reserve(t, p_obs[0].id)
                dev.publish(P_LANE, t, slot, version)
                n_pub += 1
                latest = (t, version, slot, p_obs[0].id)
                rec["publishes"].append(version)
                rec["perception"].append({"start": p_start, "end": when, "obs": p_obs[0].id,
                                          "version": version})
                if fresh_at is None and p_obs[0].id > last_used_obs:
                    fresh_at = when
                p_start, p_obs = when, newest
            elif what == "gen_start":
                ctx_frame, ver, slot, src = latest
                seed = int(round(when))
                keys += 1
                _ingest_keyed(dev, ("g", keys), seed, G_LANE, newest)
                dev.generate(ctx_frame, slot, n_gen, [(G_LANE, 0, gen.n_iterations)], [("g", keys)])
                n_gen += 1
                used_versions.add(ver)
                last_used_obs, fresh_at = src, None
                job = (when + g_cost, when, ver, ctx_frame, src)
                g_free = when + g_cost
                if policy.kind == ContextKind.AUTOREGRESSIVE:
                    rec["prefill_calls"] += 1
                    rec["decode_calls"] += gen.n_iterations - 1
                rec["generation_cost"] += g_cost
            else:
                fin, began, ver, ctx_frame, src = job
                land = int(math.ceil(fin / interval - 1e-12))
                emit = land - 1
                age = float(emit - ctx_frame)
                r = RequestRecord(observation_id=src, birth_frame=int(began // interval), birth_time=began,
                                  completion_frame=land, completion_time=fin, jct=fin - began)
                r.context_versions.append(ver)
                records.append(r)
                out_index = len(emis.items)
                dev.finish(G_LANE, out_index)
                k = emis.add(out_index, emit, (age,) * gen.n_iterations)
                for port in ports:
                    port.schedule(land, k, k)
                em = {"request": src, "time": fin, "emission_frame": emit, "land_frame": land,
                      "jct": r.jct, "action": None, "staleness_min": age, "staleness_mean": age,
                      "staleness_max": age, "staleness_final": age}
                rec["emissions"].append(em)
                emitted_rows.append((rec, em, r, k))
                job = None
        rec["published_total"] = n_pub
        rec["consumed_total"] = len(used_versions)
        rec["env_error"] = ports[0].seal()
        for port in ports[1:]:
            port.seal()
        dev.end_frame(t)
        trace.append(rec)
    if frame_hook is not None:
        frame_hook(duration, dev, emis)
    dev.synchronize()
    per_agent = emis.all()
    for rec_, em, r, k in emitted_rows:
        em["action"] = list(per_agent[0][k].values)
    if clock == "device":
        _apply_device_clock(dev, trace, records, emitted_rows)
    versions = dev.session.read_version_log(max(1, n_gen))
    dev.session.close()
    return RunResult(actions=per_agent[0], trace=trace, requests=records, agent_actions=per_agent,
                     device_versions=versions,
                     frame_times=_frame_times(dev) if clock == "device" else None)
