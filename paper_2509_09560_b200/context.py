"""The public context and its versioned ring, resident in HBM.

Replaces the reference's ContextStore / PublicContext (fp/context.py:23-175)
on the hot path.  The payload of every slot lives in device memory and is
written by producer kernels (perception epilogues); what crosses the host is
only a handle `(slot, version, frame)`.

Device layout (one ring per lock-stepped agent group):
  payload : [agents, K, slot_elems]   (fp64 for the toy policy, fp32 for DP)
  meta    : int64 [K, 2] = {frame, version}, the version released last
  state   : int64 [4]    = {version, last frame, publish count, error flag}

The host keeps a mirror of the metadata (versions, slot frames) because the
scheduler's decisions -- NotYetPublished, the newest-context fallback,
DeadlockDetected -- are host decisions in the reference too
(fp/executor.py:302-316).  Consumer kernels resolve the slot again on the
device (auras_ring_fetch: acquire-load of the version word) and log the
version they actually read, so tests can assert that host schedule and
device consumption agree.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Optional

import numpy as np

from . import _lib
from .errors import KindMismatch, NotYetPublished, OffsetOutOfRange, StaleWrite


class ContextKind(str, Enum):
    AUTOREGRESSIVE = "autoregressive"
    CONDITIONING = "conditioning"


def _checksum(vision, language, action_tokens, conditioning,
              source_observation_id: int, produced_frame: int) -> int:
    """fp/context.py:28-36."""
    crc = 0
    for arr in (vision, language, conditioning):
        if arr is not None:
            crc = zlib.crc32(np.ascontiguousarray(arr, dtype=np.float64).tobytes(), crc)
    crc = zlib.crc32(repr(tuple(action_tokens)).encode(), crc)
    crc = zlib.crc32(f"{source_observation_id}:{produced_frame}".encode(), crc)
    return crc


@dataclass(frozen=True)
class PublicContext:
    """The public context (H_o of Eq. 2; fp/context.py:39-88): a conditioning
    vector for refinement policies, or [X_V; X_L; X_A] for token policies.

    `conditioning` / the token arrays are host copies when one exists
    (standalone use, the causal transformer's merged prefill); the engine's
    contexts are device-resident and carry only their ring slot."""

    kind: ContextKind
    source_observation_id: int
    produced_frame: int
    vision_tokens: Optional[np.ndarray] = None
    language_tokens: Optional[np.ndarray] = None
    action_tokens: tuple = ()
    conditioning: Optional[np.ndarray] = None
    slot: int = -1
    checksum: int = field(default=-1)

    def __post_init__(self):
        if self.kind == ContextKind.AUTOREGRESSIVE:
            if self.vision_tokens is None or self.language_tokens is None:
                raise ValueError("autoregressive context requires vision and language tokens")
            if self.conditioning is not None:
                raise ValueError("autoregressive context must not carry a conditioning vector")
            object.__setattr__(self, "vision_tokens", np.asarray(self.vision_tokens, dtype=np.float64))
            object.__setattr__(self, "language_tokens", np.asarray(self.language_tokens, dtype=np.float64))
        elif self.kind == ContextKind.CONDITIONING:
            if self.vision_tokens is not None or self.language_tokens is not None or self.action_tokens:
                raise ValueError("conditioning context must not carry token fields")
            if self.conditioning is not None:
                object.__setattr__(self, "conditioning",
                                   np.asarray(self.conditioning, dtype=np.float64))
        else:
            raise ValueError(f"unknown context kind: {self.kind!r}")
        object.__setattr__(self, "action_tokens", tuple(int(t) for t in self.action_tokens))
        object.__setattr__(self, "checksum", self._compute_checksum())

    def _compute_checksum(self) -> int:
        return _checksum(self.vision_tokens, self.language_tokens, self.action_tokens,
                         self.conditioning, self.source_observation_id, self.produced_frame)

    def verify_checksum(self) -> bool:
        return self.checksum == self._compute_checksum()

    def with_action_tokens(self, tokens) -> "PublicContext":
        if self.kind != ContextKind.AUTOREGRESSIVE:
            raise KindMismatch("action tokens only exist on autoregressive contexts")
        return replace(self, action_tokens=tuple(tokens))

    def with_produced_frame(self, frame: int) -> "PublicContext":
        return replace(self, produced_frame=frame)


class ContextStore:
    """Ring of K versioned slots in HBM, one writer stream, many reader kernels."""

    def __init__(self, capacity: int = 2, slot_elems: int = 2, agents: int = 1,
                 dtype=None, device=None):
        import torch
        if capacity < 2:
            raise ValueError("store capacity must be at least 2")
        _lib.load()
        self.capacity = capacity
        self.agents = agents
        self.slot_elems = slot_elems
        dtype = torch.float64 if dtype is None else dtype
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.payload = torch.zeros(agents, capacity, slot_elems, dtype=dtype, device=dev)
        self.meta = torch.full((capacity, 2), -1, dtype=torch.int64, device=dev)
        self.state = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device=dev)
        # host mirror
        self._version = 0
        self._last_frame: Optional[int] = None
        self._publish_count = 0
        self._slot_frame = [None] * capacity
        self._slot_version = [0] * capacity
        self._slot_obs = [None] * capacity
        self._slot_host = [None] * capacity     # host copies of token-policy contexts

    # -- properties (fp/context.py:117-127)
    @property
    def published_version(self) -> int:
        return self._version

    @property
    def publish_count(self) -> int:
        return self._publish_count

    @property
    def last_frame(self) -> Optional[int]:
        return self._last_frame

    @property
    def slot_bytes(self) -> int:
        return self.slot_elems * self.payload.element_size()

    # -- engine-level operations (payload written by kernels)
    def slot_of(self, frame: int) -> int:
        return frame % self.capacity

    def reserve(self, frame: int, source_observation_id: Optional[int] = None):
        """Host half of publish: validate, bump the mirror, return (slot, version).
        The device half (payload kernels + auras_ring_commit) follows on the
        writer stream."""
        if self._last_frame is not None and frame < self._last_frame:
            raise StaleWrite(f"publish for frame {frame} after frame {self._last_frame}")
        self._version += 1
        self._publish_count += 1
        slot = self.slot_of(frame)
        self._slot_frame[slot] = frame
        self._slot_version[slot] = self._version
        self._slot_obs[slot] = frame if source_observation_id is None else source_observation_id
        self._slot_host[slot] = None
        self._last_frame = frame
        return slot, self._version

    def commit(self, frame: int, version: int, stream, system_scope: bool = False) -> None:
        """Release the slot's version.  `system_scope`: the writer runs on another
        GPU (disaggregated perception), so the release is st.release.sys."""
        lib = _lib.load()
        fn = lib.auras_ring_commit_sys if system_scope else lib.auras_ring_commit
        _lib.check(fn(self.meta.data_ptr(), self.state.data_ptr(), self.capacity,
                      frame, version, stream.cuda_stream), "ring_commit")

    def resolve(self, frame: int, offset: int = 0):
        """Host half of fetch_entry: (version, context frame, slot)."""
        if offset > 0 or -offset >= self.capacity:
            raise OffsetOutOfRange(f"offset {offset} outside (-{self.capacity}, 0]")
        target = frame + offset
        slot = self.slot_of(target)
        if self._slot_frame[slot] != target:
            raise NotYetPublished(f"no context published for frame {target}")
        return self._slot_version[slot], target, slot

    def resolve_latest(self):
        if self._last_frame is None:
            raise NotYetPublished("nothing published yet")
        slot = self.slot_of(self._last_frame)
        return self._slot_version[slot], self._last_frame, slot

    def device_fetch(self, target: int, out, version_log, log_index: int, stream) -> None:
        """Device half of fetch: resolve slot/version in-kernel into `out`."""
        lib = _lib.load()
        _lib.check(lib.auras_ring_fetch(self.meta.data_ptr(), self.state.data_ptr(), self.capacity,
                                        target, out.data_ptr(),
                                        0 if version_log is None else version_log.data_ptr(),
                                        log_index, stream.cuda_stream), "ring_fetch")

    # -- reference-compatible API (fp/context.py:129-164)
    def publish(self, ctx: PublicContext, frame: int) -> int:
        """fp/context.py:129-143.  A token-policy context carries its
        displacement (vision row 0) in the device slot, which is all the
        scripted token kernels read; the full [X_V; X_L; X_A] stays as a host
        copy for fetches."""
        import torch
        if ctx.kind == ContextKind.AUTOREGRESSIVE:
            vec = np.asarray(ctx.vision_tokens, dtype=np.float64)[0, :2].ravel()
        elif ctx.conditioning is None:
            raise ValueError("publish() of a host context needs its conditioning vector")
        else:
            vec = np.asarray(ctx.conditioning, dtype=np.float64).ravel()
        if vec.size > self.slot_elems:
            raise ValueError(f"context of {vec.size} elements exceeds slot of {self.slot_elems}")
        slot, version = self.reserve(frame, ctx.source_observation_id)
        stream = torch.cuda.current_stream()
        src = torch.from_numpy(vec).to(self.payload.dtype).pin_memory()
        dst = self.payload[0, slot, : vec.size]
        dst.copy_(src, non_blocking=True)
        self.commit(frame, version, stream)
        if ctx.kind == ContextKind.AUTOREGRESSIVE:
            self._slot_host[slot] = ctx
        return version

    def _host_context(self, slot: int, frame: int) -> PublicContext:
        host = self._slot_host[slot]
        if host is not None:                 # the store stamps the publishing frame
            return replace(host, produced_frame=frame, slot=slot)
        vals = self.payload[0, slot].double().cpu().numpy()
        return PublicContext(kind=ContextKind.CONDITIONING,
                             source_observation_id=self._slot_obs[slot], produced_frame=frame,
                             conditioning=vals, slot=slot)

    def fetch_entry(self, frame: int, offset: int = 0):
        version, target, slot = self.resolve(frame, offset)
        return version, self._host_context(slot, target)

    def fetch(self, frame: int, offset: int = 0) -> PublicContext:
        return self.fetch_entry(frame, offset)[1]

    def latest_entry(self):
        version, frame, slot = self.resolve_latest()
        return frame, version, self._host_context(slot, frame)

    def reserve_token_update(self, frame: int):
        """Host half of update_action_tokens (fp/context.py:166-175): the newest
        context, with the new action-token prefix, re-published as `frame`'s
        context under a new version.  Returns (source slot, slot, version); the
        device half copies the payload and releases the version.  The token
        prefix itself lives in the requests' lanes: the scripted token policy
        reads each request's own prefix (fp/policy.py:226-228), so only the
        version and the context's frame stamp change here."""
        if self._last_frame is None:
            raise NotYetPublished("nothing published yet")
        src = self.slot_of(self._last_frame)
        obs = self._slot_obs[src]
        slot, version = self.reserve(frame, obs)
        return src, slot, version

    def update_action_tokens(self, frame: int, tokens) -> int:
        """fp/context.py:166-175: the latest context with `tokens` as its
        action tokens, re-published as `frame`'s context under a new version
        (device copy + release on the current stream)."""
        import torch
        if self._last_frame is None:
            raise NotYetPublished("nothing published yet")
        host = self._slot_host[self.slot_of(self._last_frame)]
        if host is None:
            raise KindMismatch("latest context is not autoregressive")
        src, slot, version = self.reserve_token_update(frame)
        stream = torch.cuda.current_stream()
        _lib.check(_lib.load().auras_ring_copy_slot(self.payload.data_ptr(), self.slot_elems, src, slot,
                                                    stream.cuda_stream), "ring_copy_slot")
        self.commit(frame, version, stream)
        self._slot_host[slot] = host.with_action_tokens(tokens)
        return version

    def device_state(self):
        """(version, last frame, publish count, error flag) as seen by the device."""
        return tuple(int(v) for v in self.state.cpu().tolist())
