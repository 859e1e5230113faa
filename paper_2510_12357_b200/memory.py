"""Expert cache + transfer channel (drop-in for moesim.memory).

`HbmCache` is backed by the C++ cache core in libmobile (mobile_cache_*): LRU
order, pins, in-flight protection, speculative deferral and CapacityDeadlock
exactly as memory.py:65-181.  The same core drives the real device expert
cache (`offload.OffloadRuntime`), where the clock is logical and a "transfer"
is a cudaMemcpyAsync on the copy stream.  `TransferChannel` is the FIFO
channel of memory.py:29-44 (its state lives in a C struct the core updates).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native as N
from ._native import CapacityDeadlock  # noqa: F401  (re-export)
from .spec import ExpertId

HIT = "hit"
IN_FLIGHT = "in_flight"
ISSUED = "issued"
_STATUS = {0: HIT, 1: IN_FLIGHT, 2: ISSUED}


class TransferChannel:
    """Single FIFO channel: done = max(now, busy_until) + t_xfer."""

    def __init__(self, t_xfer: float, busy_until: float = 0.0, transfers_issued: int = 0):
        if t_xfer <= 0.0:
            raise ValueError(f"t_xfer must be positive, got {t_xfer}")
        self._c = N.mobile_channel(float(t_xfer), float(busy_until), int(transfers_issued))

    t_xfer = property(lambda self: self._c.t_xfer)
    busy_until = property(lambda self: self._c.busy_until)
    transfers_issued = property(lambda self: self._c.transfers_issued)

    def issue(self, now: float) -> float:
        start = max(now, self._c.busy_until)
        self._c.busy_until = start + self._c.t_xfer
        self._c.transfers_issued += 1
        return self._c.busy_until


@dataclass(frozen=True)
class RequestResult:
    status: str
    ready_time: float


@dataclass
class CacheStats:
    hits: int = 0
    coalesced: int = 0
    issued: int = 0
    evictions: int = 0
    deferrals: int = 0

    def total_requests(self) -> int:
        return self.hits + self.coalesced + self.issued


class HbmCache:
    """LRU cache of expert slots keyed by ExpertId (memory.py:65-181)."""

    def __init__(self, slots: int, _handle=None):
        if _handle is None:
            if slots < 1:
                raise ValueError(f"cache needs at least 1 expert slot, got {slots}")
            _handle = N.lib.mobile_cache_create(int(slots))
            if not _handle:
                raise ValueError(N.last_error())
            self._owned = True
        else:
            self._owned = False
        self._h = _handle
        self.slots = slots

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            N.lib.mobile_cache_destroy(self._h)
            self._h = None

    # ---- introspection
    def __contains__(self, expert: ExpertId) -> bool:
        return bool(N.lib.mobile_cache_contains(self._h, expert.layer, expert.expert))

    def __len__(self) -> int:
        return int(N.lib.mobile_cache_size(self._h))

    def ready_time(self, expert: ExpertId) -> float:
        r = C.c_double()
        if N.lib.mobile_cache_lookup(self._h, expert.layer, expert.expert, C.byref(r), None) != N.OK:
            raise KeyError(expert)
        return r.value

    def slot_of(self, expert: ExpertId) -> int:
        s = C.c_int()
        if N.lib.mobile_cache_lookup(self._h, expert.layer, expert.expert, None, C.byref(s)) != N.OK:
            raise KeyError(expert)
        return s.value

    def resident(self, expert: ExpertId, now: float) -> bool:
        return expert in self and self.ready_time(expert) <= now

    def entries(self) -> list[ExpertId]:
        n = len(self)
        buf = (C.c_int * (2 * max(n, 1)))()
        m = N.lib.mobile_cache_entries(self._h, buf, n)
        return [ExpertId(buf[2 * i], buf[2 * i + 1]) for i in range(m)]

    @property
    def stats(self) -> CacheStats:
        out = (C.c_longlong * 5)()
        N.lib.mobile_cache_stats(self._h, out)
        return CacheStats(*[int(v) for v in out])

    # ---- pinning
    def pin(self, expert: ExpertId) -> None:
        N.lib.mobile_cache_pin(self._h, expert.layer, expert.expert)

    def unpin(self, expert: ExpertId) -> None:
        N.lib.mobile_cache_unpin(self._h, expert.layer, expert.expert)

    def token_end(self) -> None:
        N.lib.mobile_cache_token_end(self._h)

    # ---- load path
    def request(self, expert: ExpertId, now: float, channel: TransferChannel, speculative: bool = False):
        st, ready, slot = C.c_int(), C.c_double(), C.c_int()
        rc = N.lib.mobile_cache_request(self._h, expert.layer, expert.expert, float(now), int(bool(speculative)),
                                        C.byref(channel._c), 0.0, C.byref(st), C.byref(ready), C.byref(slot))
        if rc == N.ERR_DEFERRED:
            return None
        N.check(rc, "cache request")
        return RequestResult(_STATUS[st.value], ready.value)

    def evict_lru(self, n: int, now: float | None = None) -> list[ExpertId]:
        buf = (C.c_int * (2 * max(n, 1)))()
        got = C.c_int()
        rc = N.lib.mobile_cache_evict_lru(self._h, int(n), float("inf") if now is None else float(now), buf,
                                          C.byref(got))
        N.check(rc, "evict_lru")
        return [ExpertId(buf[2 * i], buf[2 * i + 1]) for i in range(got.value)]
