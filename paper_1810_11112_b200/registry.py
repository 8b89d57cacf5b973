"""Pointer cache (PAPER §V-B) with the reference API
(/root/reference/pkg/src/collectium/registry.py:24-151), backed by the C++
cache in csrc/ptrcache.cpp — the same object the communicator consults on
every collective call.

``backend="sim"`` (default) reproduces the reference model exactly (fake
addresses, lowest-freed-address reuse, counted simulated driver queries);
``backend="cuda"`` allocates real device / pinned-host memory and the driver
query is one ``cuPointerGetAttributes`` call (memory type, device ordinal,
allocation range, buffer id; its measured wall time is reported by
``query_delay_seconds``); the intercept cache answers interior pointers of
registered ranges (torch sub-allocations).
"""

from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass

from . import _lib as L
from .errors import InvalidHandleError

DEFAULT_QUERY_DELAY_NS = 1000                                  # registry.py:24


class BufferKind(enum.Enum):
    HOST = "host"
    DEVICE = "device"


class Policy(enum.Enum):
    NO_CACHE = "no_cache"
    LAZY_CACHE = "lazy_cache"
    INTERCEPT_CACHE = "intercept_cache"


@dataclass(frozen=True)
class BufferHandle:
    address: int
    size: int


@dataclass
class RegistryStats:
    driver_queries: int = 0
    cache_hits: int = 0
    inserts: int = 0
    invalidations: int = 0


class BufferRegistry:
    """Handle -> kind map with a pluggable classification policy; every
    operation is serialised by the C++ registry mutex."""

    def __init__(self, policy: Policy | str = Policy.NO_CACHE,
                 query_delay_ns: int = DEFAULT_QUERY_DELAY_NS, backend: str = "sim"):
        self.policy = Policy(policy)
        self.query_delay_ns = query_delay_ns
        if backend not in ("sim", "cuda"):
            raise ValueError(f"unknown backend {backend!r}")
        self.backend = backend
        h = C.c_void_p()
        L.check(L.lib.cm_registry_create(L.POLICY[self.policy.value], int(query_delay_ns),
                                         1 if backend == "sim" else 0, C.byref(h)))
        self._h = h
        self._live: dict[int, BufferHandle] = {}

    def __del__(self):  # pragma: no cover
        h = getattr(self, "_h", None)
        try:
            if h is not None:
                L.lib.cm_registry_destroy(h)
        except Exception:
            pass
        self._h = None

    def alloc(self, kind: BufferKind, size: int) -> BufferHandle:
        if size <= 0:
            raise ValueError(f"allocation size must be positive, got {size}")
        a = C.c_uint64()
        L.check(L.lib.cm_registry_alloc(self._h, L.KIND[BufferKind(kind).value], int(size),
                                        C.byref(a)))
        h = BufferHandle(int(a.value), int(size))
        self._live[h.address] = h
        return h

    def free(self, handle: BufferHandle) -> None:
        # registry.py:90-95: a stale handle object is a double free even when
        # its address has been handed out again
        if self._live.get(handle.address) is not handle:
            raise InvalidHandleError(
                f"free of dead or unknown handle at address {handle.address:#x}")
        L.check(L.lib.cm_registry_free(self._h, handle.address))
        del self._live[handle.address]

    def classify(self, handle: BufferHandle | int) -> BufferKind:
        addr = handle.address if isinstance(handle, BufferHandle) else int(handle)
        k = C.c_int()
        L.check(L.lib.cm_registry_classify(self._h, addr, C.byref(k)))
        return BufferKind(L.KIND_NAME[k.value])

    def info(self, handle: BufferHandle | int) -> dict:
        """Classify through the policy and return what the cache entry holds:
        kind, device ordinal, allocation range and buffer id (real backend;
        the sim backend and the intercept cache know the kind / range only)."""
        addr = handle.address if isinstance(handle, BufferHandle) else int(handle)
        bi = L.BufferInfo()
        L.check(L.lib.cm_registry_info(self._h, addr, C.byref(bi)))
        return {"kind": BufferKind(L.KIND_NAME[bi.kind]), "device": int(bi.device),
                "range_start": int(bi.range_start), "range_size": int(bi.range_size),
                "buffer_id": int(bi.buffer_id)}

    def ground_truth(self, handle: BufferHandle | int) -> BufferKind:
        addr = handle.address if isinstance(handle, BufferHandle) else int(handle)
        k = C.c_int()
        L.check(L.lib.cm_registry_ground_truth(self._h, addr, C.byref(k)))
        return BufferKind(L.KIND_NAME[k.value])

    def register(self, address: int, size: int, kind: BufferKind) -> None:
        L.check(L.lib.cm_registry_register(self._h, int(address), int(size),
                                           L.KIND[BufferKind(kind).value]))

    def unregister(self, address: int) -> None:
        L.check(L.lib.cm_registry_unregister(self._h, int(address)))

    @property
    def stats(self) -> RegistryStats:
        st = L.RegStats()
        L.check(L.lib.cm_registry_stats(self._h, C.byref(st)))
        return RegistryStats(int(st.driver_queries), int(st.cache_hits), int(st.inserts),
                             int(st.invalidations))

    def query_delay_seconds(self) -> float:
        """registry.py:143-145 (sim: queries x delay; cuda: measured)."""
        ns = C.c_int64()
        L.check(L.lib.cm_registry_query_time_ns(self._h, C.byref(ns)))
        return ns.value * 1e-9

    def stats_dict(self) -> dict:
        s = self.stats
        return {"policy": self.policy.value, "driver_queries": s.driver_queries,
                "cache_hits": s.cache_hits, "inserts": s.inserts,
                "invalidations": s.invalidations}

    def stats_json(self) -> str:
        buf = C.create_string_buffer(512)
        L.check(L.lib.cm_registry_stats_json(self._h, buf, 512))
        return json.dumps(json.loads(buf.value.decode()))
