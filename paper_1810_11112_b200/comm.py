"""NVLink communicators.

``Communicator`` is one rank's endpoint (one process per GPU). It replaces
the reference Transport plugin (transport/base.py:8-57): ``rank``, ``size``
and the logical counters keep their meaning, but there is no byte
send/recv — the ranks' symmetric heaps are mapped into each other's address
space with CUDA IPC and the sm_100a kernels read peer HBM over NVSwitch.

``VirtualGroup`` drives ``size`` ranks on ONE GPU (one cooperative kernel
holds every rank's CTAs); it is the single-GPU analogue of the reference's
in-process SimNetwork and runs the very same kernels and flag protocol.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib as L
from .core import DTYPES
from .errors import ConfigError, InvalidGroupError

DEFAULT_STAGING_BYTES = int(os.environ.get("CM_STAGING_BYTES", 1 << 30))
DEFAULT_POOL_BYTES = int(os.environ.get("CM_POOL_BYTES", 1 << 30))


_raw_stream = torch._C._cuda_getCurrentRawStream


class _Base:
    _h: C.c_void_p | None = None
    _hv: int | None = None            # the handle as a plain int (fast-call path)

    def _stream(self) -> int:
        return _raw_stream(self.device.index)

    # -- tuning / policy ------------------------------------------------------
    def set_param(self, key: str, value: int) -> None:
        L.check(L.lib.cm_comm_set_param(self._h, key.encode(), int(value)))
        self.__dict__.setdefault("_knobs", {})[key] = int(value)     # read back by the façade

    def get_param(self, key: str) -> int:
        v = C.c_int64()
        L.check(L.lib.cm_comm_get_param(self._h, key.encode(), C.byref(v)))
        return int(v.value)

    def set_timeout(self, seconds: float) -> None:
        L.check(L.lib.cm_comm_set_timeout(self._h, float(seconds)))

    def set_policy(self, policy: str) -> None:
        """Pointer-cache policy used to classify send/recv buffers on every
        call: "no_cache" (driver query each call — the paper's baseline),
        "lazy_cache" (query once per address), "intercept_cache" (only
        registered/comm-allocated buffers; zero queries)."""
        L.check(L.lib.cm_comm_set_policy(self._h, L.POLICY[policy]))

    def registry_stats(self) -> dict:
        reg = C.c_void_p()
        L.check(L.lib.cm_comm_registry(self._h, C.byref(reg)))
        st = L.RegStats()
        L.check(L.lib.cm_registry_stats(reg, C.byref(st)))
        ns = C.c_int64()
        L.check(L.lib.cm_registry_query_time_ns(reg, C.byref(ns)))
        return {"driver_queries": st.driver_queries, "cache_hits": st.cache_hits,
                "inserts": st.inserts, "invalidations": st.invalidations,
                "query_time_ns": int(ns.value)}

    def register(self, tensor: torch.Tensor, kind: str | None = None) -> None:
        """Tell the intercept cache about an externally allocated buffer."""
        reg = C.c_void_p()
        L.check(L.lib.cm_comm_registry(self._h, C.byref(reg)))
        k = kind or ("device" if tensor.is_cuda else "host")
        L.check(L.lib.cm_registry_register(reg, tensor.data_ptr(),
                                           tensor.numel() * tensor.element_size(), L.KIND[k]))

    # -- synchronisation / counters ------------------------------------------
    def synchronize(self) -> None:
        """Wait for this rank's stream; raise any device-side error
        (ShapeError for mismatched peers, TransportError on timeout)."""
        if L.fast is not None:
            st = L.fast.sync(self._hv, self._stream())
        else:
            st = L.lib.cm_comm_sync(self._h, self._stream())
        if st:
            L.check(st)

    def poll(self) -> None:
        st = L.fast.poll(self._hv) if L.fast is not None else L.lib.cm_comm_poll(self._h)
        if st:
            L.check(st)

    def _counters(self):
        m, b, nv, c = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        L.check(L.lib.cm_comm_counters(self._h, C.byref(m), C.byref(b), C.byref(nv), C.byref(c)))
        return int(m.value), int(b.value), int(nv.value), int(c.value)

    @property
    def messages_sent(self) -> int:
        return self._counters()[0]

    @property
    def bytes_sent(self) -> int:
        return self._counters()[1]

    @property
    def nvlink_bytes_in(self) -> int:
        return self._counters()[2]

    @property
    def calls(self) -> int:
        return self._counters()[3]

    @property
    def launches(self) -> int:
        v = C.c_int64()
        L.check(L.lib.cm_comm_launches(self._h, C.byref(v)))
        return int(v.value)

    def close(self) -> None:
        if self._h is not None:
            L.lib.cm_comm_destroy(self._h)
            self._h = None
            self._hv = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class Communicator(_Base):
    """One rank of an NVLink group (one process per GPU).

    Bootstrap (the host control plane) runs over an initialised
    ``torch.distributed`` process group (gloo or nccl): every rank creates its
    IPC heap, the 64-byte handles are all-gathered, and each rank maps every
    peer's heap once. ``blocking=True`` mirrors the reference's blocking
    collectives: each call waits for its kernel and raises device-side errors.
    """

    def __init__(self, rank: int | None = None, size: int | None = None,
                 device: int | torch.device | None = None, group=None,
                 staging_bytes: int = DEFAULT_STAGING_BYTES,
                 pool_bytes: int = DEFAULT_POOL_BYTES,
                 policy: str = "lazy_cache", blocking: bool = True,
                 timeout_s: float | None = None):
        import torch.distributed as dist
        if rank is None or size is None:
            if not dist.is_initialized():
                if (size or 1) == 1:
                    rank, size = 0, 1
                else:
                    raise InvalidGroupError("torch.distributed is not initialised")
            else:
                rank = dist.get_rank(group)
                size = dist.get_world_size(group)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.rank, self.size = int(rank), int(size)
        self.blocking = blocking
        self._group = group
        h = C.c_void_p()
        torch.cuda.set_device(self.device)
        L.check(L.lib.cm_comm_create(self.rank, self.size, self.device.index, int(staging_bytes),
                                     int(pool_bytes), C.byref(h)))
        self._h, self._hv = h, h.value
        if self.size > 1:
            buf = (C.c_char * L.IPC_HANDLE_BYTES)()
            L.check(L.lib.cm_comm_ipc_handle(self._h, buf))
            mine = bytes(buf)
            handles = [None] * self.size
            dist.all_gather_object(handles, mine, group=group)
            allh = b"".join(handles)
            L.check(L.lib.cm_comm_connect(self._h, allh))
            dist.barrier(group=group)
        self.set_policy(policy)
        if timeout_s is not None:
            self.set_timeout(timeout_s)
        from .tuning import ll2_max_for, oneshot_max_for
        osm = oneshot_max_for(self.size)
        if osm:
            self.set_param("oneshot_max_bytes", osm)
            self.set_param("ll_max_bytes", osm)
        l2m = ll2_max_for(self.size)
        if l2m:
            self.set_param("ll2_max_bytes", l2m)
        self._sym: dict[int, int] = {}

    # -- symmetric allocation (zero-copy collectives) -------------------------
    def empty(self, numel: int, dtype: str | torch.dtype = "float32") -> torch.Tensor:
        """Collective: allocate a tensor in the symmetric IPC pool. Every rank
        must make the same sequence of calls. Collectives whose send buffer
        lives here are read by peers in place (no staging copy)."""
        tdt = DTYPES[dtype] if isinstance(dtype, str) else dtype
        nbytes = int(numel) * torch.empty((), dtype=tdt).element_size()
        ptr = C.c_void_p()
        L.check(L.lib.cm_comm_alloc(self._h, max(nbytes, 1), C.byref(ptr)))
        t = _tensor_from_ptr(ptr.value, int(numel), tdt, self.device)
        self._sym[ptr.value] = nbytes
        return t

    def free(self, t: torch.Tensor) -> None:
        p = t.data_ptr()
        if p not in self._sym:
            raise ConfigError("not a symmetric allocation of this communicator")
        del self._sym[p]
        L.check(L.lib.cm_comm_free(self._h, p))

    def register_buffers(self, tensors, tolerant: bool = False) -> list[int] | None:
        """Collective: register device tensors for zero-copy collectives (every
        rank passes its own tensors, same count and order). Each rank exports
        the CUDA-IPC handle of the allocation holding the tensor plus the
        offset; handles are all-gathered on the control plane and every peer
        allocation is opened once (cached). Afterwards, collectives whose send
        buffer lies inside a registered tensor are read by peers in place. The
        tensors must stay alive until ``deregister_buffers``.

        ``tolerant``: an allocation that cannot be exported (e.g. a virtual-
        memory segment) does not raise; every rank learns it in the same
        all-gather and the call returns None everywhere (nothing registered)."""
        import torch.distributed as dist
        mine = []
        for t in tensors:
            h = (C.c_char * L.IPC_HANDLE_BYTES)()
            off = C.c_int64()
            st = L.lib.cm_comm_export(self._h, t.data_ptr(), t.numel() * t.element_size(), h, C.byref(off))
            if st and tolerant:
                mine = None
                break
            L.check(st)
            mine.append((bytes(h), int(off.value)))
        gathered = [None] * self.size
        if self.size > 1:
            dist.all_gather_object(gathered, mine, group=self._group)
        else:
            gathered = [mine]
        if any(g is None for g in gathered):
            return None
        ids = []
        for i, t in enumerate(tensors):
            handles = b"".join(gathered[q][i][0] for q in range(self.size))
            offs = L.i64_array([gathered[q][i][1] for q in range(self.size)])
            rid = C.c_int64()
            L.check(L.lib.cm_comm_register(self._h, t.data_ptr(), t.numel() * t.element_size(),
                                           handles, offs, C.byref(rid)))
            ids.append(int(rid.value))
        return ids

    def deregister_buffers(self, tensors) -> None:
        for t in tensors:
            L.check(L.lib.cm_comm_deregister(self._h, t.data_ptr()))

    def barrier(self) -> None:
        import torch.distributed as dist
        if self.size > 1:
            dist.barrier(group=self._group)

    def close(self) -> None:
        if self._h is not None:
            try:
                torch.cuda.synchronize(self.device)
                self.barrier()
            except Exception:
                pass
        super().close()


class VirtualGroup(_Base):
    """``size`` ranks emulated on one GPU: each collective is ONE cooperative
    launch holding every rank's CTAs (flags, staging and fold order exactly as
    on a real NVLink group)."""

    def __init__(self, size: int, device: int | None = None, staging_bytes: int = 64 << 20,
                 timeout_s: float | None = 5.0):
        if size < 1:
            raise InvalidGroupError(f"group size must be >= 1, got {size}")
        dev = torch.cuda.current_device() if device is None else device
        self.device = torch.device("cuda", dev)
        self.size = int(size)
        self.rank = 0
        h = C.c_void_p()
        torch.cuda.set_device(self.device)
        L.check(L.lib.cm_comm_create_virtual(self.size, dev, int(staging_bytes), C.byref(h)))
        self._h, self._hv = h, h.value
        if timeout_s is not None:
            self.set_timeout(timeout_s)

    def register_buffers(self, per_rank_tensors) -> list[int]:
        """Register buffers for zero-copy aggregation: ``per_rank_tensors[i]``
        lists every virtual rank's i-th tensor (device memory); returns one id
        per i, the same id for all ranks (as ``Communicator.register_buffers``
        returns on every rank of a real group)."""
        ids = []
        for ts in per_rank_tensors:
            if len(ts) != self.size:
                raise InvalidGroupError(f"{len(ts)} tensors for a group of {self.size}")
            rid = C.c_int64()
            L.check(L.lib.cm_comm_register_v(self._h, L.ptr_array([t.data_ptr() for t in ts]),
                                             ts[0].numel() * ts[0].element_size(), C.byref(rid)))
            ids.append(int(rid.value))
        return ids


def _tensor_from_ptr(ptr: int, numel: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Wrap comm-owned device memory as a torch tensor (no copy, not owned)."""
    elem = torch.empty((), dtype=dtype).element_size()
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.bfloat16: "<u2",
               torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1"}[dtype]

    class _Holder:
        __cuda_array_interface__ = {"shape": (int(numel),), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3, "strides": None}

    with torch.cuda.device(device):
        t = torch.as_tensor(_Holder(), device=device)
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    assert t.data_ptr() == ptr and t.numel() * elem == numel * elem
    return t
