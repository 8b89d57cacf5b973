"""Horovod-style gradient aggregation with the reference API
(/root/reference/pkg/src/collectium/aggregation.py:22-176): negotiation,
greedy tensor fusion, one allreduce per fused buffer, and the mean.

B200 data path (``aggregate`` on a ``Communicator``): the whole fused step is
``cm_fused_allreduce`` — one batched pack kernel per fused buffer writes the
members straight into the IPC staging heap (no host concatenation, no extra
device copy before the reduce-scatter), then one collective kernel reduces in
the reference fold order with the mean fused in (IEEE x/p, identical to the
reference's float32(float64(s)/p)). The returned tensors are views of the
fused output buffer, as the reference returns slices of the mean
(aggregation.py:173-174).
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .collectives import DEFAULT_SWITCH_BYTES, CollectiveStats, _stats, _switch
from .comm import Communicator, VirtualGroup
from .core import DTYPES, GroupSpec, ReduceOp, Tensor
from .errors import ShapeError

TAG_NEGOTIATE = 2
DEFAULT_FUSION_THRESHOLD = 67108864                            # aggregation.py:25


@dataclass(frozen=True)
class GradientSet:
    """Ordered (name, Tensor) pairs for one iteration (aggregation.py:28-49)."""
    tensors: tuple[Tensor, ...]
    iteration: int = 0

    def __post_init__(self):
        object.__setattr__(self, "tensors", tuple(self.tensors))
        names = [t.name for t in self.tensors]
        if len(set(names)) != len(names):
            raise ShapeError("gradient names must be unique within a set")

    @property
    def names(self) -> list[str]:
        return [t.name for t in self.tensors]

    def get(self, name: str) -> Tensor:
        for t in self.tensors:
            if t.name == name:
                return t
        raise KeyError(name)


@dataclass(frozen=True)
class FusionConfig:
    threshold_bytes: int = DEFAULT_FUSION_THRESHOLD

    def __post_init__(self):
        if self.threshold_bytes <= 0:
            raise ValueError("fusion threshold must be positive")


@dataclass
class FusedBuffer:
    dtype: str
    payload: torch.Tensor
    members: list[tuple[str, int, int]] = field(default_factory=list)  # name, offset, len

    @property
    def nbytes(self) -> int:
        return int(self.payload.numel() * self.payload.element_size())


def _name_key(names: list[str]) -> int:
    h = hashlib.blake2b("\x00".join(names).encode("utf-8"), digest_size=8).digest()
    return int.from_bytes(h, "little", signed=True) >> 1


def negotiate_ready(local_ready: list[str], group: GroupSpec, transport) -> list[str]:
    """Intersection of all ranks' ready sets in lexicographic order, identical
    on every rank (aggregation.py:72-92).

    Fast path: one int64 MAX-allreduce over NVLink of (key, -key), key = a
    hash of the sorted names; equal keys on every rank mean identical ready
    sets, so the intersection is the local list. Otherwise the sets are
    gathered to rank 0 over the torch.distributed control plane and the
    intersection is broadcast, exactly as the reference does over its
    transport."""
    names = sorted(local_ready)
    if group.size == 1:
        return names
    tp: Communicator = transport
    key = _name_key(names)
    probe = torch.tensor([key, -key, len(names), -len(names)], dtype=torch.int64, device=tp.device)
    from .collectives import allreduce
    got, _ = allreduce(Tensor("__negotiate__", "int64", probe), ReduceOp.MAX, group, tp,
                       algo="rhd_rsa")
    mx = got.payload.tolist()
    if mx[0] == key and mx[1] == -key and mx[2] == len(names) and mx[3] == -len(names):
        return names
    import torch.distributed as dist
    gathered = [None] * group.size
    dist.all_gather_object(gathered, names, group=tp._group)
    common = set(gathered[0])
    for g in gathered[1:]:
        common &= set(g)
    return sorted(common)


def fuse_plan(tensors: list[Tensor], cfg: FusionConfig) -> list[list[int]]:
    """Greedy first-fit grouping of aggregation.py:95-130 (cm_fuse_plan)."""
    n = len(tensors)
    if n == 0:
        return []
    nbytes = L.i64_array([t.nbytes for t in tensors])
    dts = (C.c_int * n)(*[L.DTYPE[t.dtype] for t in tensors])
    group = (C.c_int * n)()
    ng = C.c_int()
    L.check(L.lib.cm_fuse_plan(n, nbytes, dts, int(cfg.threshold_bytes), group, C.byref(ng)))
    out: list[list[int]] = [[] for _ in range(ng.value)]
    for i in range(n):
        out[group[i]].append(i)
    return out


def _batched_copy(srcs, dsts, nbytes, device) -> None:
    with torch.cuda.device(device):
        L.check(L.lib.cm_batched_copy(len(srcs), L.ptr_array(srcs), L.ptr_array(dsts),
                                      L.i64_array(nbytes), torch.cuda.current_stream(device).cuda_stream))


def fuse(ready: list[Tensor], cfg: FusionConfig) -> list[FusedBuffer]:
    """aggregation.py:95-130; the concatenation is one batched-copy kernel
    launch per buffer (device tensors) instead of np.concatenate."""
    buffers = []
    for grp in fuse_plan(ready, cfg):
        members, off = [], 0
        ts = [ready[i] for i in grp]
        for t in ts:
            members.append((t.name, off, t.len))
            off += t.len
        dev = ts[0].payload.device
        payload = torch.empty(off, dtype=DTYPES[ts[0].dtype], device=dev)
        if dev.type == "cuda":
            esz = payload.element_size()
            _batched_copy([t.payload.data_ptr() for t in ts],
                          [payload.data_ptr() + o * esz for _, o, _ in members],
                          [t.nbytes for t in ts], dev)
        else:
            torch.cat([t.payload for t in ts], out=payload)
        buffers.append(FusedBuffer(ts[0].dtype, payload, members))
    return buffers


def unfuse(buf: FusedBuffer) -> list[Tensor]:
    """aggregation.py:133-135 (views of the fused payload)."""
    return [Tensor(name, buf.dtype, buf.payload[off:off + length])
            for name, off, length in buf.members]


def aggregate(grads: GradientSet, group: GroupSpec, transport: Communicator,
              algo: str = "auto", cfg: FusionConfig | None = None,
              switch_bytes: int | None = DEFAULT_SWITCH_BYTES,
              registry=None, handles: dict | None = None,
              stats_out: list[CollectiveStats] | None = None) -> GradientSet:
    """Negotiate, fuse, allreduce-sum and average this iteration's gradients;
    every rank returns the same mean tensors (aggregation.py:138-176)."""
    cfg = cfg or FusionConfig()
    tp = transport
    if group.size != tp.size:
        raise ShapeError(f"group size {group.size} does not match transport size {tp.size}")
    ready_names = negotiate_ready(grads.names, group, tp)
    if not ready_names:
        return GradientSet((), grads.iteration)
    ready = [grads.get(name) for name in ready_names]
    for t in ready:
        if t.dtype not in ("float32", "float64", "bfloat16"):
            raise ShapeError(f"aggregate averages floating-point gradients, got {t.dtype}")
    sw = _switch(switch_bytes, tp.size)
    plan = fuse_plan(ready, cfg)
    if registry is not None and handles is not None:
        for grp in plan:                      # aggregation.py:159-161
            for i in grp:
                registry.classify(handles[ready[i].name])
    out: dict[str, Tensor] = {}
    # a dtype change always closes a fused group, so consecutive same-dtype
    # runs can be issued as independent cm_fused_allreduce calls
    i = 0
    while i < len(ready):
        j = i
        while j < len(ready) and ready[j].dtype == ready[i].dtype:
            j += 1
        run = ready[i:j]
        dtype = run[0].dtype
        any_host = any(not t.is_cuda for t in run)
        dev = tp.device
        total = sum(t.len for t in run)
        fused = torch.empty(total, dtype=DTYPES[dtype], device=dev)
        counts = [t.len for t in run]
        st = (L.Stats * len(run))()
        ncalls = C.c_int()
        with torch.cuda.device(dev):
            L.check(L.lib.cm_fused_allreduce(
                tp._h, len(run), L.ptr_array([t.payload.data_ptr() for t in run]),
                L.i64_array(counts), L.DTYPE[dtype], fused.data_ptr(), L.ALGO[algo],
                int(cfg.threshold_bytes), sw, 1, tp._stream(), st, C.byref(ncalls)))
        if any_host:
            fused = fused.cpu()
        if tp.blocking or any_host:
            tp.synchronize()
        else:
            tp.poll()
        if stats_out is not None:
            stats_out.extend(_stats(st[k]) for k in range(ncalls.value))
        off = 0
        for t in run:
            out[t.name] = Tensor(t.name, dtype, fused[off:off + t.len])
            off += t.len
        i = j
    return GradientSet(tuple(out[name] for name in ready_names), grads.iteration)


def aggregate_group(per_rank: list[GradientSet], vg: VirtualGroup, algo: str = "auto",
                    cfg: FusionConfig | None = None,
                    switch_bytes: int | None = DEFAULT_SWITCH_BYTES,
                    stats_out: list[list[CollectiveStats]] | None = None) -> list[GradientSet]:
    """``aggregate`` for every rank of a single-GPU VirtualGroup: negotiation
    (local intersection), fusion with the batched-copy kernel, then one
    averaged allreduce launch per fused buffer."""
    from .collectives import allreduce_group
    cfg = cfg or FusionConfig()
    p = vg.size
    if len(per_rank) != p:
        raise ShapeError(f"{len(per_rank)} gradient sets for a group of {p}")
    common = set(per_rank[0].names)
    for g in per_rank[1:]:
        common &= set(g.names)
    names = sorted(common)
    outs = [dict() for _ in range(p)]
    if stats_out is not None:
        stats_out.extend([] for _ in range(p))
    ready0 = [per_rank[0].get(nm) for nm in names]
    for grp in fuse_plan(ready0, cfg):
        bufs = []
        for r in range(p):
            ts = [per_rank[r].get(names[i]) for i in grp]
            ts = [Tensor(t.name, t.dtype, t.payload.to(vg.device)) for t in ts]
            (fb,) = fuse(ts, FusionConfig(1 << 62))
            bufs.append(fb)
        res = allreduce_group([Tensor("__fused__", b.dtype, b.payload) for b in bufs],
                              ReduceOp.SUM, vg, algo=algo, switch_bytes=switch_bytes,
                              average=True)
        for r in range(p):
            mean, st = res[r]
            if stats_out is not None:
                stats_out[r].append(st)
            for name, off, ln in bufs[r].members:
                outs[r][name] = Tensor(name, mean.dtype, mean.payload[off:off + ln])
    return [GradientSet(tuple(outs[r][nm] for nm in names), per_rank[r].iteration)
            for r in range(p)]
