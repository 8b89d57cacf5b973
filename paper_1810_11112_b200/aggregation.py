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

import contextlib
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
        idx = self.__dict__.get("_index")
        if idx is None:
            idx = {t.name: i for i, t in enumerate(self.tensors)}
            object.__setattr__(self, "_index", idx)
        return self.tensors[idx[name]]


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

    Fast path: ``cm_agree`` — one int64 MAX allreduce over NVLink of
    (key, count, -key, -count), key = a hash of the sorted names; equal maxima
    on every rank mean identical ready sets, so the intersection is the local
    list. Otherwise the sets are gathered over the torch.distributed control
    plane and intersected exactly as the reference does at rank 0."""
    names = sorted(local_ready)
    if group.size == 1:
        return names
    if _sets_agree(transport, _name_key(names), len(names)):
        return names
    return _negotiate_gather(names, group, transport)


def _negotiate_gather(names: list[str], group: GroupSpec, tp) -> list[str]:
    import torch.distributed as dist
    gathered = [None] * group.size
    dist.all_gather_object(gathered, list(names), group=tp._group)
    common = set(gathered[0])
    for g in gathered[1:]:
        common &= set(g)
    return sorted(common)


def _sets_agree(tp: Communicator, key: int, count: int) -> bool:
    vals = (C.c_int64 * 4)(key, count, -key, -count)
    mx = (C.c_int64 * 4)()
    with torch.cuda.device(tp.device):
        L.check(L.lib.cm_agree(tp._h, vals, 4, mx, tp._stream()))
    return list(mx) == [key, count, -key, -count]


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
    launch per buffer instead of np.concatenate. CUDA-aware semantics: the
    fused buffer lives on the GPU (where its allreduce runs) even when the
    members are host tensors — pinned members are read by the kernel, pageable
    ones are moved by the copy engines; nothing is concatenated on the CPU."""
    buffers = []
    for grp in fuse_plan(ready, cfg):
        members, off = [], 0
        ts = [ready[i] for i in grp]
        for t in ts:
            members.append((t.name, off, t.len))
            off += t.len
        dev = next((t.payload.device for t in ts if t.is_cuda), None)
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        payload = torch.empty(off, dtype=DTYPES[ts[0].dtype], device=dev)
        esz = payload.element_size()
        _batched_copy([t.payload.data_ptr() for t in ts],
                      [payload.data_ptr() + o * esz for _, o, _ in members],
                      [t.nbytes for t in ts], dev)
        buffers.append(FusedBuffer(ts[0].dtype, payload, members))
    return buffers


def unfuse(buf: FusedBuffer) -> list[Tensor]:
    """aggregation.py:133-135 (views of the fused payload)."""
    return [Tensor(name, buf.dtype, buf.payload[off:off + length])
            for name, off, length in buf.members]


class _Plan:
    """Per-(GradientSet, negotiated names, config) launch plan: member order,
    same-dtype runs with their ctypes pointer/count arrays, and split sizes.
    GradientSet is immutable, so the plan is cached on it."""

    def __init__(self, grads: GradientSet, names: list[str], regmap: dict | None = None):
        self.names = names
        ready = [grads.get(nm) for nm in names]
        self.runs = []
        i = 0
        while i < len(ready):
            j = i
            while j < len(ready) and ready[j].dtype == ready[i].dtype:
                j += 1
            run = ready[i:j]
            for t in run:
                if t.dtype not in ("float32", "float64", "bfloat16"):
                    raise ShapeError(f"aggregate averages floating-point gradients, got {t.dtype}")
            counts = [t.len for t in run]
            reg = None
            if regmap is not None and all(t.name in regmap for t in run):
                reg = L.i64_array([regmap[t.name] for t in run])
            self.runs.append(dict(
                reg=reg,
                dtype=run[0].dtype, names=[t.name for t in run], counts=counts,
                total=sum(counts), any_host=any(not t.is_cuda for t in run),
                ptrs=L.ptr_array([t.payload.data_ptr() for t in run]),
                counts_c=L.i64_array(counts), n=len(run),
                stats=(L.Stats * len(run))()))
            r = self.runs[-1]       # plain addresses for the fast-call path
            r["addr"] = (C.addressof(r["ptrs"]), C.addressof(r["counts_c"]),
                         C.addressof(reg) if reg is not None else 0, C.addressof(r["stats"]))
            i = j
        self.ready = ready


def aggregate(grads: GradientSet, group: GroupSpec, transport: Communicator,
              algo: str = "auto", cfg: FusionConfig | None = None,
              switch_bytes: int | None = DEFAULT_SWITCH_BYTES,
              registry=None, handles: dict | None = None,
              stats_out: list[CollectiveStats] | None = None,
              out: GradientSet | None = None) -> GradientSet:
    """Negotiate, fuse, allreduce-sum and average this iteration's gradients;
    every rank returns the same mean tensors (aggregation.py:138-176).

    Negotiation is folded into the first fused call: every rank passes a hash
    of its sorted ready names and ``cm_fused_allreduce_agreed`` checks them
    with one NVLink MAX-allreduce before launching, in the same C call (no
    Python between the check and the launches). If the sets differ, the
    intersection is negotiated over the control plane as in the reference.

    ``out``: a GradientSet previously returned by ``aggregate`` for the same
    schema; its fused buffers are reused (stream-ordered overwrite, like
    torch ``out=``) instead of allocating new ones — the persistent-bucket
    mode of a training loop."""
    cfg = cfg or FusionConfig()
    tp = transport
    if group.size != tp.size:
        raise ShapeError(f"group size {group.size} does not match transport size {tp.size}")
    if algo not in L.ALGO:
        from .errors import ConfigError
        raise ConfigError(f"unknown algorithm {algo!r}")
    local = grads.__dict__.get("_sorted_names")
    if local is None:
        local = sorted(grads.names)
        object.__setattr__(grads, "_sorted_names", local)
        object.__setattr__(grads, "_name_key", _name_key(local))
    sw = _switch(switch_bytes, tp.size)
    explicit = grads.__dict__.get("_reg_ids")
    if tp.size == 1:
        return _aggregate_names(grads, local, tp, algo, cfg, sw, registry, handles, stats_out, out, None, explicit)
    if not local:               # nothing to fuse: plain agree + gather
        names = negotiate_ready([], group, tp)
        return _aggregate_names(grads, names, tp, algo, cfg, sw, registry, handles, stats_out, out, None, explicit)
    auto = None if explicit is not None else _auto_members(grads, local, tp)
    flags = 0 if auto is None else auto[0]
    agree = (C.c_int64 * 2)(grads.__dict__["_name_key"], len(local) | flags)
    regmap = explicit if explicit is not None else (auto[1]["ids"] if flags & _AUTO_READY else None)
    res = _aggregate_names(grads, local, tp, algo, cfg, sw, registry, handles, stats_out, out, agree, regmap)
    if res is None:             # ready sets (or member-registration states) differ across ranks
        names = _negotiate_gather(local, group, tp)
        if auto is not None and names == local:
            _auto_reset(tp, auto[1])        # the member-registration states differed: start over
        # no gathered members here: every rank packs (the modes must match)
        res = _aggregate_names(grads, names, tp, algo, cfg, sw, registry, handles, stats_out, out, None,
                               explicit)
    elif auto is not None and flags & _AUTO_ON:
        if flags & _AUTO_READY:
            auto[1]["gathered_calls"] = auto[1].get("gathered_calls", 0) + 1
        _auto_after_call(grads, local, tp, auto[1])
    return res


# Automatic member registration (the pointer cache applied to aggregate's
# fused members): after the second aggregate() of the same name set whose
# ready-set agreement passed with every rank offering it, every rank
# registers its member tensors collectively (as register_gradients does);
# from then on a rank whose members are still the registered tensors (same
# addresses, same allocation ids) offers the gathered path, and the first
# fused launch's agreement checks that every rank does — otherwise all ranks
# skip and repeat the step with packed members, and every rank drops the
# registration and counts agreed calls from zero again, so members that moved
# for good (new allocations every few steps, a resized layer) are registered
# anew; after _AUTO_MAX_RESETS such resets the name set stays packed. The
# agreed-call count is part of the agreed value, so every decision that leads
# to a collective (the registration) depends only on agreed state and ranks
# cannot diverge.
_AUTO_ON = 1 << 40          # this rank takes part (device gradients, knob on)
_AUTO_READY = 1 << 41       # ... and its members are the registered tensors
_AUTO_COUNT = 42            # bits 42-43: agreed calls so far (saturating at 3)
_AUTO_MAX_RESETS = 4


def _auto_members(grads: GradientSet, local: list[str], tp):
    """(flags, state) for this call, or None when not applicable."""
    st = tp.__dict__.setdefault("_auto_agg", {}).setdefault(
        grads.__dict__["_name_key"], {"count": 0, "ids": None, "ptrs": None, "bids": None, "disabled": False})
    if st["disabled"]:
        return 0, st
    ts = [grads.get(nm) for nm in local]
    if not all(t.is_cuda for t in ts) or tp.__dict__.get("_knobs", {}).get("auto_register", 2) <= 1:
        return 0, st
    on = _AUTO_ON | (min(st["count"], 3) << _AUTO_COUNT)
    if st["ids"] is None:
        return on, st
    ptrs = tuple(t.payload.data_ptr() for t in ts)
    if ptrs != st["ptrs"] or _buffer_ids(tp, ptrs) != st["bids"]:
        return on, st
    return on | _AUTO_READY, st


def _auto_reset(tp, st):
    """After a call whose agreement failed on the registration state (every
    rank runs this for the same call): drop this rank's registration of the
    name set and count agreed calls from zero, or stop offering for good."""
    if st["ptrs"] is not None:
        for ptr in st["ptrs"]:          # local bookkeeping only; peers' mappings stay cached
            L.lib.cm_comm_deregister(tp._h, C.c_void_p(ptr))
    st.update(count=0, ids=None, ptrs=None, bids=None)
    st["resets"] = st.get("resets", 0) + 1
    if st["resets"] > _AUTO_MAX_RESETS:
        st["disabled"] = True


def _buffer_ids(tp, ptrs) -> tuple:
    ids = (C.c_uint64 * max(1, len(ptrs)))()
    L.check(L.lib.cm_buffer_ids(tp._h, len(ptrs), L.ptr_array(list(ptrs)), ids))
    return tuple(ids[:len(ptrs)])


def _auto_after_call(grads, local, tp, st):
    """After an agreed call in which every rank offered registration."""
    st["count"] += 1
    if st["count"] == 2 and st["ids"] is None:
        ts = [grads.get(nm) for nm in local]
        ids = tp.register_buffers([t.payload for t in ts], tolerant=True)   # collective, once per name set
        if ids is None:                     # some rank's allocations cannot be shared: stay packed
            st["disabled"] = True
            return
        st["ids"] = dict(zip(local, ids))
        st["ptrs"] = tuple(t.payload.data_ptr() for t in ts)
        st["bids"] = _buffer_ids(tp, st["ptrs"])


def register_gradients(grads: GradientSet, transport: Communicator) -> None:
    """Collective: register every gradient tensor of ``grads`` (sorted by
    name, so ids agree across ranks) for zero-copy aggregation. Later
    ``aggregate`` calls on this GradientSet skip the pack: peers read the
    member tensors in place through the registered IPC mappings (the pointer
    cache of PAPER §V-B applied to peer mappings). The tensors must stay
    allocated for the lifetime of the registration."""
    tp = transport
    ordered = sorted(grads.tensors, key=lambda t: t.name)
    for t in ordered:
        if not t.is_cuda:
            raise ShapeError(f"{t.name}: only device tensors can be registered")
    ids = tp.register_buffers([t.payload for t in ordered]) if ordered else []
    object.__setattr__(grads, "_reg_ids", {t.name: i for t, i in zip(ordered, ids)})
    grads.__dict__.pop("_plans", None)


def _device_of(tp):
    """torch's current device for the bucket allocations (a no-op context
    when it already is the communicator's)."""
    if torch.cuda.current_device() == tp.device.index:
        return contextlib.nullcontext()
    return torch.cuda.device(tp.device)


def _aggregate_names(grads, names, tp, algo, cfg, sw, registry, handles, stats_out, out, agree, regmap=None):
    if not names:
        return GradientSet((), grads.iteration)
    cache = grads.__dict__.setdefault("_plans", {})
    pkey = (tuple(names), id(regmap) if regmap is not None else None)
    plan = cache.get(pkey)
    if plan is None:
        plan = cache[pkey] = _Plan(grads, names, regmap)
    if registry is not None and handles is not None:
        for grp in fuse_plan(plan.ready, cfg):       # aggregation.py:159-161
            for i in grp:
                registry.classify(handles[plan.ready[i].name])
    # out= reuses the previous result's buckets (device, or pinned host for
    # host gradients) when the schema matches
    # (checked locally but never raised: this rank's plan may be the one that
    # disagrees, and the agreement inside the call must still run on every
    # rank — a non-matching out= just gets fresh buckets)
    reuse = out.__dict__.get("_bufs") if out is not None else None
    if reuse is not None and [(f.numel(), f.is_cuda) for f in reuse] != \
            [(r["total"], not r["any_host"]) for r in plan.runs]:
        reuse = None
    # same schema and names: the result tensors are views of the reused
    # buckets already, so `out` itself is refilled and returned (torch out=)
    refill = reuse is not None and out.names == list(names)
    result: list[Tensor] = []
    bufs = []
    stream = tp._stream()
    fast = L.fast
    with _device_of(tp):
        for ri, run in enumerate(plan.runs):
            dtype = run["dtype"]
            if reuse is not None:
                fused = reuse[ri]
            elif run["any_host"]:
                # CUDA-aware semantics: host gradients get host means. The C
                # call streams H2D / collectives / D2H on separate streams
                # straight into this pinned bucket.
                fused = torch.empty(run["total"], dtype=DTYPES[dtype], pin_memory=True)
            else:
                fused = torch.empty(run["total"], dtype=DTYPES[dtype], device=tp.device)
            if fast is not None:
                pa, ca, ra, sa = run["addr"]
                status, ok, ncalls = fast.fused(
                    tp._hv, run["n"], pa, ca, L.DTYPE[dtype], fused.data_ptr(), L.ALGO[algo],
                    int(cfg.threshold_bytes), sw, 1, C.addressof(agree) if agree is not None else 0,
                    2 if agree is not None else 0, ra, stream, sa)
                if status:
                    L.check(status)
            else:
                nc, ag = C.c_int(), C.c_int(1)
                L.check(L.lib.cm_fused_allreduce_agreed(
                    tp._h, run["n"], run["ptrs"], run["counts_c"], L.DTYPE[dtype], fused.data_ptr(),
                    L.ALGO[algo], int(cfg.threshold_bytes), sw, 1, agree, 2 if agree is not None else 0,
                    C.byref(ag), run["reg"], stream, run["stats"], C.byref(nc)))
                ok, ncalls = ag.value, nc.value
            if not ok:
                return None             # nothing was launched
            agree = None
            if stats_out is not None:
                stats_out.extend(_stats(run["stats"][k]) for k in range(ncalls))
            bufs.append(fused)
            if refill:
                continue
            for nm, view in zip(run["names"], fused.split_with_sizes(run["counts"])):
                result.append(Tensor._wrap(nm, dtype, view))
    if tp.blocking or any(r["any_host"] for r in plan.runs):
        tp.synchronize()
    else:
        tp.poll()
    if refill:
        object.__setattr__(out, "iteration", grads.iteration)
        return out
    gs = GradientSet.__new__(GradientSet)
    object.__setattr__(gs, "tensors", tuple(result))
    object.__setattr__(gs, "iteration", grads.iteration)
    object.__setattr__(gs, "_bufs", bufs)
    return gs


def negotiate_ready_group(per_rank_ready: list[list[str]], vg: VirtualGroup) -> list[list[str]]:
    """``negotiate_ready`` for every rank of a VirtualGroup: the same fast path
    (``cm_agree_v``: one int64 MAX-allreduce of (key, count, -key, -count)
    over the virtual ranks) and, on a mismatch, the reference's intersection
    (aggregation.py:72-92)."""
    p = vg.size
    if len(per_rank_ready) != p:
        raise ShapeError(f"{len(per_rank_ready)} ready sets for a group of {p}")
    names = [sorted(r) for r in per_rank_ready]
    if p == 1:
        return names
    vals = []
    for nm in names:
        k = _name_key(nm)
        vals += [k, len(nm), -k, -len(nm)]
    mx = (C.c_int64 * (4 * p))()
    with torch.cuda.device(vg.device):
        L.check(L.lib.cm_agree_v(vg._h, L.i64_array(vals), 4, mx, vg._stream()))
    if all(list(mx[4 * r:4 * r + 4]) == vals[4 * r:4 * r + 4] for r in range(p)):
        return names
    common = set(names[0])
    for nm in names[1:]:
        common &= set(nm)
    return [sorted(common)] * p


def register_gradients_group(per_rank: list[GradientSet], vg: VirtualGroup) -> None:
    """``register_gradients`` for every rank of a VirtualGroup: every
    gradient (sorted by name; every rank must hold the same names) gets one
    registered-buffer id, so ``aggregate_group`` reads the members in place
    (SRC_GATHER, the registered path of real communicators)."""
    names = sorted(per_rank[0].names)
    for g in per_rank[1:]:
        if sorted(g.names) != names:
            raise ShapeError("every rank must register the same gradient names")
    for g in per_rank:
        for nm in names:
            if not g.get(nm).is_cuda:
                raise ShapeError(f"{nm}: only device tensors can be registered")
    ids = vg.register_buffers([[g.get(nm).payload for g in per_rank] for nm in names]) if names else []
    for g in per_rank:
        object.__setattr__(g, "_reg_ids", dict(zip(names, ids)))


def aggregate_group(per_rank: list[GradientSet], vg: VirtualGroup, algo: str = "auto",
                    cfg: FusionConfig | None = None,
                    switch_bytes: int | None = DEFAULT_SWITCH_BYTES,
                    stats_out: list[list[CollectiveStats]] | None = None,
                    agree: bool = True) -> list[GradientSet]:
    """``aggregate`` for every rank of a single-GPU VirtualGroup through the
    same C path as a real communicator (``cm_fused_allreduce_agreed_v``):
    inline ready-set agreement in the first fused collective, packs into each
    rank's staging (or in-place reads of registered gradients), multi-buffer
    two-shot launches with the fused mean, host gradients through the copy
    streams. If the ranks' ready sets differ, the intersection is negotiated
    as in the reference (aggregation.py:72-92) and the call repeats.

    One launch covers all virtual ranks, so the first (agreed) attempt needs
    every rank's schema to have the same shape; otherwise the intersection is
    taken up front."""
    cfg = cfg or FusionConfig()
    p = vg.size
    if len(per_rank) != p:
        raise ShapeError(f"{len(per_rank)} gradient sets for a group of {p}")
    if algo not in L.ALGO:
        from .errors import ConfigError
        raise ConfigError(f"unknown algorithm {algo!r}")
    sw = _switch(switch_bytes, p)
    local = [sorted(g.names) for g in per_rank]
    if stats_out is not None:
        stats_out.extend([] for _ in range(p))

    def shape(r):
        return [(per_rank[r].get(nm).dtype, per_rank[r].get(nm).len) for nm in local[r]]
    res = None
    if agree and p > 1 and local[0] and all(shape(r) == shape(0) for r in range(1, p)):
        vals = []
        for nm in local:
            vals += [_name_key(nm), len(nm)]
        res = _aggregate_group_names(per_rank, local, vg, algo, cfg, sw, stats_out, vals)
    if res is None:
        common = set(local[0])
        for nm in local[1:]:
            common &= set(nm)
        names = sorted(common)
        res = _aggregate_group_names(per_rank, [names] * p, vg, algo, cfg, sw, stats_out, None)
    return res


def _aggregate_group_names(per_rank, names, vg, algo, cfg, sw, stats_out, agree_vals):
    p = vg.size
    ready = [[per_rank[r].get(nm) for nm in names[r]] for r in range(p)]
    for r in range(1, p):
        if [(t.dtype, t.len) for t in ready[r]] != [(t.dtype, t.len) for t in ready[0]]:
            raise ShapeError("collective shape error: ranks disagree on the negotiated gradient shapes")
    outs: list[list[Tensor]] = [[] for _ in range(p)]
    stats: list[list[CollectiveStats]] = [[] for _ in range(p)]
    regmaps = [g.__dict__.get("_reg_ids") for g in per_rank]
    agree = L.i64_array(agree_vals) if agree_vals is not None else None
    i = 0
    stream = vg._stream()
    with torch.cuda.device(vg.device):
        while i < len(ready[0]):
            j = i
            while j < len(ready[0]) and ready[0][j].dtype == ready[0][i].dtype:
                j += 1
            dtype = ready[0][i].dtype
            if dtype not in ("float32", "float64", "bfloat16"):
                raise ShapeError(f"aggregate averages floating-point gradients, got {dtype}")
            run = [ready[r][i:j] for r in range(p)]
            n = j - i
            counts = [t.len for t in run[0]]
            any_host = any(not t.is_cuda for rr in run for t in rr)
            fused = [torch.empty(sum(counts), dtype=DTYPES[dtype], pin_memory=True) if any_host
                     else torch.empty(sum(counts), dtype=DTYPES[dtype], device=vg.device) for _ in range(p)]
            reg = None
            if all(m is not None and all(t.name in m for t in rr) for m, rr in zip(regmaps, run)):
                ids = [regmaps[0][t.name] for t in run[0]]
                if all([m[t.name] for t in rr] == ids for m, rr in zip(regmaps, run)):
                    reg = L.i64_array(ids)
            st = (L.Stats * (p * max(1, n)))()
            ncalls = C.c_int()
            agreed = (C.c_int * p)(*([1] * p))
            L.check(L.lib.cm_fused_allreduce_agreed_v(
                vg._h, n, L.ptr_array([t.payload.data_ptr() for rr in run for t in rr]), L.i64_array(counts),
                L.DTYPE[dtype], L.ptr_array([f.data_ptr() for f in fused]), L.ALGO[algo],
                int(cfg.threshold_bytes), sw, 1, agree, 2 if agree is not None else 0, agreed, reg,
                stream, st, C.byref(ncalls)))
            if agree is not None and not all(agreed):
                return None             # nothing moved on any rank
            agree = None
            for r in range(p):
                stats[r].extend(_stats(st[r * n + k]) for k in range(ncalls.value))
                for t, view in zip(run[r], fused[r].split_with_sizes(counts)):
                    outs[r].append(Tensor._wrap(t.name, dtype, view))
            i = j
    vg.synchronize()
    if stats_out is not None:
        for r in range(p):
            stats_out[r].extend(stats[r])
    return [GradientSet(tuple(outs[r]), per_rank[r].iteration) for r in range(p)]
