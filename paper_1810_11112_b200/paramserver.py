"""Parameter-server pull step on the NVLink communicator (SURVEY section 8f
item 4; the reference's paramserver.py).

Same topology object and step semantics as the reference:
``PsTopology.create(workers, ps, names)`` shards tensors round-robin over the
PS ranks in sorted name order (paramserver.py:159-165); ``run_ps_step``
(paramserver.py:171-271) has every owner average the workers' gradient
shards in worker-rank order in float64 and apply ``param - lr * mean``, and
returns the updated parameters on worker ranks (None on pure PS ranks).
Instead of byte messages through a tensor table, workers stage their
gradients in the IPC heap, owners read them over NVLink and update in one
kernel (``cm_ps_step``), and workers pull the updated shards from the owners'
heaps in the same launch. Results are bit-identical to the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .comm import Communicator, VirtualGroup
from .core import DTYPES, Tensor
from .errors import ProtocolError, ShapeError


@dataclass(frozen=True)
class PsTopology:
    """paramserver.py:139-169: worker / PS rank sets (may overlap) and the
    tensor name -> owning PS rank shard map."""
    worker_ranks: tuple
    ps_ranks: tuple
    shard_map: dict = field(default_factory=dict)

    def __post_init__(self):
        object.__setattr__(self, "worker_ranks", tuple(sorted(self.worker_ranks)))
        object.__setattr__(self, "ps_ranks", tuple(sorted(self.ps_ranks)))
        if not self.worker_ranks or not self.ps_ranks:
            raise ProtocolError("topology needs at least one worker and one PS")
        for name, owner in self.shard_map.items():
            if owner not in self.ps_ranks:
                raise ProtocolError(f"shard {name!r} maps to non-PS rank {owner}")

    @property
    def size(self) -> int:
        return max(max(self.worker_ranks), max(self.ps_ranks)) + 1

    @classmethod
    def create(cls, workers, ps, names) -> "PsTopology":
        ps = tuple(sorted(ps))
        return cls(tuple(workers), ps, {name: ps[i % len(ps)] for i, name in enumerate(sorted(names))})

    def owned_names(self, ps_rank: int) -> list:
        return sorted(n for n, o in self.shard_map.items() if o == ps_rank)


class _Schema:
    def __init__(self, topology: PsTopology, params: list, p: int):
        if topology.size > p:
            raise ShapeError(f"topology spans {topology.size} ranks, the group has {p}")
        names = sorted(t.name for t in params)
        if set(topology.shard_map) != set(names):
            raise ShapeError("shard map does not cover the parameter schema")
        by = {t.name: t for t in params}
        self.names = names
        self.dtype = by[names[0]].dtype
        if any(by[n].dtype != self.dtype for n in names):
            raise ShapeError("the parameter-server step needs one dtype per schema")
        if self.dtype not in ("float32", "float64"):
            raise ShapeError(f"unsupported parameter dtype {self.dtype}")
        self.counts = [by[n].len for n in names]
        self.total = sum(self.counts)
        self.counts_c = L.i64_array(self.counts)
        self.owners_c = (C.c_int * len(names))(*[topology.shard_map[n] for n in names])
        self.mask = sum(1 << w for w in topology.worker_ranks)


def _fused_params(params: list, names: list, device, buf=None) -> torch.Tensor:
    by = {t.name: t for t in params}
    total = sum(by[n].len for n in names)
    dt = DTYPES[by[names[0]].dtype]
    if buf is None or buf.numel() != total or buf.dtype != dt:
        buf = torch.empty(total, dtype=dt, device=device)
    torch.cat([by[n].payload.to(device).reshape(-1) for n in names], out=buf)
    return buf


def run_ps_step(rank: int, comm: Communicator, topology: PsTopology, grads: list | None, params: list,
                learning_rate: float) -> list | None:
    """One rank's side of the synchronous PS step (paramserver.py:171-271).
    Every rank of the communicator must call it (ranks outside the topology
    included). Returns the updated parameters (in ``params`` order, device
    tensors) on worker ranks, None otherwise."""
    if rank != comm.rank:
        raise ShapeError(f"rank {rank} does not match the communicator's rank {comm.rank}")
    is_worker = rank in topology.worker_ranks
    if is_worker and grads is None:
        raise ProtocolError(f"worker rank {rank} called without gradients")
    sch = _Schema(topology, params, comm.size)
    gptr = [None] * len(sch.names)
    if is_worker:
        gby = {t.name: t for t in grads}
        if set(gby) != set(sch.names):
            raise ShapeError("gradient schema does not match parameters")
        gts = [gby[n].payload.to(comm.device) for n in sch.names]
        for n, g, c in zip(sch.names, gts, sch.counts):
            if g.numel() != c or g.dtype != DTYPES[sch.dtype]:
                raise ShapeError(f"gradient {n!r} does not match its parameter")
        gptr = [g.data_ptr() for g in gts]
    buf = _fused_params(params, sch.names, comm.device)
    with torch.cuda.device(comm.device):
        L.check(L.lib.cm_ps_step(comm._h, len(sch.names), L.ptr_array([x or 0 for x in gptr]), buf.data_ptr(),
                                 sch.counts_c, L.DTYPE[sch.dtype], sch.owners_c, sch.mask,
                                 float(learning_rate), comm._stream()))
    if comm.blocking:
        comm.synchronize()
    else:
        comm.poll()
    if not is_worker:
        return None
    views = dict(zip(sch.names, buf.split(sch.counts)))
    return [Tensor._wrap(t.name, sch.dtype, views[t.name]) for t in params]


def run_ps_step_group(vg: VirtualGroup, topology: PsTopology, grads_per_rank: list, params_per_rank: list,
                      learning_rate: float) -> list:
    """``run_ps_step`` for every rank of a single-GPU VirtualGroup;
    ``grads_per_rank[r]`` is None for non-workers. Returns per-rank results."""
    p = vg.size
    sch = _Schema(topology, params_per_rank[0], p)
    gptrs, bufs, keep = [], [], []
    for r in range(p):
        if r in topology.worker_ranks:
            gby = {t.name: t.payload.to(vg.device) for t in grads_per_rank[r]}
            keep.extend(gby.values())
            gptrs.extend(gby[n].data_ptr() for n in sch.names)
        else:
            gptrs.extend([0] * len(sch.names))
        bufs.append(_fused_params(params_per_rank[r], sch.names, vg.device))
    with torch.cuda.device(vg.device):
        L.check(L.lib.cm_ps_step_v(vg._h, len(sch.names), L.ptr_array(gptrs), L.ptr_array([b.data_ptr() for b in bufs]),
                                   sch.counts_c, L.DTYPE[sch.dtype], sch.owners_c, sch.mask,
                                   float(learning_rate), vg._stream()))
    vg.synchronize()
    out = []
    for r in range(p):
        if r not in topology.worker_ranks:
            out.append(None)
            continue
        views = dict(zip(sch.names, bufs[r].split(sch.counts)))
        out.append([Tensor._wrap(t.name, sch.dtype, views[t.name]) for t in params_per_rank[r]])
    return out
