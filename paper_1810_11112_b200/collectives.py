"""Allreduce suite with the reference signatures
(/root/reference/pkg/src/collectium/collectives.py:20-260), executed by
sm_100a kernels over NVLink.

* ``allreduce(t, op, group, transport, algo="auto", switch_bytes=131072)``
  dispatches exactly like ``resolve_algorithm`` (collectives.py:239-247):
  ``rhd_rsa`` below ``switch_bytes``, ``ring_rsa`` at or above it.
* Each algorithm's result is bit-identical to the reference's because the
  kernels replay its per-element fold order (ring: chunk c folds
  x_{c-1}, ..., x_c; rhd: the recursive-halving tree; flat: ranks 0..p-1).
* ``CollectiveStats`` reports the reference's logical schedule (rounds,
  messages, bytes per rank), so count-pinning code keeps working; the bytes
  that really crossed NVLink are ``transport.nvlink_bytes_in``.
* ``transport`` is a ``Communicator`` (one rank per process); a
  ``VirtualGroup`` takes per-rank lists through ``allreduce_group``.
* ``switch_bytes=None`` selects the threshold measured on this box for this
  group size (``tuning.py``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L
from .comm import Communicator, VirtualGroup
from .core import GroupSpec, ReduceOp, Tensor
from .errors import ConfigError, ShapeError

ALGORITHMS = ("flat", "ring_rsa", "rhd_rsa", "auto")          # collectives.py:20
DEFAULT_SWITCH_BYTES = 131072                                 # collectives.py:23


@dataclass(frozen=True)
class CollectiveStats:
    """collectives.py:28-32."""
    rounds: int
    messages_per_rank: int
    bytes_sent_per_rank: int


def _stats(s: L.Stats) -> CollectiveStats:
    return CollectiveStats(int(s.rounds), int(s.messages_per_rank), int(s.bytes_sent_per_rank))


def _check_call(group: GroupSpec, tp) -> None:
    """collectives.py:50-54."""
    if group.size != tp.size:
        raise ShapeError(f"group size {group.size} does not match transport size {tp.size}")


def _switch(switch_bytes, p: int) -> int:
    if switch_bytes is None:
        from .tuning import switch_bytes_for
        return switch_bytes_for(p)
    return int(switch_bytes)


def resolve_algorithm(algo: str, nbytes: int, switch_bytes: int = DEFAULT_SWITCH_BYTES) -> str:
    """collectives.py:239-247 (computed by cm_resolve_algorithm)."""
    if algo not in L.ALGO:
        raise ConfigError(f"unknown algorithm {algo!r}")
    out = C.c_int()
    L.check(L.lib.cm_resolve_algorithm(L.ALGO[algo], int(nbytes), int(switch_bytes), C.byref(out)))
    return L.ALGO_NAME[out.value]


def _out_like(t: Tensor) -> torch.Tensor:
    return torch.empty_like(t.payload)


def _finish(tp: Communicator, out: torch.Tensor) -> None:
    if tp.blocking or not out.is_cuda:
        tp.synchronize()
    else:
        tp.poll()


def _run(fast_fn, ctypes_fn, args) -> CollectiveStats:
    """One entry-point call: through the CPython fast-call module when it is
    built (integers in, (status, rounds, messages, bytes) out), else ctypes."""
    if L.fast is not None:
        status, r, m, b = fast_fn(*args)
        if status:
            L.check(status)
        return CollectiveStats(r, m, b)
    st = L.Stats()
    L.check(ctypes_fn(*args, C.byref(st)))
    return _stats(st)


def allreduce(t: Tensor, op: ReduceOp, group: GroupSpec, transport: Communicator,
              algo: str = "auto", switch_bytes: int | None = DEFAULT_SWITCH_BYTES,
              out: torch.Tensor | None = None, average: bool = False
              ) -> tuple[Tensor, CollectiveStats]:
    """Allreduce ``t`` over the group; returns a NEW tensor (or ``out``) and
    the reference CollectiveStats of the resolved algorithm."""
    tp = transport
    if group.size != tp.size:
        _check_call(group, tp)
    sw = switch_bytes if type(switch_bytes) is int else _switch(switch_bytes, tp.size)
    a = L.ALGO.get(algo)
    if a is None:
        raise ConfigError(f"unknown algorithm {algo!r}")
    x = t.payload
    if out is None:
        res = torch.empty_like(x)
    else:
        res = out
        if res.numel() != x.shape[0] or res.dtype != x.dtype:
            raise ShapeError("output buffer does not match the input")
    st = _run(L.fast.allreduce if L.fast is not None else None, L.lib.cm_allreduce,
              (tp._hv if L.fast is not None else tp._h, x.data_ptr(), res.data_ptr(), x.shape[0],
               L.DTYPE[t.dtype], L.OP[op.value], a, sw, 1 if average else 0, tp._stream()))
    _finish(tp, res)
    return Tensor._wrap(t.name, t.dtype, res), st


def allreduce_ring(t: Tensor, op: ReduceOp, group: GroupSpec,
                   transport: Communicator) -> tuple[Tensor, CollectiveStats]:
    """Ring RSA fold order (collectives.py:107-152)."""
    return allreduce(t, op, group, transport, algo="ring_rsa")


def allreduce_rhd(t: Tensor, op: ReduceOp, group: GroupSpec,
                  transport: Communicator) -> tuple[Tensor, CollectiveStats]:
    """Recursive halving/doubling fold order (collectives.py:155-236)."""
    return allreduce(t, op, group, transport, algo="rhd_rsa")


def allreduce_flat(t: Tensor, op: ReduceOp, group: GroupSpec,
                   transport: Communicator) -> Tensor:
    """Rank-order fold (collectives.py:75-104)."""
    return allreduce(t, op, group, transport, algo="flat")[0]


def reduce_scatter(t: Tensor, op: ReduceOp, group: GroupSpec, transport: Communicator,
                   layout: str = "ring") -> tuple[Tensor, CollectiveStats]:
    """The reduce-scatter phase as a public operation: "ring" leaves chunk r
    of chunk_partition(n, p) on rank r in ring fold order
    (collectives.py:128-139); "rhd" leaves the recursive-halving segment in
    tree order (:178-216; folded odd ranks receive an empty tensor)."""
    _check_call(group, transport)
    tp = transport
    from .core import layout as _layout
    off, ln = _layout(layout, t.len, tp.size)[tp.rank]
    res = torch.empty(ln, dtype=t.payload.dtype, device=t.payload.device)
    st = _run(L.fast.reduce_scatter if L.fast is not None else None, L.lib.cm_reduce_scatter,
              (tp._hv if L.fast is not None else tp._h, t.payload.data_ptr(), res.data_ptr(), t.len,
               L.DTYPE[t.dtype], L.OP[op.value], L.LAYOUT[layout], tp._stream()))
    _finish(tp, res)
    return Tensor._wrap(t.name, t.dtype, res), st


def allgather(t: Tensor, n: int, group: GroupSpec, transport: Communicator,
              layout: str = "ring") -> tuple[Tensor, CollectiveStats]:
    """Inverse of ``reduce_scatter``: ``t`` is this rank's layout segment of
    an ``n``-element vector; every rank gets the whole vector
    (collectives.py:142-150 ring, :219-235 rhd)."""
    _check_call(group, transport)
    tp = transport
    from .core import layout as _layout
    off, ln = _layout(layout, n, tp.size)[tp.rank]
    if t.len != ln:
        raise ShapeError(f"rank {tp.rank} owns {ln} elements of the {layout} layout, got {t.len}")
    res = torch.empty(n, dtype=t.payload.dtype, device=t.payload.device)
    st = _run(L.fast.allgather if L.fast is not None else None, L.lib.cm_allgather,
              (tp._hv if L.fast is not None else tp._h, t.payload.data_ptr(), res.data_ptr(), n,
               L.DTYPE[t.dtype], L.LAYOUT[layout], tp._stream()))
    _finish(tp, res)
    return Tensor._wrap(t.name, t.dtype, res), st


# -- single-GPU group emulation -------------------------------------------------

def _vg_inputs(tensors, vg: VirtualGroup):
    if len(tensors) != vg.size:
        raise ShapeError(f"{len(tensors)} inputs for a group of {vg.size}")
    dts = {t.dtype for t in tensors}
    if len(dts) != 1:
        raise ShapeError("ranks disagree on dtype")
    ins = [t.payload if t.payload.is_cuda else t.payload.to(vg.device) for t in tensors]
    return ins, dts.pop()


def allreduce_group(tensors: list[Tensor], op: ReduceOp, vg: VirtualGroup, algo: str = "auto",
                    switch_bytes: int | None = DEFAULT_SWITCH_BYTES, average: bool = False
                    ) -> list[tuple[Tensor, CollectiveStats]]:
    """Every rank's allreduce result for per-rank inputs ``tensors`` (one
    kernel launch on one GPU)."""
    ins, dtype = _vg_inputs(tensors, vg)
    lens = {t.numel() for t in ins}
    if len(lens) != 1:
        raise ShapeError(f"collective shape error: ranks hold {sorted(lens)} elements")
    if algo not in L.ALGO:
        raise ConfigError(f"unknown algorithm {algo!r}")
    n = lens.pop()
    outs = [torch.empty_like(x) for x in ins]
    st = (L.Stats * vg.size)()
    with torch.cuda.device(vg.device):
        L.check(L.lib.cm_allreduce_v(vg._h, L.ptr_array([x.data_ptr() for x in ins]),
                                     L.ptr_array([o.data_ptr() for o in outs]), n, L.DTYPE[dtype],
                                     L.OP[op.value], L.ALGO[algo], _switch(switch_bytes, vg.size),
                                     1 if average else 0, vg._stream(), st))
    vg.synchronize()
    return [(Tensor(t.name, dtype, o), _stats(st[i])) for i, (t, o) in enumerate(zip(tensors, outs))]


def reduce_scatter_group(tensors: list[Tensor], op: ReduceOp, vg: VirtualGroup,
                         layout: str = "ring") -> list[tuple[Tensor, CollectiveStats]]:
    ins, dtype = _vg_inputs(tensors, vg)
    n = ins[0].numel()
    if any(x.numel() != n for x in ins):
        raise ShapeError("collective shape error: ranks disagree on length")
    from .core import layout as _layout
    lay = _layout(layout, n, vg.size)
    outs = [torch.empty(ln, dtype=ins[0].dtype, device=vg.device) for _, ln in lay]
    st = (L.Stats * vg.size)()
    with torch.cuda.device(vg.device):
        L.check(L.lib.cm_reduce_scatter_v(vg._h, L.ptr_array([x.data_ptr() for x in ins]),
                                          L.ptr_array([o.data_ptr() for o in outs]), n,
                                          L.DTYPE[dtype], L.OP[op.value], L.LAYOUT[layout],
                                          vg._stream(), st))
    vg.synchronize()
    return [(Tensor(t.name, dtype, o), _stats(st[i])) for i, (t, o) in enumerate(zip(tensors, outs))]


def allgather_group(segments: list[Tensor], n: int, vg: VirtualGroup,
                    layout: str = "ring") -> list[tuple[Tensor, CollectiveStats]]:
    ins, dtype = _vg_inputs(segments, vg)
    from .core import layout as _layout
    lay = _layout(layout, n, vg.size)
    for r, (x, (_, ln)) in enumerate(zip(ins, lay)):
        if x.numel() != ln:
            raise ShapeError(f"rank {r} owns {ln} elements of the {layout} layout, got {x.numel()}")
    outs = [torch.empty(n, dtype=ins[0].dtype, device=vg.device) for _ in ins]
    st = (L.Stats * vg.size)()
    with torch.cuda.device(vg.device):
        L.check(L.lib.cm_allgather_v(vg._h, L.ptr_array([x.data_ptr() for x in ins]),
                                     L.ptr_array([o.data_ptr() for o in outs]), n, L.DTYPE[dtype],
                                     L.LAYOUT[layout], vg._stream(), st))
    vg.synchronize()
    return [(Tensor(t.name, dtype, o), _stats(st[i])) for i, (t, o) in enumerate(zip(segments, outs))]


def algo_stats(algo: str, p: int, rank: int, n: int, dtype: str = "float32",
               switch_bytes: int = DEFAULT_SWITCH_BYTES) -> CollectiveStats:
    """The CollectiveStats the reference reports for this call (host logic only)."""
    st = L.Stats()
    L.check(L.lib.cm_algo_stats(L.ALGO[algo], p, rank, n, L.DTYPE[dtype], switch_bytes, C.byref(st)))
    return _stats(st)
