"""Overlapped gradient aggregation (the caller side of
the path): fused allreduces start while the backward pass is still producing
gradients, as Horovod's background coordinator and PyTorch DDP's buckets do.

The fusion plan is the reference's (aggregation.py:95-130: canonical sorted
names, greedy first-fit under the threshold) computed ONCE over the full
gradient schema, so every fused group, its ring chunking and therefore every
result bit are identical to ``aggregate`` over the complete set
(aggregation.py:138-176). Groups are launched in a fixed order that is the
same on every rank (reverse plan order by default: backward produces the
last layers first), each as soon as it and every group before it in that
order are complete, on a communication stream that waits only for the
producer-stream event of the group's last gradient. ``finish`` joins the
communication stream into the caller's stream and returns the means.

Ranks may mark gradients ready in different orders; the launch order is
static, so the collectives still match one to one across ranks (no
negotiation round per step).
"""

from __future__ import annotations

import ctypes as C
from collections import namedtuple

import torch

from . import _lib as L
from .aggregation import FusionConfig, GradientSet, fuse_plan
from .collectives import DEFAULT_SWITCH_BYTES, CollectiveStats
from .comm import Communicator
from .core import DTYPES, Tensor
from .errors import ConfigError, ShapeError
from .tuning import switch_bytes_for

_Spec = namedtuple("_Spec", "name len dtype nbytes")


class OverlappedAggregator:
    """``ready(name, grad)`` per gradient as the backward pass produces it,
    then ``finish()`` -> GradientSet of means (canonical order), identical
    to ``aggregate(all gradients)``.

    ``schema``: a GradientSet (used as a template) or ``[(name, numel,
    dtype), ...]``. ``launch_order``: "reverse" (default, last layers first)
    or "forward". ``max_ctas`` caps the CTAs of each overlapped collective
    (None: the communicator's setting) — except the last group in launch
    order, which runs once the backward pass is done and gets the full grid;
    ``cluster_pairs``: capped grids launch in 2-CTA clusters so they occupy
    whole TPCs (cuBLAS's 2-SM-cluster GEMMs keep their pairs); ``pack_ctas``
    caps the member pack that precedes each overlapped collective;
    ``priority`` is the communication stream's priority (0: normal, measured
    faster than -1 = high at N = 4, `profiles/r02_overlap_priority_n4.txt`);
    ``register_members``: at the end of the first step every rank registers
    the gradient tensors it handed to ``ready()`` (collective, the pointer
    cache's IPC side, as ``register_gradients``), and from then on peers read
    them in place — no member pack next to the backward pass. The caller
    hands over the same tensors every step (a framework's persistent
    gradient buffers); a rank whose tensors moved packs instead, which the
    fused launch's header check turns into a ShapeError on every rank.

    Stream rules (as for NCCL communicators): the means are views of
    persistent per-group buckets that the next step overwrites once its
    group's gradients are ready on the producer stream, so consume them on
    that stream before producing the next gradients; while a step is in
    flight, issue no other collective on the same communicator from another
    stream."""

    def __init__(self, schema, comm: Communicator, algo: str = "auto", cfg: FusionConfig | None = None,
                 switch_bytes: int | None = DEFAULT_SWITCH_BYTES, launch_order: str = "reverse",
                 max_ctas: int | None = 64, priority: int = 0, cluster_pairs: bool = False,
                 pack_ctas: int | None = None, register_members: bool = False):
        if isinstance(schema, GradientSet):
            specs = [(t.name, t.len, t.dtype) for t in schema.tensors]
        else:
            specs = list(schema)
        if len({nm for nm, _, _ in specs}) != len(specs):
            raise ShapeError("duplicate gradient names in the schema")
        self.comm = comm
        self.algo = algo
        self.cfg = cfg or FusionConfig()
        self.switch = switch_bytes_for(comm.size) if switch_bytes is None else int(switch_bytes)
        self.specs = sorted((_Spec(nm, int(n), dt, int(n) * torch.empty((), dtype=DTYPES[dt]).element_size())
                             for nm, n, dt in specs), key=lambda s: s.name)       # aggregation.py:77,85
        for s in self.specs:
            if s.dtype not in ("float32", "float64", "bfloat16"):
                raise ShapeError(f"aggregate averages floating-point gradients, got {s.dtype}")
        self.groups = fuse_plan(self.specs, self.cfg)
        self.by_name = {s.name: s for s in self.specs}
        self.group_of = {}
        for g, members in enumerate(self.groups):
            for i in members:
                self.group_of[self.specs[i].name] = g
        if launch_order == "reverse":
            self.order = list(range(len(self.groups)))[::-1]
        elif launch_order == "forward":
            self.order = list(range(len(self.groups)))
        else:
            raise ConfigError(f"launch_order must be 'reverse' or 'forward', got {launch_order!r}")
        dev = comm.device
        # communication stream (normal priority by default: a high-priority
        # stream's CTAs jump ahead of the backward GEMMs' and measured slower);
        # a CTA cap leaves SMs to the backward pass (the collective is
        # NVLink-bound well below 148 CTAs)
        self.stream = torch.cuda.Stream(dev, priority=priority)
        self.max_ctas = max_ctas
        self.cluster_pairs = cluster_pairs
        self.pack_ctas = pack_ctas
        self.register_members = register_members
        self._reg = [None] * len(self.groups)        # per group: member reg ids (C int64 array)
        self._regptrs = [None] * len(self.groups)    # ... and the member addresses they belong to
        self.buckets = [torch.empty(sum(self.specs[i].len for i in m), dtype=DTYPES[self.specs[m[0]].dtype],
                                    device=dev) for m in self.groups]
        self.stats = [(L.Stats * 1)() for _ in self.groups]
        # per group, allocated once: member pointer / count arrays, the
        # producer-side event, and the plain addresses the fast-call path takes
        # (ready() runs inside the backward loop, which is host-bound)
        self._ptrs = [(C.c_void_p * len(m))() for m in self.groups]
        self._counts = [L.i64_array([self.specs[i].len for i in m]) for m in self.groups]
        self._ev = [torch.cuda.Event() for _ in self.groups]
        self._gdtype = [L.DTYPE[self.specs[m[0]].dtype] for m in self.groups]
        self._addr = [(C.addressof(p), C.addressof(c), C.addressof(st), b.data_ptr())
                      for p, c, st, b in zip(self._ptrs, self._counts, self.stats, self.buckets)]
        self._cap_set = None
        # the means are views of the persistent buckets: built once, handed out
        # every step (finish() runs on the host critical path of the step)
        views = {}
        for g, m in enumerate(self.groups):
            for sp, v in zip((self.specs[i] for i in m), self.buckets[g].split([self.specs[i].len for i in m])):
                views[sp.name] = Tensor._wrap(sp.name, sp.dtype, v)
        self._views = tuple(views[sp.name] for sp in self.specs)
        self.step_stats: list[CollectiveStats] = []
        self.iteration = 0
        self._reset()

    # -- per step ---------------------------------------------------------------
    def _reset(self):
        self._cap_saved = getattr(self, "_cap_saved", None)
        self._tensors = {}
        self._missing = [len(m) for m in self.groups]
        self._events = [None] * len(self.groups)
        self._next = 0
        self.step_stats = []

    def ready(self, name: str, grad) -> None:
        """Hand over one gradient (torch CUDA tensor or Tensor) produced on
        the current stream; launches every fused group that became due."""
        t = grad.payload if isinstance(grad, Tensor) else grad
        g = self.group_of.get(name)
        if g is None:
            raise ShapeError(f"{name!r} is not in the gradient schema")
        if name in self._tensors:
            raise ShapeError(f"{name!r} marked ready twice in one step")
        spec = self.by_name[name]
        if not t.is_cuda or t.numel() != spec.len or t.dtype != DTYPES[spec.dtype] or not t.is_contiguous():
            raise ShapeError(f"{name!r}: expected a contiguous CUDA {spec.dtype} tensor of {spec.len} elements")
        t.record_stream(self.stream)              # kept alive until the collective has read it
        self._tensors[name] = t
        self._missing[g] -= 1
        if self._missing[g] == 0:
            ev = self._ev[g]
            ev.record(torch.cuda.current_stream(t.device))
            self._events[g] = ev
            self._launch_due()

    def _launch_due(self):
        while self._next < len(self.order) and self._missing[self.order[self._next]] == 0:
            self._launch(self.order[self._next])
            self._next += 1

    def _launch(self, g: int):
        members = self.groups[g]
        ptrs = self._ptrs[g]
        for k, i in enumerate(members):
            ptrs[k] = self._tensors[self.specs[i].name].data_ptr()
        self.stream.wait_event(self._events[g])
        # the last group in launch order runs after the backward pass is done:
        # nothing to leave SMs for, so it gets the full grid (the cap is set
        # once per step, not per group)
        last = self._next == len(self.order) - 1
        want = None if (last or not self.max_ctas) else self.max_ctas
        if want != self._cap_set:
            if want is not None and self._cap_saved is None:
                self._cap_saved = (self.comm.get_param("max_ctas"), self.comm.get_param("cluster_pairs"),
                                   self.comm.get_param("pack_max_ctas"))
            self.comm.set_param("max_ctas", want if want is not None else self._cap_saved[0])
            if self.cluster_pairs:   # capped grids take whole TPCs (see cm.h "cluster_pairs")
                self.comm.set_param("cluster_pairs", 2 if want is not None else self._cap_saved[1])
            if self.pack_ctas:       # the member pack next to the backward pass, capped too
                self.comm.set_param("pack_max_ctas", self.pack_ctas if want is not None else self._cap_saved[2])
            self._cap_set = want
            if want is None:
                self._cap_saved = None   # re-read next step (the caller may retune the communicator)
        if self._call(g, len(members)) != 1:
            raise ShapeError("internal: an overlapped group split into several fused buffers")

    def _call(self, g, n) -> int:
        """One fused collective for group g on the communication stream;
        returns the number of fused buffers it ran as."""
        pa, ca, sa, out = self._addr[g]
        comm = self.comm
        reg = self._reg[g]
        if reg is not None and tuple(self._ptrs[g]) != self._regptrs[g]:
            reg = None                              # moved: pack (peers see the header mismatch)
        if L.fast is not None:
            status, _, ncalls = L.fast.fused(comm._hv, n, pa, ca, self._gdtype[g], out, L.ALGO[self.algo],
                                             int(self.cfg.threshold_bytes), self.switch, 1, 0, 0,
                                             C.addressof(reg) if reg is not None else 0,
                                             self.stream.cuda_stream, sa)
            if status:
                L.check(status)
            return ncalls
        nc, ag = C.c_int(), C.c_int(1)
        L.check(L.lib.cm_fused_allreduce_agreed(
            comm._h, n, self._ptrs[g], self._counts[g], self._gdtype[g], out, L.ALGO[self.algo],
            int(self.cfg.threshold_bytes), self.switch, 1, None, 0, C.byref(ag), reg,
            self.stream.cuda_stream, self.stats[g], C.byref(nc)))
        return nc.value

    def _register_step_tensors(self):
        """Collective (every rank, end of its first step): register this
        step's gradient tensors in schema order; an allocation that cannot be
        shared on any rank leaves every rank packing."""
        ts = [self._tensors[s.name] for s in self.specs]
        ids = self.comm.register_buffers(ts, tolerant=True)
        if ids is None:
            return
        by_name = {s.name: i for s, i in zip(self.specs, ids)}
        for g, members in enumerate(self.groups):
            names = [self.specs[i].name for i in members]
            self._reg[g] = L.i64_array([by_name[nm] for nm in names])
            self._regptrs[g] = tuple(self._tensors[nm].data_ptr() for nm in names)

    def finish(self) -> GradientSet:
        """Join the communication stream into the caller's stream and return
        the means of this step (views of persistent per-group buckets)."""
        if self._next != len(self.order):
            missing = sorted(s.name for s in self.specs if s.name not in self._tensors)
            raise ShapeError(f"finish() before every gradient was ready: missing {missing[:8]}")
        torch.cuda.current_stream(self.comm.device).wait_stream(self.stream)
        if self.comm.blocking:
            st = (L.fast.sync(self.comm._hv, self.stream.cuda_stream) if L.fast is not None
                  else L.lib.cm_comm_sync(self.comm._h, self.stream.cuda_stream))
        else:
            st = L.fast.poll(self.comm._hv) if L.fast is not None else L.lib.cm_comm_poll(self.comm._h)
        if st:
            L.check(st)
        stats = [CollectiveStats(int(self.stats[g][0].rounds), int(self.stats[g][0].messages_per_rank),
                                 int(self.stats[g][0].bytes_sent_per_rank)) for g in self.order]
        if self.register_members and self.iteration == 0 and self.comm.size > 1:
            self._register_step_tensors()
        gs = GradientSet.__new__(GradientSet)
        object.__setattr__(gs, "tensors", self._views)
        object.__setattr__(gs, "iteration", self.iteration)
        self.iteration += 1
        self._reset()
        self.step_stats = stats
        return gs
