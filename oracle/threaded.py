"""Message-passing port of the reference CPU allreduce path — TEST / BASELINE
INFRASTRUCTURE.

A line-by-line restatement of the reference's per-rank programs
(``/root/reference/pkg/src/collectium/collectives.py:75-236`` and
``aggregation.py:138-176``) over an in-process transport with one OS thread
per rank: ``send`` copies the payload into the destination's FIFO for
(src, tag) and never blocks; ``recv`` blocks (transport/base.py:19-25). numpy
releases the GIL inside the element-wise kernels, so p ranks use up to p host
cores — this is the reference path as it would run on the box's host cores
(``bench.py`` CPU baseline and ``--impl reference``). Results are checked
bit-for-bit against the closed forms in ``oracle/collectives.py`` by the CPU
tests.
"""

from __future__ import annotations

import queue
import threading

import numpy as np

from . import collectives as C

TAG = 1


class ThreadTransport:
    def __init__(self, net: "ThreadNet", rank: int):
        self.net, self.rank, self.size = net, rank, net.size
        self.messages_sent = 0
        self.bytes_sent = 0

    def send(self, dst: int, payload: np.ndarray) -> None:
        self.messages_sent += 1
        self.bytes_sent += payload.nbytes
        self.net.box[(self.rank, dst)].put(payload.copy())          # tobytes() copy

    def recv(self, src: int) -> np.ndarray:
        return self.net.box[(src, self.rank)].get(timeout=600)


class ThreadNet:
    def __init__(self, size: int):
        self.size = size
        # every (src, dst) FIFO exists before the rank threads start: creating
        # them lazily from several threads (defaultdict) can lose a queue and
        # the message in it
        self.box = {(s, d): queue.Queue() for s in range(size) for d in range(size)}

    def run(self, fn):
        out = [None] * self.size
        err = []

        def body(r):
            try:
                out[r] = fn(r, ThreadTransport(self, r))
            except BaseException as exc:  # pragma: no cover
                err.append(exc)

        ths = [threading.Thread(target=body, args=(r,)) for r in range(self.size)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if err:
            raise err[0]
        return out


def _red(acc, incoming, op):
    """collectives.py:57-64"""
    return C.op2(acc, incoming, op)


def flat_rank(x: np.ndarray, op: str, tp: ThreadTransport) -> np.ndarray:
    """collectives.py:82-104"""
    p = tp.size
    if p == 1:
        return x
    if tp.rank == 0:
        acc = x.copy()
        for src in range(1, p):
            acc = _red(acc, tp.recv(src), op)
        for dst in range(1, p):
            tp.send(dst, acc)
        return acc
    tp.send(0, x)
    return tp.recv(0)


def ring_rank(x: np.ndarray, op: str, tp: ThreadTransport) -> np.ndarray:
    """collectives.py:107-152"""
    p, rank = tp.size, tp.rank
    if p == 1:
        return x
    chunks = C.chunk_partition(len(x), p)
    data = x.copy()
    left, right = (rank - 1) % p, (rank + 1) % p
    for step in range(p - 1):
        si, ri = (rank + step + 1) % p, (rank + step + 2) % p
        off, ln = chunks[si]
        tp.send(left, data[off:off + ln])
        incoming = tp.recv(right)
        off, ln = chunks[ri]
        data[off:off + ln] = _red(incoming, data[off:off + ln], op)
    for step in range(p - 1):
        si, ri = (rank + step) % p, (rank + step + 1) % p
        off, ln = chunks[si]
        tp.send(left, data[off:off + ln])
        incoming = tp.recv(right)
        off, ln = chunks[ri]
        data[off:off + ln] = incoming
    return data


def rhd_rank(x: np.ndarray, op: str, tp: ThreadTransport) -> np.ndarray:
    """collectives.py:155-236"""
    p, rank = tp.size, tp.rank
    if p == 1:
        return x
    m, excess, steps = C.rhd_params(p)
    data = x.copy()
    if rank < 2 * excess and rank % 2 == 1:
        tp.send(rank - 1, data)
        return tp.recv(rank - 1)
    if rank < 2 * excess:
        data = _red(data, tp.recv(rank + 1), op)
        vrank = rank // 2
    else:
        vrank = rank - excess
    lo, hi = 0, len(x)
    for k in range(steps):
        pv = vrank ^ (1 << k)
        partner = C.rhd_real(pv, p)
        mid = lo + (hi - lo) // 2
        if vrank < pv:
            s_lo, s_hi, k_lo, k_hi = mid, hi, lo, mid
        else:
            s_lo, s_hi, k_lo, k_hi = lo, mid, mid, hi
        tp.send(partner, data[s_lo:s_hi])
        incoming = tp.recv(partner)
        if vrank < pv:
            data[k_lo:k_hi] = _red(data[k_lo:k_hi], incoming, op)
        else:
            data[k_lo:k_hi] = _red(incoming, data[k_lo:k_hi], op)
        lo, hi = k_lo, k_hi
    for k in reversed(range(steps)):
        pv = vrank ^ (1 << k)
        partner = C.rhd_real(pv, p)
        tp.send(partner, data[lo:hi])
        incoming = tp.recv(partner)
        if vrank < pv:
            data[hi:hi + len(incoming)] = incoming
            hi += len(incoming)
        else:
            data[lo - len(incoming):lo] = incoming
            lo -= len(incoming)
    if rank < 2 * excess:
        tp.send(rank + 1, data)
    return data


_ALGO = {"flat": flat_rank, "ring_rsa": ring_rank, "rhd_rsa": rhd_rank}


def allreduce_rank(x, op, algo, tp, switch_bytes=C.DEFAULT_SWITCH_BYTES):
    concrete = C.resolve_algorithm(algo, x.nbytes, switch_bytes)
    return _ALGO[concrete](x, op, tp)


def aggregate_rank(grads: list[tuple[str, np.ndarray]], tp: ThreadTransport, algo="auto",
                   threshold=67108864, switch_bytes=C.DEFAULT_SWITCH_BYTES):
    """aggregation.py:138-176 for float32 gradients (negotiation is trivial:
    every rank holds the same names, so the sorted local list is the
    intersection)."""
    from .aggregation import fuse_plan
    p = tp.size
    lookup = dict(grads)
    names = sorted(lookup)
    mem = [(nm, "float32", lookup[nm].nbytes) for nm in names]
    out = {}
    for grp in fuse_plan(mem, threshold):
        gn = [names[i] for i in grp]
        payload = np.concatenate([lookup[nm] for nm in gn]) if len(gn) > 1 else lookup[gn[0]].copy()
        summed = allreduce_rank(payload, "sum", algo, tp, switch_bytes)
        mean = (summed.astype(np.float64) / p).astype(np.float32)
        off = 0
        for nm in gn:
            ln = len(lookup[nm])
            out[nm] = mean[off:off + ln]
            off += ln
    return out
