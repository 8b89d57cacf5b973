"""Numpy restatement of the reference allreduce suite — TEST INFRASTRUCTURE.

Closed forms of the per-element fold order each reference algorithm produces
(SURVEY.md Appendix A), plus the reference's per-rank message/byte accounting.
Each function cites the reference lines it restates; all paths are relative to
``/root/reference/pkg/src/collectium/``.

Dtype extensions (the reference only accepts float32/float64, ``core.py:18-21``):
* ``int32``/``int64``: wrap-around sum, exact in any order.
* ``bfloat16`` (stored as uint16 bit patterns): every fold runs in float32 in the
  reference order and rounds ONCE to bfloat16 (round-to-nearest-even, NaN ->
  0x7FC0) at the end; partial sums are never stored in bfloat16
  (SURVEY.md §8c).
"""

from __future__ import annotations

import numpy as np

ALGORITHMS = ("flat", "ring_rsa", "rhd_rsa", "auto")          # collectives.py:20
DEFAULT_SWITCH_BYTES = 131072                                 # collectives.py:23

# storage dtype (wire bytes) and accumulation dtype per element type
STORAGE = {
    "float32": np.dtype("<f4"),
    "float64": np.dtype("<f8"),
    "bfloat16": np.dtype("<u2"),
    "int32": np.dtype("<i4"),
    "int64": np.dtype("<i8"),
}
ACCUM = {
    "float32": np.dtype("<f4"),
    "float64": np.dtype("<f8"),
    "bfloat16": np.dtype("<f4"),
    "int32": np.dtype("<i4"),
    "int64": np.dtype("<i8"),
}
FLOATS = ("float32", "float64", "bfloat16")


def itemsize(dtype: str) -> int:
    return STORAGE[dtype].itemsize


# -- element conversions -------------------------------------------------------

def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bits; NaN -> 0x7FC0."""
    x = np.asarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(np.isnan(x), np.uint16(0x7FC0), rounded).astype(np.uint16)


def to_acc(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bfloat16":
        return bf16_to_f32(x)
    return np.asarray(x, dtype=STORAGE[dtype])


def from_acc(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bfloat16":
        return f32_to_bf16(a)
    return np.asarray(a, dtype=STORAGE[dtype])


def op2(acc: np.ndarray, incoming: np.ndarray, op: str) -> np.ndarray:
    """``_reduce_arrays`` (collectives.py:57-64): ``acc`` is the first
    operand. SUM is IEEE/wrapping add; MAX is numpy ``maximum``, which is
    ``(a > b or isnan(a)) ? a : b`` bit for bit (NaN payloads and signed zeros
    included — verified against numpy 2.3 in tests)."""
    if op == "sum":
        with np.errstate(over="ignore"):
            return acc + incoming
    if op == "max":
        if acc.dtype.kind == "f":
            return np.where((acc > incoming) | np.isnan(acc), acc, incoming)
        return np.where(acc > incoming, acc, incoming)
    raise ValueError(f"unknown op {op!r}")


# -- layout helpers --------------------------------------------------------------

def chunk_partition(n: int, p: int) -> list[tuple[int, int]]:
    """core.py:113-130 — first ``n mod p`` chunks get one extra element."""
    if p < 1:
        raise ValueError(f"cannot partition over p={p} processes")
    if n < 0:
        raise ValueError(f"negative element count {n}")
    base, rem = divmod(n, p)
    out, off = [], 0
    for i in range(p):
        ln = base + (1 if i < rem else 0)
        out.append((off, ln))
        off += ln
    return out


def rhd_params(p: int) -> tuple[int, int, int]:
    """collectives.py:172-174: m = 2^floor(log2 p), excess, steps."""
    m = 1 << (p.bit_length() - 1)
    return m, p - m, m.bit_length() - 1


def rhd_vrank(rank: int, p: int) -> int | None:
    """collectives.py:180-192; None for folded odd ranks."""
    _, excess, _ = rhd_params(p)
    if rank < 2 * excess:
        return None if rank % 2 == 1 else rank // 2
    return rank - excess


def rhd_real(v: int, p: int) -> int:
    """collectives.py:194-195."""
    _, excess, _ = rhd_params(p)
    return 2 * v if v < excess else v + excess


def rhd_segment(vrank: int, n: int, p: int) -> tuple[int, int]:
    """Segment [lo, hi) vrank owns after recursive halving
    (collectives.py:198-216): bit k of vrank picks the upper half at step k."""
    _, _, steps = rhd_params(p)
    lo, hi = 0, n
    for k in range(steps):
        mid = lo + (hi - lo) // 2
        if (vrank >> k) & 1:
            lo = mid
        else:
            hi = mid
    return lo, hi


def rhd_layout(n: int, p: int) -> list[tuple[int, int]]:
    """Per REAL rank (offset, length) after the RHD reduce-scatter; folded odd
    ranks own nothing (offset 0, length 0)."""
    out = []
    for r in range(p):
        v = rhd_vrank(r, p)
        if v is None:
            out.append((0, 0))
        else:
            lo, hi = rhd_segment(v, n, p)
            out.append((lo, hi - lo))
    return out


def layout(kind: str, n: int, p: int) -> list[tuple[int, int]]:
    if kind in ("ring", "ring_rsa"):
        return chunk_partition(n, p)
    if kind in ("rhd", "rhd_rsa"):
        return rhd_layout(n, p)
    raise ValueError(f"unknown layout {kind!r}")


# -- fold orders (closed forms) ----------------------------

def _acc_all(xs, dtype):
    return [to_acc(np.asarray(x), dtype) for x in xs]


def ring_fold(xs_acc: list[np.ndarray], op: str) -> np.ndarray:
    """collectives.py:128-139: chunk c ends as fold(x_{c-1}, x_{c-2}, ..., x_c)
    (the travelling partial is the accumulator, local data folds in)."""
    p = len(xs_acc)
    n = len(xs_acc[0])
    out = np.empty(n, dtype=xs_acc[0].dtype)
    for c, (off, ln) in enumerate(chunk_partition(n, p)):
        sl = slice(off, off + ln)
        acc = xs_acc[(c - 1) % p][sl].copy()
        for k in range(2, p + 1):
            acc = op2(acc, xs_acc[(c - k) % p][sl], op)
        out[sl] = acc
    return out


def rhd_fold(xs_acc: list[np.ndarray], op: str) -> np.ndarray:
    """collectives.py:178-229: leaves L_v = x_{2v} op x_{2v+1} (v < excess) or
    x_{v+excess}; then a balanced tree, lower subtree as first operand."""
    p = len(xs_acc)
    m, excess, _ = rhd_params(p)
    leaves = []
    for v in range(m):
        if v < excess:
            leaves.append(op2(xs_acc[2 * v], xs_acc[2 * v + 1], op))
        else:
            leaves.append(xs_acc[v + excess].copy())
    s = 1
    while s < m:
        for v in range(0, m, 2 * s):
            leaves[v] = op2(leaves[v], leaves[v + s], op)
        s *= 2
    return leaves[0]


def flat_fold(xs_acc: list[np.ndarray], op: str) -> np.ndarray:
    """collectives.py:89-95: the root folds ranks 0..p-1 in order."""
    acc = xs_acc[0].copy()
    for x in xs_acc[1:]:
        acc = op2(acc, x, op)
    return acc


_FOLDS = {"ring_rsa": ring_fold, "rhd_rsa": rhd_fold, "flat": flat_fold}


def resolve_algorithm(algo: str, nbytes: int,
                      switch_bytes: int = DEFAULT_SWITCH_BYTES) -> str:
    """collectives.py:239-247."""
    if algo not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algo!r}")
    if algo != "auto":
        return algo
    if switch_bytes <= 0:
        raise ValueError("switch_bytes must be > 0 for auto dispatch")
    return "rhd_rsa" if nbytes < switch_bytes else "ring_rsa"


def allreduce_acc(xs, op: str, algo: str, dtype: str) -> np.ndarray:
    """Allreduce result in the ACCUMULATION dtype (before bf16 rounding)."""
    xs_acc = _acc_all(xs, dtype)
    lens = {len(x) for x in xs_acc}
    if len(lens) != 1:
        raise ValueError(f"ranks disagree on length: {sorted(lens)}")
    if len(xs_acc) == 1:
        return xs_acc[0].copy()
    return _FOLDS[algo](xs_acc, op)


def allreduce(xs, op: str = "sum", algo: str = "auto", dtype: str = "float32",
              switch_bytes: int = DEFAULT_SWITCH_BYTES) -> np.ndarray:
    """Every rank's (identical) allreduce output for inputs ``xs[rank]``
    (collectives.py:250-260). p=1 returns the input unchanged."""
    nbytes = len(xs[0]) * itemsize(dtype)
    concrete = resolve_algorithm(algo, nbytes, switch_bytes)
    if len(xs) == 1:
        return np.asarray(xs[0], dtype=STORAGE[dtype]).copy()
    return from_acc(allreduce_acc(xs, op, concrete, dtype), dtype)


def reduce_scatter(xs, op: str = "sum", layout_kind: str = "ring",
                   dtype: str = "float32") -> list[np.ndarray]:
    """Per-rank reduce-scatter outputs, pinned to the reference RS phases:
    ring (collectives.py:128-139) — rank r owns chunk r in ring fold order;
    rhd (:178-216) — vrank v owns its bit-reversed halving segment in tree
    order, folded odd ranks own nothing."""
    p = len(xs)
    n = len(xs[0])
    algo = "ring_rsa" if layout_kind in ("ring", "ring_rsa") else "rhd_rsa"
    full = from_acc(allreduce_acc(xs, op, algo, dtype), dtype)
    return [full[off:off + ln].copy() for off, ln in layout(layout_kind, n, p)]


def allgather(segments, n: int, layout_kind: str = "ring",
              dtype: str = "float32") -> np.ndarray:
    """Inverse of ``reduce_scatter``: rank r contributes its layout segment."""
    p = len(segments)
    out = np.zeros(n, dtype=STORAGE[dtype])
    for r, (off, ln) in enumerate(layout(layout_kind, n, p)):
        seg = np.asarray(segments[r], dtype=STORAGE[dtype])
        if len(seg) != ln:
            raise ValueError(f"rank {r} segment has {len(seg)} elements, layout says {ln}")
        out[off:off + ln] = seg
    return out


# -- per-rank logical accounting (CollectiveStats, collectives.py:28-47) ---------

def ring_stats(p: int, n: int, isz: int, rank: int) -> tuple[int, int, int]:
    """collectives.py:119-152: 2(p-1) rounds and messages; bytes are the sent
    chunk lengths (RS sends chunk r+s+1, AG sends chunk r+s)."""
    if p == 1:
        return (0, 0, 0)
    ch = chunk_partition(n, p)
    b = sum(ch[(rank + s + 1) % p][1] for s in range(p - 1))
    b += sum(ch[(rank + s) % p][1] for s in range(p - 1))
    return (2 * (p - 1), 2 * (p - 1), b * isz)


def _rhd_segments_all(n: int, p: int):
    """Trace every vrank's (lo, hi) through halving then doubling, collecting
    the per-vrank sent element counts (collectives.py:198-229)."""
    m, _, steps = rhd_params(p)
    seg = {v: (0, n) for v in range(m)}
    sent = {v: [] for v in range(m)}
    for k in range(steps):
        new = {}
        for v in range(m):
            lo, hi = seg[v]
            mid = lo + (hi - lo) // 2
            pv = v ^ (1 << k)
            if v < pv:
                sent[v].append(hi - mid)
                new[v] = (lo, mid)
            else:
                sent[v].append(mid - lo)
                new[v] = (mid, hi)
        seg = new
    for k in reversed(range(steps)):
        new = {}
        for v in range(m):
            lo, hi = seg[v]
            pv = v ^ (1 << k)
            plo, phi = seg[pv]
            sent[v].append(hi - lo)
            incoming = phi - plo
            new[v] = (lo, hi + incoming) if v < pv else (lo - incoming, hi)
        seg = new
    return sent


def rhd_stats(p: int, n: int, isz: int, rank: int) -> tuple[int, int, int]:
    """collectives.py:169-236 message/byte accounting incl. the fold phase."""
    if p == 1:
        return (0, 0, 0)
    _, excess, steps = rhd_params(p)
    rounds = 2 * steps + (2 if excess else 0)
    v = rhd_vrank(rank, p)
    if v is None:
        return (rounds, 1, n * isz)
    sent = _rhd_segments_all(n, p)[v]
    msgs, b = len(sent), sum(sent)
    if rank < 2 * excess:       # serve the folded partner (collectives.py:234-235)
        msgs += 1
        b += n
    return (rounds, msgs, b * isz)


def flat_stats(p: int, n: int, isz: int, rank: int) -> tuple[int, int, int]:
    """collectives.py:82-104."""
    if p == 1:
        return (0, 0, 0)
    if rank == 0:
        return (2, p - 1, (p - 1) * n * isz)
    return (2, 1, n * isz)


def stats(algo: str, p: int, n: int, dtype: str, rank: int,
          switch_bytes: int = DEFAULT_SWITCH_BYTES) -> tuple[int, int, int]:
    isz = itemsize(dtype)
    concrete = resolve_algorithm(algo, n * isz, switch_bytes)
    fn = {"ring_rsa": ring_stats, "rhd_rsa": rhd_stats, "flat": flat_stats}[concrete]
    return fn(p, n, isz, rank)


def reduce_scatter_stats(layout_kind: str, p: int, n: int, dtype: str,
                         rank: int) -> tuple[int, int, int]:
    """RS phase only: ring RS (collectives.py:128-139); rhd fold + halving
    (:180-216)."""
    isz = itemsize(dtype)
    if p == 1:
        return (0, 0, 0)
    if layout_kind in ("ring", "ring_rsa"):
        ch = chunk_partition(n, p)
        return (p - 1, p - 1, isz * sum(ch[(rank + s + 1) % p][1] for s in range(p - 1)))
    _, excess, steps = rhd_params(p)
    rounds = steps + (1 if excess else 0)
    v = rhd_vrank(rank, p)
    if v is None:
        return (rounds, 1, n * isz)
    sent = _rhd_segments_all(n, p)[v][:steps]
    return (rounds, steps, isz * sum(sent))


def allgather_stats(layout_kind: str, p: int, n: int, dtype: str,
                    rank: int) -> tuple[int, int, int]:
    """AG phase only: ring AG (collectives.py:142-150); rhd doubling + serving
    the folded partner (:219-235)."""
    isz = itemsize(dtype)
    if p == 1:
        return (0, 0, 0)
    if layout_kind in ("ring", "ring_rsa"):
        ch = chunk_partition(n, p)
        return (p - 1, p - 1, isz * sum(ch[(rank + s) % p][1] for s in range(p - 1)))
    _, excess, steps = rhd_params(p)
    rounds = steps + (1 if excess else 0)
    v = rhd_vrank(rank, p)
    if v is None:
        return (rounds, 0, 0)
    sent = _rhd_segments_all(n, p)[v][steps:]
    msgs, b = len(sent), sum(sent)
    if rank < 2 * excess:
        msgs += 1
        b += n
    return (rounds, msgs, isz * b)
