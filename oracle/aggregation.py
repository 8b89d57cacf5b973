"""Numpy restatement of tensor fusion + averaging — TEST INFRASTRUCTURE.

Restates ``/root/reference/pkg/src/collectium/aggregation.py``:
negotiation order (:72-92), greedy fusion (:95-130) and the post-allreduce mean
(:167-174).  Inputs are given for all ranks at once (``per_rank[rank]`` is a
list of ``(name, array)``), since the oracle simulates the whole group.
"""

from __future__ import annotations

import numpy as np

from . import collectives as C

DEFAULT_FUSION_THRESHOLD = 67108864                           # aggregation.py:25


def negotiate(per_rank_names: list[list[str]]) -> list[str]:
    """aggregation.py:72-92: sorted intersection of all ranks' ready names."""
    common = set(per_rank_names[0])
    for names in per_rank_names[1:]:
        common &= set(names)
    return sorted(common)


def fuse_plan(members: list[tuple[str, str, int]], threshold: int) -> list[list[int]]:
    """aggregation.py:95-130 greedy first-fit. ``members`` = (name, dtype,
    nbytes) in canonical order; returns groups of member indices."""
    if threshold <= 0:
        raise ValueError("fusion threshold must be positive")
    groups: list[list[int]] = []
    cur: list[int] = []
    cur_bytes = 0
    cur_dtype = None
    for i, (_, dtype, nbytes) in enumerate(members):
        if cur and (cur_dtype != dtype or cur_bytes + nbytes > threshold):
            groups.append(cur)
            cur, cur_bytes = [], 0
        if not cur:
            cur_dtype = dtype
        cur.append(i)
        cur_bytes += nbytes
        if cur_bytes >= threshold:
            groups.append(cur)
            cur, cur_bytes = [], 0
    if cur:
        groups.append(cur)
    return groups


def mean_from_acc(s_acc: np.ndarray, p: int, dtype: str) -> np.ndarray:
    """aggregation.py:167-172. float32: float32(float64(s)/p) — identical to
    IEEE float32 s/(float)p; float64: s/p. bfloat16 (extension): the float32
    accumulator divided by (float)p, rounded once to bfloat16."""
    if dtype == "float32":
        return (s_acc.astype(np.float64) / p).astype(np.float32)
    if dtype == "float64":
        return s_acc / p
    if dtype == "bfloat16":
        return C.f32_to_bf16(s_acc / np.float32(p))
    raise ValueError(f"aggregate averages float tensors only, got {dtype}")


def aggregate(per_rank: list[list[tuple[str, np.ndarray]]], dtype: str,
              algo: str = "auto", threshold: int = DEFAULT_FUSION_THRESHOLD,
              switch_bytes: int = C.DEFAULT_SWITCH_BYTES):
    """aggregation.py:138-176. Returns (means: dict name -> array,
    groups: list of member-name lists, per-group concrete algorithm)."""
    p = len(per_rank)
    names = negotiate([[nm for nm, _ in g] for g in per_rank])
    lookup = [dict(g) for g in per_rank]
    isz = C.itemsize(dtype)
    members = [(nm, dtype, len(lookup[0][nm]) * isz) for nm in names]
    out: dict[str, np.ndarray] = {}
    groups_out, algos = [], []
    for group in fuse_plan(members, threshold):
        gnames = [names[i] for i in group]
        fused = [np.concatenate([np.asarray(lookup[r][nm]) for nm in gnames])
                 if len(gnames) > 1 else np.asarray(lookup[r][gnames[0]]).copy()
                 for r in range(p)]
        nbytes = len(fused[0]) * isz
        concrete = C.resolve_algorithm(algo, nbytes, switch_bytes)
        if p == 1:
            s_acc = C.to_acc(fused[0], dtype)
        else:
            s_acc = C.allreduce_acc(fused, "sum", concrete, dtype)
        mean = mean_from_acc(s_acc, p, dtype)
        off = 0
        for nm in gnames:
            ln = len(lookup[0][nm])
            out[nm] = mean[off:off + ln]
            off += ln
        groups_out.append(gnames)
        algos.append(concrete)
    return out, groups_out, algos
