"""Deterministic input recipes shared by the golden generator and the tests.

Pure numpy; no reference import, so it works on the GPU box too.
"""

from __future__ import annotations

import numpy as np

SIZES = (0, 1, 2, 3, 5, 7, 8, 17, 33, 64, 65, 1000, 4099)

_STORE = {"float32": np.float32, "float64": np.float64}


def allreduce_inputs(p: int, n: int, dtype: str, op: str = "sum", seed: int = 7):
    """Scaled normals spanning 10^-3..10^3 so fold order shows up in the bits;
    for op="max" also plant signed zeros, ties and NaN payloads."""
    out = []
    for r in range(p):
        rng = np.random.default_rng([seed, p, n, r, 0 if op == "sum" else 1])
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)
        x = x.astype(_STORE[dtype])
        if op == "max" and n:
            x[::5] = 0.0 if r % 2 else -0.0
            x[1::7] = -0.0 if r % 2 else 0.0
            if dtype == "float32":
                nan = np.array([0x7FC00000 | (r + 1), 0xFFC00000 | (r + 9)], np.uint32).view(np.float32)
            else:
                nan = np.array([0x7FF8000000000000 | (r + 1), 0xFFF8000000000000 | (r + 9)],
                               np.uint64).view(np.float64)
            x[(2 + r) % n::11] = nan[0]
            x[(3 + 2 * r) % n::13] = nan[1]
            x[4::17] = 1.5  # ties across ranks
        out.append(x)
    return out


def c1_inputs():
    """BASELINE config 1: default_rng([0, 1048576, rank])
    standard normals, 262144 fp32 per rank, 4 ranks."""
    return [np.random.default_rng([0, 1048576, r]).standard_normal(262144, dtype=np.float32)
            for r in range(4)]


def agg_schema(p: int):
    """Ragged gradient schema (names deliberately out of lexicographic order)."""
    rng = np.random.default_rng([17, p])
    lens = [int(v) for v in rng.integers(1, 400, size=23)]
    lens[3] = 0 + 5          # small
    lens[7] = 1029           # > 4096 B at fp32 -> singleton groups at threshold 4096
    names = [f"g{(i * 7) % 23:02d}" for i in range(23)]
    return list(zip(names, lens))


def agg_inputs(schema, p: int, dtype: str):
    per_rank = []
    for r in range(p):
        tensors = []
        for i, (nm, n) in enumerate(schema):
            rng = np.random.default_rng([17, i, r])
            tensors.append((nm, rng.standard_normal(n).astype(_STORE[dtype])))
        per_rank.append(tensors)
    return per_rank


def synth_gradients(seed: int, iteration: int, layer_elems, rank: int):
    """Same recipe as the reference bench (bench.py:224-232):
    default_rng([seed, iteration, layer, rank]).standard_normal(n, float32)."""
    out = []
    for idx, n in enumerate(layer_elems):
        rng = np.random.default_rng([seed, iteration, idx, rank])
        out.append((f"layer{idx:04d}", rng.standard_normal(n, dtype=np.float32)))
    return out


MODELS = {
    # simcost.py:152-163 builtin_models: n_layers x layer_bytes (fp32)
    "mobilenet_like": [600_000 // 4] * 28,
    "resnet50_like": [1_920_000 // 4] * 53,
}


def criterion3_trace():
    """test_acceptance.py:108-135 scripted 1000-op trace (kinds as strings)."""
    rng = np.random.default_rng(42)
    ops, live, nxt = [], [], 0
    while len(ops) < 1000:
        roll = rng.integers(0, 10)
        if roll < 4 or not live or len(ops) >= 998:
            if len(ops) >= 998 and live:
                ops.append(("classify", live[int(rng.integers(len(live)))]))
                continue
            kind = "host" if rng.integers(2) else "device"
            ops.append(("alloc", nxt, kind, int(rng.integers(1, 4096))))
            ops.append(("classify", nxt))
            live.append(nxt)
            nxt += 1
        elif roll < 6 and len(live) > 1:
            idx = live.pop(int(rng.integers(len(live))))
            ops.append(("free", idx))
        else:
            ops.append(("classify", live[int(rng.integers(len(live)))]))
    return ops


def random_trace(seed: int, length: int):
    rng = np.random.default_rng([99, seed])
    ops, live, nxt = [], [], 0
    for _ in range(length):
        c = int(rng.integers(0, 4))
        if c == 0 or not live:
            ops.append(("alloc", nxt, "host" if rng.integers(2) else "device",
                        int(rng.integers(1, 4096))))
            live.append(nxt)
            nxt += 1
        elif c == 1:
            idx = live.pop(int(rng.integers(len(live))))
            ops.append(("free", idx))
            if rng.integers(4) == 0:
                ops.append(("free", idx))  # double free -> InvalidHandleError
        else:
            ops.append(("classify", live[int(rng.integers(len(live)))]))
    return ops


def staleness_trace():
    return [("alloc", 0, "host", 64), ("classify", 0), ("free", 0),
            ("alloc", 1, "device", 64), ("classify", 1)]


def registry_traces():
    out = [("criterion3", criterion3_trace()), ("staleness", staleness_trace())]
    for s in range(6):
        out.append((f"random{s}", random_trace(s, 150)))
    return out
