"""Generate golden fixtures by running the UNMODIFIED reference (build
container only; needs /root/reference and the greenlet shim in oracle/refshim).

    python tests/golden/gen_golden.py          # rewrites tests/golden/golden.json

Inputs are NOT stored: every case records the seed recipe, and tests rebuild
the inputs with numpy's default_rng (PCG64 + ziggurat normals, stable across
numpy >= 1.17). Outputs are stored as SHA-256 of the little-endian result
bytes (plus the full result for small cases) together with the reference's
CollectiveStats per rank.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402
from tests.golden import inputs as I  # noqa: E402

ref = reference.load()


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def run_allreduce(arrays, dtype, algo, op="sum", switch=None):
    p = len(arrays)
    group = ref.GroupSpec(p)
    rop = ref.ReduceOp.SUM if op == "sum" else ref.ReduceOp.MAX
    kw = {} if switch is None else {"switch_bytes": switch}

    def prog(rank, tp):
        out, st = ref.allreduce(ref.Tensor("x", dtype, arrays[rank]), rop, group, tp,
                                algo=algo, **kw)
        return out.to_bytes(), [st.rounds, st.messages_per_rank, st.bytes_sent_per_rank]

    res = reference.run_group(p, prog)
    outs = {r[0] for r in res}
    assert len(outs) == 1, "reference ranks disagree"
    return res[0][0], [r[1] for r in res]


def allreduce_cases():
    cases = []
    for dtype in ("float32", "float64"):
        for algo in ("flat", "ring_rsa", "rhd_rsa"):
            for p in range(1, 10):
                for n in I.SIZES:
                    arrays = I.allreduce_inputs(p, n, dtype, "sum")
                    out, st = run_allreduce(arrays, dtype, algo)
                    c = dict(kind="allreduce", dtype=dtype, algo=algo, p=p, n=n, op="sum",
                             sha=sha(out), stats=st)
                    if n <= 65:
                        c["hex"] = out.hex()
                    cases.append(c)
        # MAX with signed zeros / NaN payloads
        for algo in ("flat", "ring_rsa", "rhd_rsa"):
            for p in (2, 3, 4, 5, 6, 8):
                for n in (1, 7, 23, 64, 257):
                    arrays = I.allreduce_inputs(p, n, dtype, "max")
                    out, st = run_allreduce(arrays, dtype, algo, op="max")
                    cases.append(dict(kind="allreduce", dtype=dtype, algo=algo, p=p, n=n,
                                      op="max", sha=sha(out), stats=st, hex=out.hex()))
    # auto dispatch across the switch boundary (fp64: 16384 elements = 131072 B)
    for p in (2, 3, 4):
        for n in (16383, 16384):
            arrays = I.allreduce_inputs(p, n, "float64", "sum")
            out, st = run_allreduce(arrays, "float64", "auto")
            cases.append(dict(kind="allreduce", dtype="float64", algo="auto", p=p, n=n,
                              op="sum", sha=sha(out), stats=st))
    return cases


def c1_cases():
    """BASELINE config 1: 4 ranks, 1 MiB fp32, sum."""
    arrays = I.c1_inputs()
    out = []
    for algo in ("auto", "ring_rsa", "rhd_rsa", "flat"):
        res, st = run_allreduce(arrays, "float32", algo)
        out.append(dict(kind="c1", algo=algo, sha=sha(res), stats=st))
    return out


def aggregate_cases():
    cases = []
    for dtype in ("float32", "float64"):
        for p in (1, 2, 3, 4, 5, 8):
            schema = I.agg_schema(p)
            per_rank = I.agg_inputs(schema, p, dtype)
            for algo in ("auto", "ring_rsa", "rhd_rsa", "flat"):
                for thr in (1, 4096, 1 << 30):
                    group = ref.GroupSpec(p)

                    def prog(rank, tp):
                        gs = ref.GradientSet(tuple(ref.Tensor(nm, dtype, a)
                                                   for nm, a in per_rank[rank]))
                        stats = []
                        out = ref.aggregate(gs, group, tp, algo=algo,
                                            cfg=ref.FusionConfig(threshold_bytes=thr),
                                            stats_out=stats)
                        return ([t.name for t in out.tensors],
                                [t.to_bytes() for t in out.tensors],
                                [[s.rounds, s.messages_per_rank, s.bytes_sent_per_rank]
                                 for s in stats])

                    res = reference.run_group(p, prog)
                    assert all(r[1] == res[0][1] for r in res)
                    cases.append(dict(kind="aggregate", dtype=dtype, p=p, algo=algo,
                                      threshold=thr, names=res[0][0],
                                      sha=[sha(b) for b in res[0][1]],
                                      stats=[r[2] for r in res]))
    return cases


def model_cases():
    """BASELINE configs 4/5 gradient sets through the reference aggregate."""
    out = []
    models = ref.builtin_models()
    from collectium.bench import synth_gradients  # reference bench
    for model, p in (("mobilenet_like", 8), ("resnet50_like", 4)):
        spec = models[model]
        group = ref.GroupSpec(p)

        def prog(rank, tp):
            grads = synth_gradients(0, 0, spec, rank)
            stats = []
            res = ref.aggregate(grads, group, tp, stats_out=stats)
            h = hashlib.sha256()
            for t in res.tensors:
                h.update(t.to_bytes())
            return h.hexdigest(), len(stats)

        res = reference.run_group(p, prog)
        assert len({r[0] for r in res}) == 1
        out.append(dict(kind="model", model=model, p=p, seed=0, iteration=0,
                        sha=res[0][0], calls=res[0][1]))
    return out


def registry_cases():
    Policy, Kind = ref.Policy, ref.BufferKind
    cases = []
    for name, trace in I.registry_traces():
        for pol in ("no_cache", "lazy_cache", "intercept_cache"):
            reg = ref.BufferRegistry(Policy(pol))
            handles = {}
            answers = []
            for op in trace:
                try:
                    if op[0] == "alloc":
                        handles[op[1]] = reg.alloc(Kind(op[2]), op[3])
                    elif op[0] == "free":
                        reg.free(handles[op[1]])
                    else:
                        answers.append(reg.classify(handles[op[1]]).value)
                except ref.CollectiumError as exc:
                    answers.append(type(exc).__name__)
            cases.append(dict(kind="registry", trace=name, policy=pol,
                              answers=answers, stats=reg.stats_dict(),
                              addresses={str(k): h.address for k, h in handles.items()}))
    return cases


def main():
    data = dict(
        note="generated by tests/golden/gen_golden.py from the unmodified reference",
        numpy=np.__version__,
        cases=allreduce_cases() + c1_cases() + aggregate_cases() + model_cases()
        + registry_cases(),
    )
    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump(data, fh, separators=(",", ":"))
    print(f"wrote {len(data['cases'])} cases to {path}")


if __name__ == "__main__":
    main()
