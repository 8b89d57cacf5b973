"""The oracle against the LIVE reference (build container only: needs
/root/reference and the greenlet shim in oracle/refshim; skipped elsewhere).

Random cases beyond the committed golden grid — group sizes, lengths,
value scales, algorithms, fusion thresholds — run through the unmodified
reference package and through the numpy restatement in oracle/; results must
be bit-identical, stats equal.
"""

import os

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")


@pytest.fixture(scope="module")
def ref():
    from oracle import reference
    return reference


def _run(reference, p, prog):
    return reference.run_group(p, prog)


@pytest.mark.parametrize("seed", range(12))
def test_random_allreduce_cases_bit_identical(ref, seed):
    from oracle import collectives as OC
    R = ref.load()
    rng = np.random.default_rng([2026, seed])
    p = int(rng.integers(1, 10))
    n = int(rng.integers(0, 40_000))
    dtype = ("float32", "float64")[seed % 2]
    algo = ("flat", "ring_rsa", "rhd_rsa", "auto")[seed % 4]
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(dtype) for _ in range(p)]

    def prog(rank, tp):
        out, st = R.allreduce(R.Tensor("x", dtype, xs[rank]), R.ReduceOp.SUM, R.GroupSpec(p), tp, algo=algo)
        return out.to_bytes(), (st.rounds, st.messages_per_rank, st.bytes_sent_per_rank)

    res = _run(ref, p, prog)
    want = OC.allreduce(xs, "sum", algo, dtype).tobytes()
    for r, (out, st) in enumerate(res):
        assert out == want, (p, n, algo, r)
        assert st == OC.stats(algo, p, n, dtype, r)


@pytest.mark.parametrize("seed", range(4))
def test_random_aggregate_cases_bit_identical(ref, seed):
    from oracle import aggregation as OA
    R = ref.load()
    rng = np.random.default_rng([77, seed])
    p = int(rng.integers(2, 7))
    lens = [int(x) for x in rng.integers(1, 30_000, size=int(rng.integers(3, 12)))]
    thr = int(rng.choice([4096, 65536, 1 << 20]))
    per_rank = [[(f"g{i:03d}", rng.standard_normal(n).astype(np.float32)) for i, n in enumerate(lens)]
                for _ in range(p)]

    def prog(rank, tp):
        gs = R.GradientSet(tuple(R.Tensor(nm, "float32", a) for nm, a in per_rank[rank]))
        res = R.aggregate(gs, R.GroupSpec(p), tp, cfg=R.FusionConfig(thr))
        return {t.name: t.to_bytes() for t in res.tensors}

    res = _run(ref, p, prog)
    want, _, _ = OA.aggregate(per_rank, "float32", "auto", thr)
    for out in res:
        assert out.keys() == want.keys()
        assert all(out[k] == want[k].tobytes() for k in out)
