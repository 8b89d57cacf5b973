"""Pin the CPU oracle against golden fixtures produced by the reference.

CPU-only (no GPU marker): the oracle restatement (oracle/) must reproduce the
reference's output bytes and CollectiveStats for every committed case before
it is trusted as the checker of the CUDA path.
"""

import hashlib

import numpy as np
import pytest

from oracle import aggregation as OA
from oracle import collectives as OC
from oracle import registry as OR
from tests.golden import inputs as I
from tests.golden.load import of_kind


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


ALLREDUCE = of_kind("allreduce")


@pytest.mark.parametrize("case", ALLREDUCE,
                         ids=[f"{c['dtype']}-{c['algo']}-{c['op']}-p{c['p']}-n{c['n']}"
                              for c in ALLREDUCE])
def test_allreduce_matches_reference(case):
    p, n, dtype, algo, op = case["p"], case["n"], case["dtype"], case["algo"], case["op"]
    xs = I.allreduce_inputs(p, n, dtype, op)
    out = OC.allreduce(xs, op, algo, dtype)
    assert _sha(out) == case["sha"]
    if "hex" in case:
        assert out.tobytes().hex() == case["hex"]
    for r in range(p):
        assert list(OC.stats(algo, p, n, dtype, r)) == case["stats"][r]


def test_c1_config_matches_reference():
    xs = I.c1_inputs()
    for case in of_kind("c1"):
        out = OC.allreduce(xs, "sum", case["algo"], "float32")
        assert _sha(out) == case["sha"], case["algo"]
        for r in range(4):
            assert list(OC.stats(case["algo"], 4, 262144, "float32", r)) == case["stats"][r]


AGG = of_kind("aggregate")


@pytest.mark.parametrize("case", AGG, ids=[f"{c['dtype']}-p{c['p']}-{c['algo']}-t{c['threshold']}"
                                           for c in AGG])
def test_aggregate_matches_reference(case):
    p, dtype = case["p"], case["dtype"]
    schema = I.agg_schema(p)
    per_rank = I.agg_inputs(schema, p, dtype)
    means, groups, algos = OA.aggregate(per_rank, dtype, case["algo"], case["threshold"])
    assert sorted(means) == case["names"]
    assert [_sha(means[nm]) for nm in case["names"]] == case["sha"]
    # one allreduce per fused buffer with the reference's per-call stats
    lens = dict(schema)
    for r in range(p):
        got = []
        for gnames, algo in zip(groups, algos):
            n = sum(lens[nm] for nm in gnames)
            got.append(list(OC.stats(algo, p, n, dtype, r)))
        assert got == case["stats"][r]
        assert len(groups) == len(case["stats"][r])


@pytest.mark.parametrize("case", of_kind("model"), ids=lambda c: c["model"])
def test_model_gradient_sets_match_reference(case):
    p = case["p"]
    layers = I.MODELS[case["model"]]
    per_rank = [I.synth_gradients(case["seed"], case["iteration"], layers, r) for r in range(p)]
    means, groups, _ = OA.aggregate(per_rank, "float32")
    h = hashlib.sha256()
    for nm in sorted(means):
        h.update(means[nm].tobytes())
    assert h.hexdigest() == case["sha"]
    assert len(groups) == case["calls"]


REG = of_kind("registry")


@pytest.mark.parametrize("case", REG, ids=[f"{c['trace']}-{c['policy']}" for c in REG])
def test_registry_replay_matches_reference(case):
    trace = dict(I.registry_traces())[case["trace"]]
    answers, st, addr = OR.replay(trace, case["policy"])
    assert answers == case["answers"]
    assert {"policy": case["policy"], **st} == case["stats"]
    assert {str(k): v for k, v in addr.items()} == case["addresses"]


def test_max_semantics_match_numpy():
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        a = rng.standard_normal(997).astype(dt)
        b = rng.standard_normal(997).astype(dt)
        a[::5], b[::5] = -0.0, 0.0
        a[::7] = np.nan
        b[1::11] = -np.nan
        a[2::13] = b[2::13]
        ref = np.maximum(a, b)
        got = OC.op2(a, b, "max")
        assert ref.tobytes() == got.tobytes()


def test_chunk_partition_examples():
    assert OC.chunk_partition(262144, 4) == [(0, 65536), (65536, 65536),
                                             (131072, 65536), (196608, 65536)]
    assert OC.chunk_partition(1, 8) == [(0, 1)] + [(1, 0)] * 7
    assert [o for o, _ in OC.chunk_partition(262145, 4)] == [0, 65537, 131073, 196609]


def test_rhd_layout_example():
    # p=8, n=64 bit-reversed ownership
    lay = OC.rhd_layout(64, 8)
    assert [lo for lo, _ in lay] == [0, 32, 16, 48, 8, 40, 24, 56]
    assert all(ln == 8 for _, ln in lay)


def test_int_and_bf16_extensions():
    rng = np.random.default_rng(5)
    for p in (1, 2, 3, 5, 8):
        xs = [rng.integers(-2**31, 2**31 - 1, size=77, dtype=np.int64).astype(np.int32)
              for _ in range(p)]
        want = np.sum(np.stack(xs).astype(np.int64), axis=0).astype(np.int32)  # wraps
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            assert np.array_equal(OC.allreduce(xs, "sum", algo, "int32"), want)
        xb = [OC.f32_to_bf16(rng.standard_normal(513).astype(np.float32)) for _ in range(p)]
        f64 = np.sum(np.stack([OC.bf16_to_f32(x).astype(np.float64) for x in xb]), axis=0)
        absum = np.sum(np.stack([np.abs(OC.bf16_to_f32(x)).astype(np.float64) for x in xb]), axis=0)
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            y = OC.bf16_to_f32(OC.allreduce(xb, "sum", algo, "bfloat16")).astype(np.float64)
            assert np.all(np.abs(y - f64) <= 1e-2 * absum + 1e-30)


def test_bf16_rounding_known_values():
    f = np.array([1.0, 1.00390625, 1.005859375, -2.5, np.inf, -np.inf, np.nan, 3.0e38],
                 dtype=np.float32)
    bits = OC.f32_to_bf16(f)
    assert bits[0] == 0x3F80
    assert bits[1] == 0x3F80          # tie -> even
    assert bits[2] == 0x3F81          # above tie -> up
    assert bits[3] == 0xC020
    assert bits[4] == 0x7F80 and bits[5] == 0xFF80 and bits[6] == 0x7FC0


def test_fuse_plan_reference_examples():
    # test_aggregation.py:71-92 (fp32 tensors of 16,16,48,128 bytes)
    mem = [(f"t{i}", "float32", b) for i, b in enumerate([16, 16, 48, 128])]
    assert OA.fuse_plan(mem, 64) == [[0, 1], [2], [3]]
    assert OA.fuse_plan(mem, 2**40) == [[0, 1, 2, 3]]
    assert OA.fuse_plan(mem[:3], 1) == [[0], [1], [2]]
    mixed = [("a", "float32", 8), ("b", "float64", 16)]
    assert OA.fuse_plan(mixed, 2**20) == [[0], [1]]


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_threaded_port_matches_closed_forms(p):
    """oracle/threaded.py (the CPU baseline / --impl reference path) is the
    reference's message-passing schedule; it must equal the closed forms."""
    from oracle import threaded as T
    for n in (0, 1, 7, 64, 1001):
        for dtype in ("float32", "float64"):
            xs = I.allreduce_inputs(p, n, dtype, "sum")
            for algo in ("flat", "ring_rsa", "rhd_rsa"):
                outs = T.ThreadNet(p).run(lambda r, tp: T.allreduce_rank(xs[r], "sum", algo, tp))
                want = OC.allreduce(xs, "sum", algo, dtype)
                for o in outs:
                    assert o.tobytes() == want.tobytes()


def test_threaded_aggregate_matches_reference_model_golden():
    from oracle import threaded as T
    case = [c for c in of_kind("model") if c["model"] == "mobilenet_like"][0]
    p = case["p"]
    layers = I.MODELS[case["model"]]
    grads = [I.synth_gradients(0, 0, layers, r) for r in range(p)]
    outs = T.ThreadNet(p).run(lambda r, tp: T.aggregate_rank(grads[r], tp))
    h = hashlib.sha256()
    for nm in sorted(outs[0]):
        h.update(outs[0][nm].tobytes())
    assert h.hexdigest() == case["sha"]
