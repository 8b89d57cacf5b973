"""GPU parity tier on ONE B200: p virtual ranks per cooperative launch.

The same collective kernels, flag protocol, staging and fold orders as the
multi-GPU path run here with every rank's CTAs in one launch
(VirtualGroup). Results are compared with the reference golden fixtures
(float32/float64: bit-exact SHA-256 of the output bytes) and with the CPU
oracle (bf16, ints, large sizes).

Tolerances (BASELINE north_star / SURVEY §8c): fp32/fp64 and ints are
bit-exact (the kernels replay the reference fold order); bf16 accumulates in
fp32 and must be bit-identical to the oracle's fp32-fold-then-round, and
within 1e-2 * sum|x| of the fp64 sum.
"""

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1810_11112_b200 as P  # noqa: E402
from oracle import aggregation as OA  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from tests.golden import inputs as I  # noqa: E402
from tests.golden.load import of_kind  # noqa: E402

OPS = {"sum": P.ReduceOp.SUM, "max": P.ReduceOp.MAX}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


_VG = {}


def vg(p):
    if p not in _VG:
        _VG[p] = P.VirtualGroup(p, 0, staging_bytes=128 << 20, timeout_s=5.0)
    return _VG[p]


def dev_tensors(arrays, dtype):
    return [P.Tensor(f"r{r}", dtype, torch.from_numpy(np.ascontiguousarray(a)).cuda())
            for r, a in enumerate(arrays)]


ALLREDUCE = of_kind("allreduce")


@pytest.mark.parametrize("case", ALLREDUCE,
                         ids=[f"{c['dtype']}-{c['algo']}-{c['op']}-p{c['p']}-n{c['n']}"
                              for c in ALLREDUCE])
def test_allreduce_bit_exact_vs_reference_golden(case):
    p, n, dtype, algo, op = case["p"], case["n"], case["dtype"], case["algo"], case["op"]
    arrays = I.allreduce_inputs(p, n, dtype, op)
    res = P.allreduce_group(dev_tensors(arrays, dtype), OPS[op], vg(p), algo=algo)
    outs = [t.to_bytes() for t, _ in res]
    assert len(set(outs)) == 1, "ranks differ"
    assert sha(outs[0]) == case["sha"]
    for r, (_, st) in enumerate(res):
        assert [st.rounds, st.messages_per_rank, st.bytes_sent_per_rank] == case["stats"][r]


def test_c1_config_bit_exact():
    xs = I.c1_inputs()
    for case in of_kind("c1"):
        res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, vg(4), algo=case["algo"])
        for t, _ in res:
            assert sha(t.to_bytes()) == case["sha"], case["algo"]


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("algo", ["ring_rsa", "rhd_rsa", "flat"])
@pytest.mark.parametrize("n", [262145, 1 << 20, 3_000_001])
def test_large_fp32_vs_oracle(p, algo, n):
    rng = np.random.default_rng([p, n])
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32)
          for _ in range(p)]
    want = OC.allreduce(xs, "sum", algo, "float32")
    res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, vg(p), algo=algo)
    for t, _ in res:
        assert t.to_bytes() == want.tobytes()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", ["ring_rsa", "rhd_rsa"])
def test_pipelined_two_shot_vs_oracle(p, algo):
    """Large messages take the pipelined two-shot (reducer/gather warps with
    per-warp progress flags); force small chunks so every CTA runs many."""
    g = vg(p)
    n = 6_000_007
    rng = np.random.default_rng([p, 99])
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32)
          for _ in range(p)]
    want = OC.allreduce(xs, "sum", algo, "float32")
    for chunk in (1024, 8192):
        g.set_param("stream_chunk", chunk)
        res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, g, algo=algo)
        for t, _ in res:
            assert t.to_bytes() == want.tobytes(), chunk
    g.set_param("stream_chunk", 1)   # back to the default (off)


_VGL = {}


def vg_logp(p):
    """A virtual group whose rhd_rsa runs the literal log2(p)-step recursive
    halving/doubling kernel (pairwise flags) instead of the direct kernels."""
    if p not in _VGL:
        g = P.VirtualGroup(p, 0, staging_bytes=128 << 20, timeout_s=5.0)
        g.set_param("rhd_logp", 2)
        _VGL[p] = g
    return _VGL[p]


RHD_GOLDEN = [c for c in ALLREDUCE if c["algo"] == "rhd_rsa"]


@pytest.mark.parametrize("case", RHD_GOLDEN,
                         ids=[f"{c['dtype']}-{c['op']}-p{c['p']}-n{c['n']}" for c in RHD_GOLDEN])
def test_rhd_logp_kernel_bit_exact_vs_reference_golden(case):
    p, n, dtype, op = case["p"], case["n"], case["dtype"], case["op"]
    arrays = I.allreduce_inputs(p, n, dtype, op)
    res = P.allreduce_group(dev_tensors(arrays, dtype), OPS[op], vg_logp(p), algo="rhd_rsa")
    for r, (t, st) in enumerate(res):
        assert sha(t.to_bytes()) == case["sha"], r
        assert [st.rounds, st.messages_per_rank, st.bytes_sent_per_rank] == case["stats"][r]


@pytest.mark.parametrize("p", [2, 3, 5, 6, 7, 8, 12, 16])
@pytest.mark.parametrize("n", [1, 1000, 262145, 3_000_001])
def test_rhd_logp_kernel_vs_oracle(p, n):
    rng = np.random.default_rng([p, n, 5])
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32)
          for _ in range(p)]
    want = OC.allreduce(xs, "sum", "rhd_rsa", "float32")
    g = vg_logp(p)
    for _ in range(2):                     # both staging parities
        res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, g, algo="rhd_rsa")
        for t, _ in res:
            assert t.to_bytes() == want.tobytes()
    ints = [rng.integers(-2**31, 2**31 - 1, size=n, dtype=np.int64) for _ in range(p)]
    res = P.allreduce_group(dev_tensors(ints, "int64"), P.ReduceOp.SUM, g, algo="rhd_rsa")
    want = OC.allreduce(ints, "sum", "rhd_rsa", "int64")
    for t, _ in res:
        assert t.to_bytes() == want.tobytes()


@pytest.mark.parametrize("dtype", ["int32", "int64"])
@pytest.mark.parametrize("p", [2, 3, 7, 8])
def test_int_bit_exact(dtype, p):
    rng = np.random.default_rng([11, p])
    info = np.iinfo(dtype)
    for n in (1, 7, 65, 100_003):
        xs = [rng.integers(info.min, info.max, size=n, dtype=dtype) for _ in range(p)]
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            want = OC.allreduce(xs, "sum", algo, dtype)
            for op in ("sum", "max"):
                want = OC.allreduce(xs, op, algo, dtype)
                res = P.allreduce_group(dev_tensors(xs, dtype), OPS[op], vg(p), algo=algo)
                assert res[0][0].to_bytes() == want.tobytes()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_bf16_matches_oracle_and_tolerance(p):
    rng = np.random.default_rng([13, p])
    for n in (1, 9, 4097, 500_001):
        xs = [OC.f32_to_bf16(rng.standard_normal(n).astype(np.float32)) for _ in range(p)]
        f64 = np.sum([OC.bf16_to_f32(x).astype(np.float64) for x in xs], axis=0)
        absum = np.sum([np.abs(OC.bf16_to_f32(x)).astype(np.float64) for x in xs], axis=0)
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            want = OC.allreduce(xs, "sum", algo, "bfloat16")
            tens = [P.Tensor(f"r{r}", "bfloat16", torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda())
                    for r, x in enumerate(xs)]
            res = P.allreduce_group(tens, P.ReduceOp.SUM, vg(p), algo=algo)
            got = np.frombuffer(res[0][0].to_bytes(), dtype=np.uint16)
            assert np.array_equal(got, want), algo
            y = OC.bf16_to_f32(got).astype(np.float64)
            assert np.all(np.abs(y - f64) <= 1e-2 * absum + 1e-30)   # stated bf16 tolerance


@pytest.mark.parametrize("layout", ["ring", "rhd"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 8])
def test_reduce_scatter_and_allgather(layout, p):
    for n in (0, 1, 5, 64, 1000, 65537):
        xs = I.allreduce_inputs(p, n, "float32", "sum")
        want = OC.reduce_scatter(xs, "sum", layout, "float32")
        res = P.reduce_scatter_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, vg(p), layout=layout)
        for r, (t, st) in enumerate(res):
            assert t.to_bytes() == want[r].tobytes(), (r, n)
            assert (st.rounds, st.messages_per_rank, st.bytes_sent_per_rank) == \
                OC.reduce_scatter_stats(layout, p, n, "float32", r)
        segs = [P.Tensor(f"s{r}", "float32", t.payload) for r, (t, _) in enumerate(res)]
        full = OC.allgather(want, n, layout, "float32")
        gathered = P.allgather_group(segs, n, vg(p), layout=layout)
        for r, (t, st) in enumerate(gathered):
            assert t.to_bytes() == full.tobytes()
            assert (st.rounds, st.messages_per_rank, st.bytes_sent_per_rank) == \
                OC.allgather_stats(layout, p, n, "float32", r)


AGG = of_kind("aggregate")


@pytest.mark.parametrize("case", AGG, ids=[f"{c['dtype']}-p{c['p']}-{c['algo']}-t{c['threshold']}"
                                           for c in AGG])
def test_aggregate_bit_exact_vs_reference_golden(case):
    p, dtype = case["p"], case["dtype"]
    schema = I.agg_schema(p)
    per_rank = I.agg_inputs(schema, p, dtype)
    sets = [P.GradientSet(tuple(P.Tensor(nm, dtype, torch.from_numpy(a).cuda()) for nm, a in g))
            for g in per_rank]
    stats = []
    outs = P.aggregate_group(sets, vg(p), algo=case["algo"],
                             cfg=P.FusionConfig(case["threshold"]), stats_out=stats)
    for r in range(p):
        assert outs[r].names == case["names"]
        assert [sha(t.to_bytes()) for t in outs[r].tensors] == case["sha"]
        assert [[s.rounds, s.messages_per_rank, s.bytes_sent_per_rank] for s in stats[r]] == case["stats"][r]


@pytest.mark.parametrize("case", of_kind("model"), ids=lambda c: c["model"])
def test_model_gradient_sets_bit_exact(case):
    p = case["p"]
    layers = I.MODELS[case["model"]]
    sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                for nm, a in I.synth_gradients(0, 0, layers, r)))
            for r in range(p)]
    outs = P.aggregate_group(sets, vg(p))
    for r in range(p):
        h = hashlib.sha256()
        for t in outs[r].tensors:
            h.update(t.to_bytes())
        assert h.hexdigest() == case["sha"]


def test_bf16_aggregate_matches_oracle():
    p = 4
    schema = I.agg_schema(p)
    per_rank = I.agg_inputs(schema, p, "float32")
    bf = [[(nm, OC.f32_to_bf16(a)) for nm, a in g] for g in per_rank]
    want, _, _ = OA.aggregate(bf, "bfloat16", "auto", 4096)
    sets = [P.GradientSet(tuple(P.Tensor(nm, "bfloat16", torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda())
                                for nm, a in g)) for g in bf]
    outs = P.aggregate_group(sets, vg(p), cfg=P.FusionConfig(4096))
    for t in outs[0].tensors:
        assert np.array_equal(np.frombuffer(t.to_bytes(), np.uint16), want[t.name])


def test_back_to_back_epochs_and_graph_capture():
    """Epoch/parity reuse: many consecutive calls with changing sizes and
    algorithms, then the same call replayed from a CUDA graph."""
    p = 4
    g = vg(p)
    rng = np.random.default_rng(5)
    for it in range(60):
        n = int(rng.integers(0, 70000))
        algo = ("ring_rsa", "rhd_rsa", "flat", "auto")[it % 4]
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        want = OC.allreduce(xs, "sum", algo, "float32")
        res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, g, algo=algo)
        assert res[0][0].to_bytes() == want.tobytes()
    # CUDA graph: epochs advance on the device, so replays stay correct
    import ctypes as C
    from paper_1810_11112_b200 import _lib as L
    n = 40000
    xs = [torch.randn(n, device="cuda") for _ in range(p)]
    outs = [torch.empty_like(x) for x in xs]
    st = (L.Stats * p)()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for _ in range(3):
                L.check(L.lib.cm_allreduce_v(g._h, L.ptr_array([x.data_ptr() for x in xs]),
                                             L.ptr_array([o.data_ptr() for o in outs]), n,
                                             L.DTYPE["float32"], 0, L.ALGO["ring_rsa"], 131072, 0,
                                             s.cuda_stream, st))
    for _ in range(5):
        for x in xs:
            x.normal_()
        graph.replay()
        torch.cuda.synchronize()
        g.poll()
        want = OC.allreduce([x.cpu().numpy() for x in xs], "sum", "ring_rsa", "float32")
        for o in outs:
            assert o.cpu().numpy().tobytes() == want.tobytes()
    del C


def test_local_reduce_and_batched_copy():
    rng = np.random.default_rng(9)
    for dtype in ("float32", "float64", "int32"):
        for n in (1, 3, 1000, 100_001):
            a = rng.standard_normal(n).astype(dtype) if "float" in dtype else rng.integers(-9, 9, n).astype(dtype)
            b = rng.standard_normal(n).astype(dtype) if "float" in dtype else rng.integers(-9, 9, n).astype(dtype)
            for op in ("sum", "max"):
                got = P.local_reduce(P.Tensor("a", dtype, torch.from_numpy(a).cuda()),
                                     P.Tensor("b", dtype, torch.from_numpy(b).cuda()), OPS[op])
                assert got.to_bytes() == OC.op2(a, b, op).tobytes()
    # host payloads are staged through the device and come back on the host
    got = P.local_reduce(P.Tensor("a", "float64", [1.0, 2.0]), P.Tensor("b", "float64", [3.0, 4.0]),
                         P.ReduceOp.SUM)
    assert not got.is_cuda and got.numpy().tolist() == [4.0, 6.0]
    # fuse()/unfuse() on device tensors = one batched-copy launch
    ts = [P.Tensor(f"t{i}", "float32", torch.randn(n, device="cuda")) for i, n in enumerate((5, 1, 64, 1023, 4))]
    (buf,) = P.fuse(ts, P.FusionConfig(1 << 30))
    assert torch.equal(buf.payload, torch.cat([t.payload for t in ts]))
    for a, b in zip(ts, P.unfuse(buf)):
        assert torch.equal(a.payload, b.payload)


@pytest.mark.parametrize("sizes", [(480_000,) * 53, (65_536, 4, 1_000_000, 262_144), (1_000_003, 77, 5, 999_999)])
def test_large_fuse_unfuse_bulk_and_sm_copy(sizes):
    """Large packs: 16-byte aligned members go through the TMA bulk-copy
    kernel, others through the SM copy; both must equal torch.cat."""
    ts = [P.Tensor(f"t{i:03d}", "float32", torch.randn(n, device="cuda")) for i, n in enumerate(sizes)]
    (buf,) = P.fuse(ts, P.FusionConfig(1 << 40))
    assert torch.equal(buf.payload, torch.cat([t.payload for t in ts]))
    for a, b in zip(ts, P.unfuse(buf)):
        assert torch.equal(a.payload, b.payload)


def test_p1_identity_and_errors():
    x = torch.randn(17, device="cuda")
    (t, st), = P.allreduce_group([P.Tensor("x", "float32", x)], P.ReduceOp.SUM, vg(1))
    assert torch.equal(t.payload, x) and (st.rounds, st.messages_per_rank) == (0, 0)
    with pytest.raises(P.ShapeError):
        P.allreduce_group([P.Tensor("x", "float32", torch.zeros(3 + r, device="cuda")) for r in range(2)],
                          P.ReduceOp.SUM, vg(2))
    with pytest.raises(P.ConfigError):
        P.allreduce_group([P.Tensor("x", "float32", torch.zeros(3, device="cuda"))] * 2,
                          P.ReduceOp.SUM, vg(2), algo="tree")
    with pytest.raises(P.ConfigError):
        P.allreduce_group([P.Tensor("x", "float32", torch.zeros(3, device="cuda"))] * 2,
                          P.ReduceOp.SUM, vg(2), switch_bytes=0)


def test_single_rank_communicator_aggregate_host_and_device():
    """p = 1 real communicator (BASELINE C5 at N=1): device gradients -> one
    batched copy; pinned / pageable / mixed host gradients -> chunked H2D + D2H
    on the copy streams into pinned host buckets (refilled with out=)."""
    comm = P.Communicator(rank=0, size=1, device=0, staging_bytes=64 << 20, pool_bytes=2 << 20)
    layers = [480_000] * 40 + [1_000_003, 77]
    g = I.synth_gradients(0, 0, layers, 0)
    flat = torch.empty(sum(a.size for _, a in g), dtype=torch.float32).pin_memory()
    for kind in ("device", "pinned", "pageable", "mixed", "flat"):
        def mk(scale):
            ts, off = [], 0
            for i, (nm, a) in enumerate(g):
                x = torch.from_numpy(a * scale)
                if kind == "device" or (kind == "mixed" and i % 3 == 0):
                    x = x.cuda()
                elif kind in ("pinned", "mixed"):
                    x = x.pin_memory()
                elif kind == "flat":              # views of one pinned buffer: coalesced copies
                    v = flat[off:off + a.size]
                    v.copy_(x)
                    x = v
                off += a.size
                ts.append(P.Tensor(nm, "float32", x))
            return P.GradientSet(tuple(ts))
        res = P.aggregate(mk(1), P.GroupSpec(1), comm)
        assert all(t.to_bytes() == (a * 1).tobytes() for t, (_, a) in zip(res.tensors, sorted(g)))
        res2 = P.aggregate(mk(3), P.GroupSpec(1), comm, out=res)
        assert res2 is res
        assert all(t.to_bytes() == (a * 3).tobytes() for t, (_, a) in zip(res.tensors, sorted(g)))
        assert all(t.is_cuda == (kind == "device") for t in res.tensors)
    # graded pipeline pieces (ramped at both ends) for other piece sizes and a
    # total below one piece (eight even pieces)
    for chunk_kb, lay in ((64, layers), (1024, [77, 1000, 3]), (8192, [5, 300_000])):
        comm.set_param("host_chunk_kb", chunk_kb)
        gg = I.synth_gradients(1, 0, lay, 0)
        fl = torch.empty(sum(a.size for _, a in gg), dtype=torch.float32).pin_memory()
        ts, off = [], 0
        for nm, a in gg:
            v = fl[off:off + a.size]
            v.copy_(torch.from_numpy(a))
            ts.append(P.Tensor(nm, "float32", v))
            off += a.size
        res = P.aggregate(P.GradientSet(tuple(ts)), P.GroupSpec(1), comm)
        assert all(t.to_bytes() == dict(gg)[t.name].tobytes() for t in res.tensors), chunk_kb
    comm.set_param("host_chunk_kb", 8192)
    comm.close()


def test_overlapped_aggregator_single_rank():
    comm = P.Communicator(rank=0, size=1, device=0, staging_bytes=64 << 20, pool_bytes=2 << 20)
    layers = [480_000] * 20 + [77, 1_000_003]
    g = I.synth_gradients(0, 0, layers, 0)
    ov = P.OverlappedAggregator([(nm, a.size, "float32") for nm, a in g], comm, cfg=P.FusionConfig(8 << 20))
    assert len(ov.groups) > 2
    for nm, a in reversed(g):
        ov.ready(nm, torch.from_numpy(a).cuda())
    res = ov.finish()
    assert res.names == sorted(nm for nm, _ in g)
    assert all(t.to_bytes() == dict(g)[t.name].tobytes() for t in res.tensors)
    with pytest.raises(P.ShapeError):
        ov.ready("nope", torch.zeros(3, device="cuda"))
    ov.ready(g[0][0], torch.from_numpy(g[0][1]).cuda())
    with pytest.raises(P.ShapeError):
        ov.ready(g[0][0], torch.from_numpy(g[0][1]).cuda())
    with pytest.raises(P.ShapeError):
        ov.finish()
    comm.close()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_dynamic_allgather_and_sm_reduce_variants(p):
    """Opt-in kernel variants must stay bit-identical: the task-queue allgather
    (dyn_ag) and the SM-load reduce (bulk_rs off)."""
    g = P.VirtualGroup(p, 0, staging_bytes=64 << 20, timeout_s=5.0)
    n = 3_000_017
    rng = np.random.default_rng([p, 123])
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32) for _ in range(p)]
    for algo in ("ring_rsa", "rhd_rsa"):
        want = OC.allreduce(xs, "sum", algo, "float32").tobytes()
        for knobs in ({"dyn_ag": 2}, {"bulk_rs": 1}, {"bulk_rs": 3, "dyn_ag": 2},
                      {"bulk_stage_kb": 16}, {"bulk_stage_kb": 112}):
            for k, v in knobs.items():
                g.set_param(k, v)
            for _ in range(2):
                res = P.allreduce_group(dev_tensors(xs, "float32"), P.ReduceOp.SUM, g, algo=algo)
                assert all(t.to_bytes() == want for t, _ in res), knobs
            g.set_param("dyn_ag", 1)
            g.set_param("bulk_rs", 6)
            g.set_param("bulk_stage_kb", 64)
    g.close()
