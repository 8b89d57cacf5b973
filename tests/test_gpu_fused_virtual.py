"""GPU parity of the exact aggregate() kernel path on ONE B200.

``aggregate_group`` drives ``cm_fused_allreduce_agreed_v``, the same C path a
real communicator takes at N >= 2 (``cm_fused_allreduce_agreed``):

* inline ready-set agreement in the start-barrier records of the first fused
  collective (forced onto the full grid), later launches gated;
* the separate LL agreement kernel (``inline_agree=1``) with gated launches;
* multi-buffer two-shot launches (``nbuf > 1``) fed by the pack kernel
  (SRC_PRESTAGED) or by in-place reads of registered gradients (SRC_GATHER);
* host gradients (pinned / pageable / mixed) through the H2D / D2H copy
  streams;
* the fused IEEE mean.

Results are compared with the reference golden fixtures (model gradient sets)
and with the oracle restatement of aggregation.py (pinned against the golden
aggregate cases in tests/test_oracle_golden.py): bit-exact for fp32/fp64.
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

_VG = {}


def vg(p, **params):
    key = (p, tuple(sorted(params.items())))
    if key not in _VG:
        g = P.VirtualGroup(p, 0, staging_bytes=128 << 20, timeout_s=5.0)
        for k, v in params.items():
            g.set_param(k, v)
        _VG[key] = g
    return _VG[key]


def sets_of(per_rank, dtype="float32", where="device"):
    out = []
    for r, g in enumerate(per_rank):
        ts = []
        for i, (nm, a) in enumerate(g):
            x = torch.from_numpy(np.ascontiguousarray(a))
            if where == "device" or (where == "mixed" and (i + r) % 3 == 0):
                x = x.cuda()
            elif where in ("pinned", "mixed"):
                x = x.pin_memory()
            ts.append(P.Tensor(nm, dtype, x))
        out.append(P.GradientSet(tuple(ts)))
    return out


def check(outs, want, names=None):
    for r, o in enumerate(outs):
        if names is not None:
            assert o.names == names, r
        for t in o.tensors:
            assert t.to_bytes() == want[t.name].tobytes(), (r, t.name)


@pytest.mark.parametrize("case", of_kind("model"), ids=lambda c: c["model"])
@pytest.mark.parametrize("registered", [False, True])
def test_model_golden_through_fused_path(case, registered):
    """BASELINE C4 (MobileNet, p=8) / C5 (ResNet-50, p=4) gradient sets through
    the headline kernel configuration, against the reference's SHA."""
    p = case["p"]
    layers = I.MODELS[case["model"]]
    sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                for nm, a in I.synth_gradients(0, 0, layers, r)))
            for r in range(p)]
    g = vg(p)
    if registered:
        P.register_gradients_group(sets, g)
    l0 = g.launches
    outs = P.aggregate_group(sets, g)
    for r in range(p):
        h = hashlib.sha256()
        for t in outs[r].tensors:
            h.update(t.to_bytes())
        assert h.hexdigest() == case["sha"], r
    # one multi-buffer collective (+ one pack unless registered) per step
    assert g.launches - l0 == (1 if registered else 1 + p)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["prestaged", "registered"])
@pytest.mark.parametrize("variant", ["barrier", "overlap", "ws"])
def test_multi_buffer_launches_vs_oracle(p, mode, variant):
    """8 MiB fusion threshold: the ResNet-like set splits into 13 fused groups,
    batched MAXBUF=4 per multi-buffer launch (nbuf > 1); with the RS->AG
    barrier, the CTA-split overlap and the warp-specialised overlap (the
    allgather follows the reduce-scatter's per-chunk progress)."""
    layers = I.MODELS["resnet50_like"][:24] + [77, 1_000_003, 5]
    per_rank = [I.synth_gradients(3, 1, layers, r) for r in range(p)]
    for algo in ("auto", "ring_rsa", "rhd_rsa"):
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
        assert len(groups) > 4
        sets = sets_of(per_rank)
        g = vg(p, **{"barrier": {}, "overlap": {"overlap": 2}, "ws": {"ws": 2}}[variant])
        if mode == "registered":
            P.register_gradients_group(sets, g)
        stats = []
        outs = P.aggregate_group(sets, g, algo=algo, cfg=P.FusionConfig(8 << 20), stats_out=stats)
        check(outs, want, sorted(nm for nm, _ in per_rank[0]))
        for r in range(p):
            assert len(stats[r]) == len(groups)
            for s, grp in zip(stats[r], groups):
                n = sum(a.size for nm, a in per_rank[0] if nm in grp)
                ref = OC.stats(OC.resolve_algorithm(algo, 4 * n), p, n, "float32", r)
                assert (s.rounds, s.messages_per_rank, s.bytes_sent_per_rank) == ref


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("agree_mode", ["inline", "ll_kernel"])
def test_disagreement_skips_everywhere_then_falls_back(p, agree_mode):
    """Rank 1 holds a different name of the same shape: the device-side check
    fails on every rank, no rank moves data, the intersection is negotiated
    and the collectives that follow stay in step (epochs unchanged by the
    gated no-op launches)."""
    g = vg(p) if agree_mode == "inline" else vg(p, inline_agree=1)
    layers = [300_000, 1_000_000, 5, 2_000_000, 64]
    per_rank = [I.synth_gradients(5, 0, layers, r) for r in range(p)]
    # same shapes (so the agreed attempt runs on the device), one name differs
    renamed = [list(x) for x in per_rank]
    renamed[1][2] = ("layer0002_rank1_only", renamed[1][2][1])
    l0 = g.launches
    P.aggregate_group(sets_of(per_rank), g, cfg=P.FusionConfig(4 << 20))
    agreed_launches = g.launches - l0
    l0 = g.launches
    outs = P.aggregate_group(sets_of(renamed), g, cfg=P.FusionConfig(4 << 20))
    common = sorted(set(nm for nm, _ in per_rank[0]) - {per_rank[0][2][0]})
    want, _, _ = OA.aggregate([[(nm, a) for nm, a in x if nm in common] for x in per_rank], "float32",
                              "auto", 4 << 20)
    check(outs, want, common)
    assert g.launches - l0 >= agreed_launches + 2     # the gated attempt, then the fallback
    # later calls (agreed, different sizes) still line up
    for it in range(3):
        pr = [I.synth_gradients(6, it, layers[: 2 + it], r) for r in range(p)]
        want, _, _ = OA.aggregate(pr, "float32", "auto", 4 << 20)
        check(P.aggregate_group(sets_of(pr), g, cfg=P.FusionConfig(4 << 20)), want)
        xs = [np.random.default_rng([it, r]).standard_normal(70_001).astype(np.float32) for r in range(p)]
        res = P.allreduce_group([P.Tensor("x", "float32", torch.from_numpy(x).cuda()) for x in xs],
                                P.ReduceOp.SUM, g)
        assert res[0][0].to_bytes() == OC.allreduce(xs, "sum", "auto", "float32").tobytes()


@pytest.mark.parametrize("p", [2, 3, 4])
def test_disagreement_with_logp_rhd_gated(p):
    """rhd_logp routes later rhd groups to the log2(p)-step kernel, which is
    gated as well; the first launch is forced onto the pull kernel."""
    g = vg(p, rhd_logp=2)
    layers = [1000, 70_000, 3, 90_000]
    per_rank = [I.synth_gradients(8, 0, layers, r) for r in range(p)]
    for algo in ("rhd_rsa", "auto"):
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 300_000)
        assert len(groups) > 1
        check(P.aggregate_group(sets_of(per_rank), g, algo=algo, cfg=P.FusionConfig(300_000)), want)
        renamed = [list(x) for x in per_rank]
        renamed[0][0] = ("layer0000x", renamed[0][0][1])
        common = sorted(nm for nm, _ in per_rank[0][1:])
        want, _, _ = OA.aggregate([[(nm, a) for nm, a in x if nm in common] for x in per_rank], "float32",
                                  algo, 300_000)
        check(P.aggregate_group(sets_of(renamed), g, algo=algo, cfg=P.FusionConfig(300_000)), want, common)


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("where", ["pinned", "pageable", "mixed"])
def test_host_gradients_through_copy_streams(p, where):
    layers = [480_000] * 12 + [1_000_003, 77]
    per_rank = [I.synth_gradients(9, 0, layers, r) for r in range(p)]
    want, _, _ = OA.aggregate(per_rank, "float32", "auto", 8 << 20)
    outs = P.aggregate_group(sets_of(per_rank, where=where), vg(p), cfg=P.FusionConfig(8 << 20))
    check(outs, want)
    assert all(not t.is_cuda for o in outs for t in o.tensors)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", ["ring_rsa", "rhd_rsa", "auto"])
@pytest.mark.parametrize("split", [1, 2])
def test_host_gradients_in_pipeline_pieces(p, algo, split):
    """Host gradients move H2D -> collective -> D2H in host_piece_kb pieces (the
    piece-th 1/K of every rank's segment, so every element keeps its owner and
    fold order): bit-identical to the whole-group launch and the reference;
    host_split=1 is the one-launch-per-group pipeline."""
    layers = [480_000] * 12 + [1_000_003, 77, 65_536]
    per_rank = [I.synth_gradients(19, 0, layers, r) for r in range(p)]
    want, _, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
    g = vg(p, host_piece_kb=300, host_split=split)
    for where in ("pinned", "mixed"):
        outs = P.aggregate_group(sets_of(per_rank, where=where), g, algo=algo, cfg=P.FusionConfig(8 << 20))
        check(outs, want)
        assert all(not t.is_cuda for o in outs for t in o.tensors)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_bf16_and_fp64_fused(p):
    layers = [100_000, 7, 300_001, 64]
    per_rank = [I.synth_gradients(4, 0, layers, r) for r in range(p)]
    want, _, _ = OA.aggregate(per_rank, "float64", "auto", 1 << 20)
    f64 = [[(nm, a.astype(np.float64)) for nm, a in g] for g in per_rank]
    want, _, _ = OA.aggregate(f64, "float64", "auto", 1 << 20)
    check(P.aggregate_group(sets_of(f64, "float64"), vg(p), cfg=P.FusionConfig(1 << 20)), want)
    bf = [[(nm, OC.f32_to_bf16(a)) for nm, a in g] for g in per_rank]
    want, _, _ = OA.aggregate(bf, "bfloat16", "auto", 1 << 20)
    sets = [P.GradientSet(tuple(P.Tensor(nm, "bfloat16", torch.from_numpy(a.view(np.int16)).view(torch.bfloat16)
                                         .cuda()) for nm, a in g)) for g in bf]
    outs = P.aggregate_group(sets, vg(p), cfg=P.FusionConfig(1 << 20))
    for o in outs:
        for t in o.tensors:
            assert np.array_equal(np.frombuffer(t.to_bytes(), np.uint16), want[t.name])


@pytest.mark.parametrize("p", [2, 3, 8])
def test_negotiate_ready_group(p):
    g = vg(p)
    same = [["b", "a", "c"] for _ in range(p)]
    assert P.negotiate_ready_group(same, g) == [["a", "b", "c"]] * p
    diff = [["a", "b", "c"] if r else ["b", "c", "d"] for r in range(p)]
    assert P.negotiate_ready_group(diff, g) == [["b", "c"]] * p


def test_fuse_host_members_lands_on_the_device():
    """fuse() of host tensors (pageable and pinned): the fused buffer is a
    device tensor (the copy engines / the batched-copy kernel move the
    members; nothing is concatenated on the CPU), unfuse() gives device views."""
    rng = np.random.default_rng(3)
    arrays = [rng.standard_normal(n).astype(np.float32) for n in (5, 70_001, 3, 4096)]
    ts = []
    for i, a in enumerate(arrays):
        x = torch.from_numpy(a)
        if i % 2:
            x = x.pin_memory()
        ts.append(P.Tensor(f"t{i}", "float32", x))
    (buf,) = P.fuse(ts, P.FusionConfig(1 << 30))
    assert buf.payload.is_cuda
    torch.cuda.synchronize()
    assert buf.payload.cpu().numpy().tobytes() == np.concatenate(arrays).tobytes()
    for a, t in zip(arrays, P.unfuse(buf)):
        assert t.is_cuda and t.to_bytes() == a.tobytes()
