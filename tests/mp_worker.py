"""Per-rank parity program for the multi-GPU tier (one process per GPU).

Launched by tests/test_gpu_multi.py as
    torchrun --nproc-per-node N tests/mp_worker.py
Each rank checks its results against the golden fixtures / CPU oracle and
exits non-zero on the first mismatch (the message names rank and case).
"""

import hashlib
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1810_11112_b200 as P  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from tests.golden import inputs as I  # noqa: E402
from tests.golden.load import of_kind  # noqa: E402

OPS = {"sum": P.ReduceOp.SUM, "max": P.ReduceOp.MAX}


def sha(b):
    return hashlib.sha256(b).hexdigest()


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = P.Communicator(staging_bytes=256 << 20, pool_bytes=512 << 20, timeout_s=20.0)
    group = P.GroupSpec(world)
    checks = 0

    def expect(cond, what):
        nonlocal checks
        checks += 1
        if not cond:
            raise AssertionError(f"rank {rank}: {what}")

    # 1. golden allreduce cases for this group size (sum + max, f32/f64, all algos)
    for case in of_kind("allreduce"):
        if case["p"] != world:
            continue
        arrays = I.allreduce_inputs(world, case["n"], case["dtype"], case["op"])
        t = P.Tensor("x", case["dtype"], torch.from_numpy(arrays[rank]).cuda())
        out, st = P.allreduce(t, OPS[case["op"]], group, comm, algo=case["algo"])
        expect(sha(out.to_bytes()) == case["sha"], f"golden {case['dtype']} {case['algo']} {case['op']} n={case['n']}")
        expect([st.rounds, st.messages_per_rank, st.bytes_sent_per_rank] == case["stats"][rank],
               f"stats {case['algo']} n={case['n']}")
    if world == 4:
        xs = I.c1_inputs()
        for case in of_kind("c1"):
            out, _ = P.allreduce(P.Tensor("x", "float32", torch.from_numpy(xs[rank]).cuda()),
                                 P.ReduceOp.SUM, group, comm, algo=case["algo"])
            expect(sha(out.to_bytes()) == case["sha"], f"C1 {case['algo']}")

    # 1b. the literal log2(p)-step recursive halving/doubling kernel (rhd_logp):
    # golden rhd cases, then large vectors copy-in / zero-copy / in-place
    comm.set_param("rhd_logp", 2)
    for case in of_kind("allreduce"):
        if case["p"] != world or case["algo"] != "rhd_rsa":
            continue
        arrays = I.allreduce_inputs(world, case["n"], case["dtype"], case["op"])
        t = P.Tensor("x", case["dtype"], torch.from_numpy(arrays[rank]).cuda())
        out, _ = P.allreduce(t, OPS[case["op"]], group, comm, algo="rhd_rsa")
        expect(sha(out.to_bytes()) == case["sha"], f"rhd log-p golden {case['dtype']} {case['op']} n={case['n']}")
    for n in (1, 262145, 5_000_011):
        rng = np.random.default_rng([23, n])
        xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32)
              for _ in range(world)]
        want = OC.allreduce(xs, "sum", "rhd_rsa", "float32").tobytes()
        x = torch.from_numpy(xs[rank]).cuda()
        for _ in range(2):
            out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, algo="rhd_rsa")
            expect(out.to_bytes() == want, f"rhd log-p copy-in n={n}")
        sym = comm.empty(n, "float32")
        sym.copy_(x)
        P.allreduce(P.Tensor("x", "float32", sym), P.ReduceOp.SUM, group, comm, algo="rhd_rsa", out=sym)
        expect(sym.cpu().numpy().tobytes() == want, f"rhd log-p zero-copy in-place n={n}")
        comm.free(sym)
    comm.set_param("rhd_logp", 1)

    # 2. large messages: copy-in, zero-copy (symmetric pool), in-place, host buffers
    for n in (262145, 1 << 22, 5_000_011, 20_000_003):
        rng = np.random.default_rng([21, n])
        xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)).astype(np.float32)
              for _ in range(world)]
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            want = OC.allreduce(xs, "sum", algo, "float32").tobytes()
            x = torch.from_numpy(xs[rank]).cuda()
            out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, algo=algo)
            expect(out.to_bytes() == want, f"copy-in {algo} n={n}")
            sym = comm.empty(n, "float32")
            sym.copy_(x)
            out, _ = P.allreduce(P.Tensor("x", "float32", sym), P.ReduceOp.SUM, group, comm, algo=algo)
            expect(out.to_bytes() == want, f"zero-copy {algo} n={n}")
            P.allreduce(P.Tensor("x", "float32", sym), P.ReduceOp.SUM, group, comm, algo=algo, out=sym)
            expect(sym.cpu().numpy().tobytes() == want, f"zero-copy in-place {algo} n={n}")
            comm.free(sym)
            host = P.Tensor("x", "float32", xs[rank])           # numpy -> host tensor
            out, _ = P.allreduce(host, P.ReduceOp.SUM, group, comm, algo=algo)
            expect(not out.is_cuda and out.to_bytes() == want, f"host buffer {algo} n={n}")

    # 2b. registered buffers: peers read ordinary torch tensors in place after a
    # collective registration (pointer cache of IPC handles); views inside a
    # registered tensor resolve to it with an offset; mixed modes interoperate
    n = 9_000_011
    rng = np.random.default_rng([22, n])
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    big = torch.from_numpy(xs[rank]).cuda()
    comm.register_buffers([big])
    for algo in ("ring_rsa", "rhd_rsa", "flat"):
        want = OC.allreduce(xs, "sum", algo, "float32").tobytes()
        out, _ = P.allreduce(P.Tensor("x", "float32", big), P.ReduceOp.SUM, group, comm, algo=algo)
        expect(out.to_bytes() == want, f"registered {algo}")
        sub = [x[1000:5_000_000] for x in xs]
        out, _ = P.allreduce(P.Tensor("x", "float32", big[1000:5_000_000]), P.ReduceOp.SUM, group, comm,
                             algo=algo)
        expect(out.to_bytes() == OC.allreduce(sub, "sum", algo, "float32").tobytes(), f"registered view {algo}")
        other = big.clone() if rank % 2 else big        # odd ranks: unregistered copy
        out, _ = P.allreduce(P.Tensor("x", "float32", other), P.ReduceOp.SUM, group, comm, algo=algo)
        expect(out.to_bytes() == want, f"mixed registered/copy-in {algo}")
    comm.deregister_buffers([big])

    # 2c. other element types: int32/int64 wrap-around (bit-exact), bf16 (fp32
    # accumulation, one rounding; bit-identical to the oracle's definition)
    for dtype in ("int32", "int64"):
        info = np.iinfo(dtype)
        for n in (5, 70_001, 3_000_017):
            rng = np.random.default_rng([31, n])
            xs = [rng.integers(info.min, info.max, size=n, dtype=dtype) for _ in range(world)]
            for algo in ("ring_rsa", "rhd_rsa"):
                out, _ = P.allreduce(P.Tensor("x", dtype, torch.from_numpy(xs[rank]).cuda()), P.ReduceOp.SUM,
                                     group, comm, algo=algo)
                expect(out.to_bytes() == OC.allreduce(xs, "sum", algo, dtype).tobytes(), f"{dtype} {algo} n={n}")
    for n in (9, 70_001, 3_000_017):
        rng = np.random.default_rng([32, n])
        xs = [OC.f32_to_bf16(rng.standard_normal(n).astype(np.float32)) for _ in range(world)]
        for algo in ("ring_rsa", "rhd_rsa"):
            t = torch.from_numpy(xs[rank].view(np.int16)).view(torch.bfloat16).cuda()
            out, _ = P.allreduce(P.Tensor("x", "bfloat16", t), P.ReduceOp.SUM, group, comm, algo=algo)
            expect(out.to_bytes() == OC.allreduce(xs, "sum", algo, "bfloat16").tobytes(), f"bf16 {algo} n={n}")

    # 3. reduce-scatter / allgather
    for layout in ("ring", "rhd"):
        for n in (0, 3, 1000, 1 << 20):
            xs = I.allreduce_inputs(world, n, "float32", "sum") if n < 5000 else \
                [np.random.default_rng([5, r]).standard_normal(n).astype(np.float32) for r in range(world)]
            want = OC.reduce_scatter(xs, "sum", layout, "float32")
            seg, _ = P.reduce_scatter(P.Tensor("x", "float32", torch.from_numpy(xs[rank]).cuda()),
                                      P.ReduceOp.SUM, group, comm, layout=layout)
            expect(seg.to_bytes() == want[rank].tobytes(), f"reduce_scatter {layout} n={n}")
            full, _ = P.allgather(seg, n, group, comm, layout=layout)
            expect(full.to_bytes() == OC.allgather(want, n, layout, "float32").tobytes(),
                   f"allgather {layout} n={n}")

    # 4. fused aggregate through cm_fused_allreduce (staged pack + fused mean)
    for case in of_kind("aggregate"):
        if case["p"] != world:
            continue
        schema = I.agg_schema(world)
        mine = I.agg_inputs(schema, world, case["dtype"])[rank]
        gs = P.GradientSet(tuple(P.Tensor(nm, case["dtype"], torch.from_numpy(a).cuda()) for nm, a in mine))
        stats = []
        res = P.aggregate(gs, group, comm, algo=case["algo"],
                          cfg=P.FusionConfig(case["threshold"]), stats_out=stats)
        expect(res.names == case["names"], "aggregate names")
        expect([sha(t.to_bytes()) for t in res.tensors] == case["sha"],
               f"aggregate {case['dtype']} {case['algo']} thr={case['threshold']}")
        expect([[s.rounds, s.messages_per_rank, s.bytes_sent_per_rank] for s in stats]
               == case["stats"][rank], "aggregate stats")
    for case in of_kind("model"):
        if case["p"] != world:
            continue
        layers = I.MODELS[case["model"]]
        for host in (False, True):
            grads = I.synth_gradients(0, 0, layers, rank)
            gs = P.GradientSet(tuple(P.Tensor(nm, "float32", a if host else torch.from_numpy(a).cuda())
                                     for nm, a in grads))
            res = P.aggregate(gs, group, comm)
            h = hashlib.sha256()
            for t in res.tensors:
                h.update(t.to_bytes())
            expect(h.hexdigest() == case["sha"], f"model {case['model']} host={host}")

    # 4c. multi-buffer launches: many large fused groups (threshold 8 MB) share
    # one pack + one launch per MAXBUF groups; results vs the oracle
    from oracle import aggregation as OA
    layers = [480_000] * 12 + [1_000_003, 77]
    per_rank = [I.synth_gradients(3, 0, layers, r) for r in range(world)]
    for algo in ("ring_rsa", "rhd_rsa", "auto"):
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
        for mb in (2, 1):
            comm.set_param("multi_buffer", mb)
            gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                     for nm, a in per_rank[rank]))
            stats = []
            res = P.aggregate(gs, group, comm, algo=algo, cfg=P.FusionConfig(8 << 20), stats_out=stats)
            expect(len(stats) == len(groups), "multi-buffer call count")
            expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors),
                   f"multi-buffer aggregate {algo} mb={mb}")
    comm.set_param("multi_buffer", 2)
    # the two overlapped two-shot variants of the multi-buffer launch
    for knobs in ({"ws": 2}, {"overlap": 2}):
        for k, v in knobs.items():
            comm.set_param(k, v)
        for algo in ("ring_rsa", "rhd_rsa"):
            want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
            gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                     for nm, a in per_rank[rank]))
            res = P.aggregate(gs, group, comm, algo=algo, cfg=P.FusionConfig(8 << 20))
            expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors), f"{knobs} aggregate {algo}")
        comm.set_param("ws", 1)
        comm.set_param("overlap", 1)
    # opt-in TMA bulk-copy pack (bulk_copy) into the staging heap
    comm.set_param("bulk_copy", 2)
    aligned = [I.synth_gradients(5, 0, [480_000] * 12 + [1_000_004, 76], r) for r in range(world)]
    for algo in ("ring_rsa", "rhd_rsa"):
        want, groups, _ = OA.aggregate(aligned, "float32", algo, 8 << 20)
        gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                 for nm, a in aligned[rank]))
        res = P.aggregate(gs, group, comm, algo=algo, cfg=P.FusionConfig(8 << 20))
        expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors), f"bulk-copy pack {algo}")
    comm.set_param("bulk_copy", 1)
    # registered gradients: peers' member tensors are read in place (no pack)
    for algo in ("ring_rsa", "rhd_rsa"):
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
        gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                 for nm, a in per_rank[rank]))
        P.register_gradients(gs, comm)
        for _ in range(2):
            res = P.aggregate(gs, group, comm, algo=algo, cfg=P.FusionConfig(8 << 20))
            expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors),
                   f"registered-gradient aggregate {algo}")
        comm.deregister_buffers([t.payload for t in gs.tensors])
    for case in of_kind("model"):
        if case["p"] != world:
            continue
        grads = I.synth_gradients(0, 0, I.MODELS[case["model"]], rank)
        gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in grads))
        P.register_gradients(gs, comm)
        res = P.aggregate(gs, group, comm)
        h = hashlib.sha256()
        for t in res.tensors:
            h.update(t.to_bytes())
        expect(h.hexdigest() == case["sha"], f"registered model {case['model']}")
        comm.deregister_buffers([t.payload for t in gs.tensors])

    # 4b. host gradients through the copy-stream pipeline (H2D / collectives /
    # D2H overlapped): pinned, pageable and mixed host/device members, many
    # fused groups, persistent pinned output buckets refilled by out=
    # (host_piece_kb=300: every fused group moves in ~300 KiB pieces)
    for algo, chunk_kb in (("ring_rsa", 4096), ("auto", 4096), ("ring_rsa", 300), ("rhd_rsa", 300)):
        comm.set_param("host_piece_kb", chunk_kb)
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
        want2, _, _ = OA.aggregate([[(nm, a * 2) for nm, a in pr] for pr in per_rank], "float32", algo, 8 << 20)
        flat = torch.empty(sum(a.size for _, a in per_rank[rank]), dtype=torch.float32).pin_memory()
        for kind in ("pinned", "pageable", "mixed", "flat"):
            def mk(scale):
                ts, off = [], 0
                for i, (nm, a) in enumerate(per_rank[rank]):
                    x = torch.from_numpy(a * scale)
                    if kind == "pinned" or (kind == "mixed" and i % 2 == 0):
                        x = x.pin_memory()
                    elif kind == "mixed":
                        x = x.cuda()
                    elif kind == "flat":
                        v = flat[off:off + a.size]
                        v.copy_(x)
                        x = v
                    off += a.size
                    ts.append(P.Tensor(nm, "float32", x))
                return P.GradientSet(tuple(ts))
            res = P.aggregate(mk(1), group, comm, algo=algo, cfg=P.FusionConfig(8 << 20))
            expect(all(not t.is_cuda for t in res.tensors), f"host means stay on the host {kind}")
            expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors), f"host aggregate {algo} {kind}")
            res2 = P.aggregate(mk(2), group, comm, algo=algo, cfg=P.FusionConfig(8 << 20), out=res)
            expect(res2 is res and all(t.to_bytes() == want2[t.name].tobytes() for t in res2.tensors),
                   f"host aggregate out= refill {algo} {kind} chunk {chunk_kb}")
    comm.set_param("host_piece_kb", 4096)

    # 4e. a fused group larger than the staging area is a ConfigError on every rank
    small = P.Communicator(staging_bytes=16 << 20, pool_bytes=2 << 20, timeout_s=20.0)
    gbig = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                               for nm, a in I.synth_gradients(0, 0, [3_000_000] * 4, rank)))
    try:
        P.aggregate(gbig, group, small)
        expect(False, "oversized fused group must raise ConfigError")
    except P.ConfigError:
        pass
    small.close()

    # 4d. overlapped aggregation: groups launched from a communication stream
    # while "backward" still produces gradients; every rank marks them ready
    # in a different order; results equal aggregate() of the full set
    for algo in ("auto", "ring_rsa"):
        want, groups, _ = OA.aggregate(per_rank, "float32", algo, 8 << 20)
        schema = [(nm, a.size, "float32") for nm, a in per_rank[rank]]
        ov = P.OverlappedAggregator(schema, comm, algo=algo, cfg=P.FusionConfig(8 << 20))
        expect(len(ov.groups) == len(groups), "overlap group count")
        rng = np.random.default_rng([77, rank])
        for step in range(2):
            order = list(rng.permutation(len(per_rank[rank])))
            spin = torch.randn(1024, 1024, device="cuda")
            for i in order:
                nm, a = per_rank[rank][i]
                spin = spin @ spin.T * 1e-3                      # producer-stream work in between
                ov.ready(nm, torch.from_numpy(a).cuda())
            res = ov.finish()
            expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors),
                   f"overlapped aggregate {algo} step {step}")
            expect(len(ov.step_stats) == len(groups), "overlap stats")

    # 4m. overlapped aggregation with registered members: persistent gradient
    # buffers handed over every step, registered collectively at the end of
    # step 0 and read in place by peers afterwards (no member pack); the
    # buffers are overwritten by the next step's "backward" right after
    # finish(), so peers must be done reading them by then. Bit-exact.
    want, groups, _ = OA.aggregate(per_rank, "float32", "auto", 8 << 20)
    want2, _, _ = OA.aggregate([[(nm, a * 2) for nm, a in pr] for pr in per_rank], "float32", "auto", 8 << 20)
    bufs = {nm: torch.empty(a.size, device="cuda") for nm, a in per_rank[rank]}
    ov = P.OverlappedAggregator([(nm, a.size, "float32") for nm, a in per_rank[rank]], comm,
                                cfg=P.FusionConfig(8 << 20), register_members=True)
    rng = np.random.default_rng([78, rank])
    for step in range(4):
        scale = 1 + (step % 2)
        for i in rng.permutation(len(per_rank[rank])):
            nm, a = per_rank[rank][i]
            bufs[nm].copy_(torch.from_numpy(a * scale))
            ov.ready(nm, bufs[nm])
        res = ov.finish()
        w = want if scale == 1 else want2
        expect(all(t.to_bytes() == w[t.name].tobytes() for t in res.tensors),
               f"overlapped aggregate, registered members, step {step}")
        if step == 0:
            expect(all(r is not None for r in ov._reg), "members registered after the first step")

    # 4j. launch knobs: plain launches (pdl off) and 2-CTA-cluster capped grids
    # give the same bits; grid sizes change from call to call (epoch slots)
    for knobs in ({"pdl": 1}, {"cluster_pairs": 2, "max_ctas": 16}, {"pdl": 2, "max_ctas": 148}):
        for k, v in knobs.items():
            comm.set_param(k, v)
        for n in (700, 300_001, 2_500_007):
            xs = [np.random.default_rng([41, n, r]).standard_normal(n).astype(np.float32) for r in range(world)]
            for algo in ("ring_rsa", "rhd_rsa"):
                out, _ = P.allreduce(P.Tensor("x", "float32", torch.from_numpy(xs[rank]).cuda()),
                                     P.ReduceOp.SUM, group, comm, algo=algo)
                expect(out.to_bytes() == OC.allreduce(xs, "sum", algo, "float32").tobytes(),
                       f"launch knobs {knobs} {algo} n={n}")
    comm.set_param("cluster_pairs", 1)
    want, groups, _ = OA.aggregate(per_rank, "float32", "auto", 8 << 20)
    ov = P.OverlappedAggregator([(nm, a.size, "float32") for nm, a in per_rank[rank]], comm,
                                cfg=P.FusionConfig(8 << 20), max_ctas=16, cluster_pairs=True)
    for step in range(2):
        for nm, a in per_rank[rank]:
            ov.ready(nm, torch.from_numpy(a).cuda())
        res = ov.finish()
        expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors),
               f"overlapped aggregate, 2-CTA clusters, step {step}")
    expect(comm.get_param("cluster_pairs") == 1 and comm.get_param("max_ctas") == 148,
           "overlapped aggregator restores the launch knobs")

    # 4l. automatic member registration: plain gradient tensors (no
    # register_gradients) are registered collectively after the second agreed
    # aggregate of a name set; later steps read them in place. A rank that
    # swaps a tensor for a new allocation makes every rank repeat the step
    # with packed members, drop the registration and register the members
    # anew after two more agreed calls. Bit-exact throughout.
    auto_layers = [300_001, 1_000_003, 7, 2_000_000, 65_536]
    auto_rank = [[(f"auto{i:03d}", a) for i, (_, a) in enumerate(I.synth_gradients(11, 0, auto_layers, r))]
                 for r in range(world)]
    want, _, _ = OA.aggregate(auto_rank, "float32", "auto", 64 << 20)
    auto_ts = [torch.from_numpy(a).cuda() for _, a in auto_rank[rank]]
    key = None
    for step in range(10):
        if step == 5 and rank == 0:
            auto_ts[1] = auto_ts[1].clone()            # a new allocation on rank 0 only
        gs = P.GradientSet(tuple(P.Tensor(nm, "float32", t) for (nm, _), t in zip(auto_rank[rank], auto_ts)))
        res = P.aggregate(gs, group, comm)
        expect(all(t.to_bytes() == want[t.name].tobytes() for t in res.tensors), f"auto-registered aggregate step {step}")
        key = gs.__dict__["_name_key"]
        st = comm.__dict__["_auto_agg"][key]
        if step == 1:
            expect(st["ids"] is not None, "members registered after the second agreed call")
        if step == 4:
            expect(st.get("gathered_calls", 0) == 3, f"gathered path used: {st.get('gathered_calls')}")
        if step == 5:
            expect(st["ids"] is None and st.get("resets") == 1,
                   "a rank's new allocation drops the registration on every rank")
        if step == 7:
            expect(st["ids"] is not None, "members registered again after two more agreed calls")
    expect(not st["disabled"] and st.get("gathered_calls", 0) == 5,
           f"gathered path used again after re-registration: {st.get('gathered_calls')}")

    # 4k. the façade's two call paths into the C ABI (the fast-call module and
    # plain ctypes) give the same bits and stats
    from paper_1810_11112_b200 import _lib as LF
    expect(LF.fast is not None, "fast-call module loaded")
    fast = LF.fast
    n = 123_457
    xs = [np.random.default_rng([43, r]).standard_normal(n).astype(np.float32) for r in range(world)]
    res = {}
    for path in ("fast", "ctypes"):
        LF.fast = fast if path == "fast" else None
        try:
            x = P.Tensor("x", "float32", torch.from_numpy(xs[rank]).cuda())
            ar, st = P.allreduce(x, P.ReduceOp.SUM, group, comm, algo="ring_rsa")
            rs, st2 = P.reduce_scatter(x, P.ReduceOp.SUM, group, comm)
            ag, st3 = P.allgather(P.Tensor("s", "float32", rs.payload.clone()), n, group, comm)
            gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in per_rank[rank]))
            agg = P.aggregate(gs, group, comm, cfg=P.FusionConfig(8 << 20))
            res[path] = (ar.to_bytes(), st, rs.to_bytes(), st2, ag.to_bytes(), st3,
                         [t.to_bytes() for t in agg.tensors])
        finally:
            LF.fast = fast
    expect(res["fast"] == res["ctypes"], "fast-call and ctypes paths agree")
    expect(res["fast"][0] == OC.allreduce(xs, "sum", "ring_rsa", "float32").tobytes(), "fast-call allreduce exact")

    # 4f. parameter-server pull step (paramserver.py:171-271): co-located and
    # split topologies, two steps each, bit-exact vs the oracle restatement
    from oracle import paramserver as OPSV
    sizes = [300_001, 17, 1 << 20, 4096, 99_999, 2, 65_536]
    pnames = [f"p{i:02d}" for i in range(len(sizes))]
    rngp = np.random.default_rng([41, world])
    params0 = {nm: rngp.standard_normal(n).astype(np.float32) for nm, n in zip(pnames, sizes)}
    for workers, ps in ((list(range(world)), list(range(world))),
                        (list(range(world)), [world - 1]),
                        (list(range(1, world)), [0])):
        topo = P.PsTopology.create(workers, ps, pnames)
        cur = dict(params0)
        mine = [P.Tensor(nm, "float32", torch.from_numpy(cur[nm]).cuda()) for nm in pnames]
        for step in range(2):
            gr = [{nm: np.random.default_rng([42, step, w, i]).standard_normal(n).astype(np.float32)
                   for i, (nm, n) in enumerate(zip(pnames, sizes))} for w in workers]
            want = OPSV.ps_step(gr, cur, workers, 0.05)
            my_g = None
            if rank in workers:
                my_g = [P.Tensor(nm, "float32", torch.from_numpy(gr[workers.index(rank)][nm]).cuda()) for nm in pnames]
            res = P.run_ps_step(rank, comm, topo, my_g, mine, 0.05)
            if rank in workers:
                expect(all(t.to_bytes() == want[t.name].tobytes() for t in res),
                       f"ps step workers={workers} ps={ps} step={step}")
                mine = res
            else:
                expect(res is None, "pure PS rank returns None")
                mine = [P.Tensor(nm, "float32", torch.from_numpy(want[nm]).cuda()) for nm in pnames]
            cur = want

    # 4a. out= refill: persistent buckets are overwritten with the next step's means
    layers = I.MODELS["mobilenet_like"]
    g1 = I.synth_gradients(0, 0, layers, rank)
    gs1 = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in g1))
    gs2 = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a * 2).cuda()) for nm, a in g1))
    r1 = P.aggregate(gs1, group, comm)
    first = [t.payload.clone() for t in r1.tensors]
    r2 = P.aggregate(gs2, group, comm, out=r1)
    expect(r2 is r1, "out= returns the refilled GradientSet")
    expect(all(torch.equal(t.payload, 2 * f) for t, f in zip(r2.tensors, first)), "out= refill values")

    # 4b. aggregate with differing ready sets: the device-side agreement check
    # fails and the intersection is negotiated (aggregation.py:152-155)
    schema = I.agg_schema(world)
    mine = I.agg_inputs(schema, world, "float32")[rank]
    extra = [("zz_only_rank0", np.ones(7, np.float32))] if rank == 0 else []
    gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in mine + extra))
    res = P.aggregate(gs, group, comm)
    expect(res.names == sorted(nm for nm, _ in schema), "aggregate partial readiness intersection")
    res2 = P.aggregate(gs, group, comm)          # second call takes the same fallback
    expect([t.to_bytes() for t in res2.tensors] == [t.to_bytes() for t in res.tensors], "fallback repeatable")

    # 4g. differing PLANS under a pending agreement: rank 0 holds an extra
    # 5M-element tensor (more fused groups and launches than its peers), the
    # last rank an extra small tensor that sorts first (its first group is a
    # small LL-sized one). The call structure must not depend on the plan:
    # the check fails identically everywhere, no rank moves data, the
    # intersection is aggregated, and the collectives that follow line up.
    base = I.synth_gradients(11, 0, [480_000] * 20 + [3, 1_000_000, 64], rank)
    extra = []
    if rank == 0:
        extra = [("layer9999_big", np.full(5_000_000, 1.0, np.float32))]
    if rank == world - 1:
        extra = [("aaa_small_first", np.full(100, 2.0, np.float32))]
    want_i, _, _ = OA.aggregate([I.synth_gradients(11, 0, [480_000] * 20 + [3, 1_000_000, 64], r)
                                 for r in range(world)], "float32", "auto", 8 << 20)
    for inline in (2, 1):
        comm.set_param("inline_agree", inline)
        for thr in (8 << 20, 64 << 20):
            want_t, _, _ = OA.aggregate([I.synth_gradients(11, 0, [480_000] * 20 + [3, 1_000_000, 64], r)
                                         for r in range(world)], "float32", "auto", thr)
            gs = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in base + extra))
            prev = P.aggregate(P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda())
                                                   for nm, a in base)), group, comm, cfg=P.FusionConfig(thr))
            res = P.aggregate(gs, group, comm, cfg=P.FusionConfig(thr), out=prev)   # out= of another plan
            expect(res.names == sorted(nm for nm, _ in base), f"differing plans: names inline={inline} thr={thr}")
            expect(all(t.to_bytes() == want_t[t.name].tobytes() for t in res.tensors),
                   f"differing plans: values inline={inline} thr={thr}")
            for k in range(4):
                gk = P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in base))
                rk = P.aggregate(gk, group, comm, cfg=P.FusionConfig(8 << 20))
                expect(all(t.to_bytes() == want_i[t.name].tobytes() for t in rk.tensors),
                       f"after differing plans: aggregate {k} inline={inline} thr={thr}")
                x = torch.full((70_001 + k,), float(rank + k), device="cuda")
                out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm)
                expect(bool(torch.all(out.payload == float(sum(r + k for r in range(world))))),
                       f"after differing plans: allreduce {k} inline={inline} thr={thr}")
    comm.set_param("inline_agree", 2)
    # ... and with pinned host gradients, whose fused groups move through the
    # host pipeline in pieces (rank 0's extra tensor changes its piece and
    # launch count): every gated piece is skipped, the intersection is
    # aggregated, later host and device calls line up
    def host_set(items):
        return P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).pin_memory()) for nm, a in items))
    want_t, _, _ = OA.aggregate([I.synth_gradients(11, 0, [480_000] * 20 + [3, 1_000_000, 64], r)
                                 for r in range(world)], "float32", "auto", 64 << 20)
    for piece_kb in (4096, 700):
        comm.set_param("host_piece_kb", piece_kb)
        res = P.aggregate(host_set(base + extra), group, comm, cfg=P.FusionConfig(64 << 20))
        expect(res.names == sorted(nm for nm, _ in base) and not res.tensors[0].is_cuda,
               f"differing plans, host pieces {piece_kb}: names")
        expect(all(t.to_bytes() == want_t[t.name].tobytes() for t in res.tensors),
               f"differing plans, host pieces {piece_kb}: values")
        for k in range(2):
            rk = P.aggregate(host_set(base), group, comm, cfg=P.FusionConfig(64 << 20))
            expect(all(t.to_bytes() == want_t[t.name].tobytes() for t in rk.tensors),
                   f"after differing plans, host pieces {piece_kb}: aggregate {k}")
            x = torch.full((70_001 + k,), float(rank + k), device="cuda")
            out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm)
            expect(bool(torch.all(out.payload == float(sum(r + k for r in range(world))))),
                   f"after differing plans, host pieces {piece_kb}: allreduce {k}")
    comm.set_param("host_piece_kb", 4096)

    # 4n. allreduce() of host buffers: a pinned (or pageable) send moves H2D /
    # collective / D2H in pieces (host_split), bit-exact vs the oracle for
    # both layouts; host_split=1 is the one-launch path
    n = 3_000_017
    xs = [np.random.default_rng([47, r]).standard_normal(n).astype(np.float32) for r in range(world)]
    for split, piece_kb in ((2, 4096), (2, 300), (1, 4096)):
        comm.set_param("host_split", split)
        comm.set_param("host_piece_kb", piece_kb)
        for where in ("pinned", "pageable"):
            x = torch.from_numpy(xs[rank].copy())
            if where == "pinned":
                x = x.pin_memory()
            for algo in ("ring_rsa", "rhd_rsa"):
                out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, algo=algo)
                expect(not out.is_cuda and out.to_bytes() == OC.allreduce(xs, "sum", algo, "float32").tobytes(),
                       f"host allreduce {where} {algo} split={split} piece={piece_kb}")
    comm.set_param("host_split", 2)
    comm.set_param("host_piece_kb", 4096)

    # 4i. the communicator's pointer cache (registry.py:104-131): every call
    # classifies send and recv; no_cache queries the driver each time,
    # lazy_cache once per address, intercept_cache never (unregistered
    # buffers are rejected with UnknownBufferError)
    xs_small = torch.full((1000,), float(rank + 1), device="cuda")
    ys_small = torch.empty_like(xs_small)
    want_small = float(sum(r + 1 for r in range(world)))
    for pol in ("no_cache", "lazy_cache", "intercept_cache"):
        comm.set_policy(pol)
        if pol == "intercept_cache":
            try:
                P.allreduce(P.Tensor("x", "float32", xs_small), P.ReduceOp.SUM, group, comm, out=ys_small)
                expect(False, "intercept_cache must reject an unregistered buffer")
            except P.UnknownBufferError:
                pass
            comm.register(xs_small)
            comm.register(ys_small)
        q0 = comm.registry_stats()["driver_queries"]
        for _ in range(10):
            P.allreduce(P.Tensor("x", "float32", xs_small), P.ReduceOp.SUM, group, comm, out=ys_small)
            expect(bool(torch.all(ys_small == want_small)), f"policy {pol} result")
        dq = comm.registry_stats()["driver_queries"] - q0
        expect(dq == {"no_cache": 20, "lazy_cache": 2, "intercept_cache": 0}[pol], f"policy {pol}: {dq} queries")
    comm.set_policy("lazy_cache")

    # 4h. automatic registration (pointer cache -> IPC mapping, no host
    # collective): plain torch tensors are copied in on first sight, then read
    # in place once every peer has mapped their allocation; a freed and
    # re-allocated range gets a new mailbox slot. Results stay bit-exact.
    comm.set_param("auto_register", 2)
    z0 = comm.get_param("auto_zero_copy_calls")
    n_big = 3_000_017
    for rep in range(3):
        bufs = [torch.empty(n_big + 1000 * t, device="cuda") for t in range(3)]
        for it in range(4):
            for t, x in enumerate(bufs):
                rng = np.random.default_rng([rep, it, t, rank])
                xs_all = [np.random.default_rng([rep, it, t, r]).standard_normal(x.numel()).astype(np.float32)
                          for r in range(world)]
                x.copy_(torch.from_numpy(xs_all[rank]))
                algo = ("ring_rsa", "rhd_rsa", "auto")[(it + t) % 3]
                out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, algo=algo)
                expect(out.to_bytes() == OC.allreduce(xs_all, "sum", algo, "float32").tobytes(),
                       f"auto-registered allreduce rep={rep} it={it} t={t}")
                del rng
        seg, _ = P.reduce_scatter(P.Tensor("x", "float32", bufs[0]), P.ReduceOp.SUM, group, comm)
        xs_all = [np.random.default_rng([rep, 3, 0, r]).standard_normal(bufs[0].numel()).astype(np.float32)
                  for r in range(world)]
        expect(seg.to_bytes() == OC.reduce_scatter(xs_all, "sum", "ring", "float32")[rank].tobytes(),
               f"auto-registered reduce_scatter rep={rep}")
        segx = seg.payload.clone()
        full, _ = P.allgather(P.Tensor("s", "float32", segx), bufs[0].numel(), group, comm)
        expect(full.to_bytes() == OC.allgather(OC.reduce_scatter(xs_all, "sum", "ring", "float32"),
                                               bufs[0].numel(), "ring", "float32").tobytes(),
               f"auto-registered allgather rep={rep}")
        del bufs, segx
        torch.cuda.synchronize()
        torch.cuda.empty_cache()            # the ranges go back to the driver; new ones may reuse them
    # a CUDA graph captured on a never-seen plain tensor: no synchronous
    # registration inside the capture (copy-in), replays stay exact
    gx = torch.empty(2_000_003, device="cuda")
    gy = torch.empty_like(gx)
    cs = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    from paper_1810_11112_b200 import _lib as LL
    import ctypes as CT
    gst = LL.Stats()
    comm.blocking = False
    with torch.cuda.stream(cs):
        with torch.cuda.graph(graph, stream=cs):
            LL.check(LL.lib.cm_allreduce(comm._h, gx.data_ptr(), gy.data_ptr(), gx.numel(), 0, 0,
                                         LL.ALGO["ring_rsa"], 131072, 0, cs.cuda_stream, CT.byref(gst)))
    for it in range(3):
        xs_all = [np.random.default_rng([9, it, r]).standard_normal(gx.numel()).astype(np.float32)
                  for r in range(world)]
        gx.copy_(torch.from_numpy(xs_all[rank]))
        torch.cuda.synchronize()
        dist.barrier()
        graph.replay()
        torch.cuda.synchronize()
        comm.poll()
        expect(gy.cpu().numpy().tobytes() == OC.allreduce(xs_all, "sum", "ring_rsa", "float32").tobytes(),
               f"graph-captured allreduce on a plain tensor, replay {it}")
    comm.blocking = True
    expect(comm.get_param("auto_published") >= 3, "allocations published in the mailbox")
    expect(comm.get_param("auto_mapped") >= 3, "peers' allocations mapped")
    expect(comm.get_param("auto_zero_copy_calls") > z0, "plain tensors read in place")

    # 5. negotiation: partial intersection falls back to the control plane
    ready = ["a", "b", "c"] if rank == 0 else ["b", "c", "d"]
    expect(P.negotiate_ready(ready, group, comm) == ["b", "c"], "negotiate partial")
    expect(P.negotiate_ready(["z", "y"], group, comm) == ["y", "z"], "negotiate full")

    # 6. peer shape mismatch is detected on the device -> ShapeError everywhere
    bad = torch.zeros(3 + rank, device="cuda")
    try:
        P.allreduce(P.Tensor("x", "float32", bad), P.ReduceOp.SUM, group, comm)
        expect(False, "mismatched lengths did not raise")
    except P.ShapeError:
        checks += 1
    # the communicator stays usable afterwards
    x = torch.full((10,), float(rank), device="cuda")
    out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm)
    expect(out.payload.cpu().tolist() == [float(sum(range(world)))] * 10, "usable after ShapeError")

    # 7. back-to-back stress with changing sizes (epoch/parity reuse), async
    comm.blocking = False
    rng = np.random.default_rng(77)
    sizes = [int(s) for s in rng.integers(0, 300000, size=200)]
    outs = []
    for i, n in enumerate(sizes):
        x = torch.full((n,), float(rank + i), device="cuda")
        algo = ("ring_rsa", "rhd_rsa", "auto", "flat")[i % 4]
        out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, algo=algo)
        outs.append((n, i, out.payload))
    comm.synchronize()
    for n, i, o in outs:
        want = float(sum(r + i for r in range(world)))
        expect(n == 0 or bool(torch.all(o == want)), f"stress call {i} n={n}")
    comm.blocking = True

    dist.barrier()
    comm.close()
    print(f"rank {rank}: {checks} checks passed", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    try:
        main()
    except Exception:
        traceback.print_exc()
        sys.stdout.flush()
        os._exit(1)
