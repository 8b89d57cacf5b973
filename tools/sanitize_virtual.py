"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every kernel family, on virtual groups (one GPU), each result
checked against the oracle:

    compute-sanitizer --tool memcheck python tools/sanitize_virtual.py

one-shot LL, LL two-shot, pull one-/two-shot (bulk-engine and SM-load reduce),
reduce-scatter / allgather, the log2(p) RHD kernel, the fused multi-buffer
aggregate (packed and gathered registered members, inline and kernel
agreement incl. a disagreement), the parameter-server step and the batched
copies. Sizes are small: the tools slow kernels down by orders of magnitude,
so the device-side wait budget is raised to 600 s.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from oracle import aggregation as OA  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from oracle import paramserver as OPS  # noqa: E402
from tests.golden import inputs as I  # noqa: E402

torch.cuda.set_device(0)
checks = 0


def ok(cond, what):
    global checks
    checks += 1
    if not cond:
        raise SystemExit(f"MISMATCH: {what}")


def dev(xs, dtype="float32"):
    return [P.Tensor(f"r{r}", dtype, torch.from_numpy(np.ascontiguousarray(x)).cuda()) for r, x in enumerate(xs)]


for p in (2, 3, 4):
    vg = P.VirtualGroup(p, 0, staging_bytes=16 << 20, timeout_s=600.0)
    rng = np.random.default_rng(p)
    # sizes: LL one-shot, LL two-shot, pull two-shot (bulk reduce; unaligned tails)
    for n in (5, 3000, 70_001, 300_007):
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        for algo in ("ring_rsa", "rhd_rsa", "flat"):
            res = P.allreduce_group(dev(xs), P.ReduceOp.SUM, vg, algo=algo)
            ok(res[0][0].to_bytes() == OC.allreduce(xs, "sum", algo, "float32").tobytes(), f"p{p} {algo} n{n}")
    # pull one-shot (above the LL one-shot limit) and the SM-load reduce
    vg.set_param("ll_max_bytes", 1024)
    vg.set_param("oneshot_max_bytes", 1 << 20)
    xs = [rng.standard_normal(50_000).astype(np.float32) for _ in range(p)]
    res = P.allreduce_group(dev(xs), P.ReduceOp.SUM, vg, algo="rhd_rsa")
    ok(res[0][0].to_bytes() == OC.allreduce(xs, "sum", "rhd_rsa", "float32").tobytes(), f"p{p} pull one-shot")
    vg.set_param("oneshot_max_bytes", 32768)
    vg.set_param("ll_max_bytes", 32768)
    vg.set_param("bulk_rs", 1)
    xs = [rng.standard_normal(400_003).astype(np.float32) for _ in range(p)]
    res = P.allreduce_group(dev(xs), P.ReduceOp.SUM, vg, algo="ring_rsa")
    ok(res[0][0].to_bytes() == OC.allreduce(xs, "sum", "ring_rsa", "float32").tobytes(), f"p{p} SM-load reduce")
    vg.set_param("bulk_rs", 6)
    # reduce-scatter / allgather
    for layout in ("ring", "rhd"):
        xs = [rng.standard_normal(100_001).astype(np.float32) for _ in range(p)]
        want = OC.reduce_scatter(xs, "sum", layout, "float32")
        rs = P.reduce_scatter_group(dev(xs), P.ReduceOp.SUM, vg, layout=layout)
        ok(all(t.to_bytes() == want[r].tobytes() for r, (t, _) in enumerate(rs)), f"p{p} RS {layout}")
        ag = P.allgather_group([P.Tensor("s", "float32", t.payload) for t, _ in rs], 100_001, vg, layout=layout)
        ok(ag[0][0].to_bytes() == OC.allgather(want, 100_001, layout, "float32").tobytes(), f"p{p} AG {layout}")
    # log2(p)-step RHD
    vg.set_param("rhd_logp", 2)
    xs = [rng.standard_normal(90_001).astype(np.float32) for _ in range(p)]
    res = P.allreduce_group(dev(xs), P.ReduceOp.SUM, vg, algo="rhd_rsa")
    ok(res[0][0].to_bytes() == OC.allreduce(xs, "sum", "rhd_rsa", "float32").tobytes(), f"p{p} log-p rhd")
    vg.set_param("rhd_logp", 1)
    # fused aggregate: packed and registered (gather), inline + kernel agreement, disagreement
    layers = [70_000, 5, 130_001, 64, 90_000]
    per_rank = [I.synth_gradients(1, 0, layers, r) for r in range(p)]
    want, _, _ = OA.aggregate(per_rank, "float32", "auto", 600_000)
    for inline in (2, 1):
        vg.set_param("inline_agree", inline)
        sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in g))
                for g in per_rank]
        outs = P.aggregate_group(sets, vg, cfg=P.FusionConfig(600_000))
        ok(all(t.to_bytes() == want[t.name].tobytes() for t in outs[p - 1].tensors), f"p{p} fused packed")
        P.register_gradients_group(sets, vg)
        outs = P.aggregate_group(sets, vg, cfg=P.FusionConfig(600_000))
        ok(all(t.to_bytes() == want[t.name].tobytes() for t in outs[0].tensors), f"p{p} fused gathered")
        ren = [list(g) for g in per_rank]
        ren[p - 1][1] = ("layer0001x", ren[p - 1][1][1])
        sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).cuda()) for nm, a in g))
                for g in ren]
        outs = P.aggregate_group(sets, vg, cfg=P.FusionConfig(600_000))
        common = [nm for nm, _ in per_rank[0] if nm != "layer0001"]
        w2, _, _ = OA.aggregate([[(nm, a) for nm, a in g if nm in common] for g in per_rank], "float32",
                                "auto", 600_000)
        ok(outs[0].names == sorted(common) and all(t.to_bytes() == w2[t.name].tobytes() for t in outs[0].tensors),
           f"p{p} fused disagreement")
    vg.set_param("inline_agree", 2)
    # parameter-server step
    sizes = [3000, 7, 20_001]
    names = [f"p{i}" for i in range(len(sizes))]
    params = {nm: rng.standard_normal(n).astype(np.float32) for nm, n in zip(names, sizes)}
    grads = [{nm: rng.standard_normal(n).astype(np.float32) for nm, n in zip(names, sizes)} for _ in range(p)]
    topo = P.PsTopology.create(list(range(p)), list(range(p)), names)
    res = P.run_ps_step_group(vg, topo, [[P.Tensor(nm, "float32", torch.from_numpy(grads[r][nm]).cuda())
                                          for nm in names] for r in range(p)],
                              [[P.Tensor(nm, "float32", torch.from_numpy(params[nm]).cuda()) for nm in names]
                               for _ in range(p)], 0.1)
    wps = OPS.ps_step(grads, params, list(range(p)), 0.1)
    ok(all(t.to_bytes() == wps[t.name].tobytes() for t in res[0]), f"p{p} ps step")
    vg.close()
# batched copies (SM and TMA bulk engine)
ts = [P.Tensor(f"t{i}", "float32", torch.randn(n, device="cuda")) for i, n in enumerate((65_536, 3, 262_144, 64))]
(buf,) = P.fuse(ts, P.FusionConfig(1 << 40))
ok(torch.equal(buf.payload, torch.cat([t.payload for t in ts])), "fuse")
torch.cuda.synchronize()
print(f"sanitize_virtual: {checks} checks passed", flush=True)
