"""Per-phase device timing of one collective kernel (diagnostics).

    torchrun --nproc-per-node N tools/phase_trace.py --bytes 524288 --algo ring_rsa

Every CTA stamps %globaltimer at: start, copied-in, start barrier, reduced,
mid barrier, end (cm_comm_set_trace). Prints, for rank 0, the median over
CTAs of each phase duration (us) averaged over iterations.
"""
import argparse
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from paper_1810_11112_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bytes", type=int, default=524288)
ap.add_argument("--algo", default="ring_rsa")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--zc", action="store_true")
ap.add_argument("--param", action="append", default=[])
ap.add_argument("--agg", action="store_true", help="trace the C5 aggregate step (registered gradients)")
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=max(256 << 20 if a.agg else 64 << 20, a.bytes * 2), pool_bytes=max(64 << 20, a.bytes * 2),
                      blocking=False)
for kv in a.param:
    k, v = kv.split("=")
    comm.set_param(k, int(v))
n = a.bytes // 4
x = comm.empty(n) if a.zc else torch.empty(n, device="cuda")
x.normal_()
y = torch.empty(n, device="cuda")
ctas = 1024
tr = torch.zeros(ctas * 8, dtype=torch.int64, device="cuda")
tr0 = torch.zeros(ctas * 8, dtype=torch.int64, device="cuda")
gap = 0.0
fin_us = 0.0
L.check(L.lib.cm_comm_set_trace(comm._h, tr.data_ptr(), ctas))
st = L.Stats()
phases = ["copyin", "start_barrier", "reduce", "mid_barrier", "allgather"]
acc = [0.0] * 5
tot = 0.0
skew = [0.0] * 6
if a.agg:
    import bench  # noqa: E402
    gs = bench.make_grads("resnet50_like", rank, torch.device("cuda", local))
    P.register_gradients(gs, comm)
    agg_out = [None]
    for _ in range(3):
        agg_out[0] = P.aggregate(gs, P.GroupSpec(world), comm, out=agg_out[0])
    comm.synchronize()
for it in range(a.iters + 3):
    tr.zero_()
    dist.barrier()
    if a.agg:
        # back-to-back pair: the second call is traced without the host barrier skew
        agg_out[0] = P.aggregate(gs, P.GroupSpec(world), comm, out=agg_out[0])
        tr.zero_()
        agg_out[0] = P.aggregate(gs, P.GroupSpec(world), comm, out=agg_out[0])
    else:
        # back-to-back pair as well: the second call is traced (the first into
        # tr0, for the gap between the two kernels on this GPU)
        tr0.zero_()
        for rep in range(2):
            L.check(L.lib.cm_comm_set_trace(comm._h, (tr if rep else tr0).data_ptr(), ctas))
            L.check(L.lib.cm_allreduce(comm._h, x.data_ptr(), y.data_ptr(), n, 0, 0, L.ALGO[a.algo], 131072, 0,
                                       torch.cuda.current_stream().cuda_stream, C.byref(st)))
    comm.synchronize()
    if not a.agg and it >= 3:
        t0v = tr0.view(ctas, 8).cpu()
        t1v = tr.view(ctas, 8).cpu()
        ends = t0v[:, 5][t0v[:, 5] > 0]
        fin = t0v[:, 6][t0v[:, 6] > 0]
        starts = t1v[:, 0][t1v[:, 0] > 0]
        if len(ends) and len(starts):
            gap += float(starts.min() - ends.max()) / 1e3
        if len(fin) and len(ends):
            fin_us += float(fin.max() - ends.max()) / 1e3
    t = tr.view(ctas, 8).cpu()
    used = t[:, 0] > 0
    t = t[used].double()
    if it < 3:
        continue
    for k in range(5):
        d = (t[:, k + 1] - t[:, k])
        d = d[(t[:, k + 1] > 0) & (t[:, k] > 0)]
        acc[k] += float(d.median()) / 1e3 if len(d) else 0.0
    tot += float((t[:, 5].max() - t[:, 0].min())) / 1e3
    for k in range(6):
        col = t[:, k][t[:, k] > 0]
        skew[k] += float(col.max() - t[:, 0].min()) / 1e3 if len(col) else 0.0
row = [v / a.iters for v in acc] + [tot / a.iters, gap / a.iters, fin_us / a.iters]
rows = [None] * world
dist.all_gather_object(rows, row)
if rank == 0 and world > 1:
    for r, rw in enumerate(rows):
        print(f"  rank {r}: span {rw[5]:.2f} gap-before {rw[6]:.2f} (epoch hand-off {rw[7]:.2f}) | " + " ".join(f"{ph} {v:.2f}" for ph, v in zip(phases, rw[:5])),
              flush=True)
if rank == 0:
    what = "C5 aggregate (registered, 2 fused groups)" if a.agg else f"bytes={a.bytes} algo={a.algo} zc={a.zc}"
    print(f"p={world} {what} ctas={int(used.sum())} "
          f"kernel span {tot / a.iters:.2f} us | " +
          " ".join(f"{ph} {v / a.iters:.2f}" for ph, v in zip(phases, acc)) +
          " | last CTA past stamp k (from first start): " + " ".join(f"{v / a.iters:.1f}" for v in skew),
          flush=True)
L.check(L.lib.cm_comm_set_trace(comm._h, None, 0))
comm.close()
dist.destroy_process_group()
