"""Where does the headline collective lose time? (diagnostics)

    torchrun --nproc-per-node N tools/mb_probe.py

Times, max over ranks, with and without an L2 flush between iterations:
aggregate() of the C5 set (registered and not), one allreduce of a single
101.76 MB buffer, and the two fused buffers as two separate allreduces.
"""
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1810_11112_b200 as P  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
dev = torch.device("cuda", local)
comm = P.Communicator(rank, world, local, staging_bytes=256 << 20, pool_bytes=64 << 20, blocking=False)
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    comm.set_param(k, int(v))
group = P.GroupSpec(world)
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)


def timed(fn, flush, it=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    for _ in range(it):
        if flush:
            fw.zero_()
            fr.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ts)
    t = torch.tensor([ms])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() * 1e3


gs = bench.make_grads("resnet50_like", rank, dev)
st = {"o": None}


def agg():
    st["o"] = P.aggregate(gs, group, comm, out=st["o"])


big = torch.randn(25_440_000, device=dev)
b0, b1 = big[:16_320_000], big[16_320_000:]
out = torch.empty_like(big)


def one():
    P.allreduce(P.Tensor("x", "float32", big), P.ReduceOp.SUM, group, comm, algo="ring_rsa", out=out)


def two():
    P.allreduce(P.Tensor("x", "float32", b0), P.ReduceOp.SUM, group, comm, algo="ring_rsa", out=out[:16_320_000])
    P.allreduce(P.Tensor("x", "float32", b1), P.ReduceOp.SUM, group, comm, algo="ring_rsa", out=out[16_320_000:])


res = {}
for name, fn in (("aggregate_unreg", agg), ("single_101MB", one), ("two_buffers", two)):
    for fl in (False, True):
        res[f"{name}{'_flush' if fl else ''}"] = timed(fn, fl)
P.register_gradients(gs, comm)
st["o"] = None
comm.register_buffers([big])
for name, fn in (("aggregate_reg", agg), ("single_101MB_reg", one)):
    for fl in (False, True):
        res[f"{name}{'_flush' if fl else ''}"] = timed(fn, fl)
if rank == 0:
    print(f"p={world} " + " | ".join(f"{k} {v:.1f}us" for k, v in res.items()), flush=True)
comm.close()
dist.destroy_process_group()
