"""allreduce() of a pinned host tensor (100 MB fp32) at N ranks: pieced
H2D / collective / D2H (host_split=2) vs one launch between whole copies.

    torchrun --nproc-per-node 2 tools/host_allreduce_ab.py
"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
comm = P.Communicator(rank, world, local, staging_bytes=256 << 20, pool_bytes=64 << 20)
group = P.GroupSpec(world)
x = torch.randn(25_440_000).pin_memory()
y = torch.empty_like(x).pin_memory()      # out=: no per-call pinned allocation
for rep in range(2):
    for split in (1, 2):
        comm.set_param("host_split", split)
        for _ in range(3):
            P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, out=y)
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(10):
            P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, group, comm, out=y)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 10 * 1e3
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"N={world} host allreduce 101.76 MB host_split={split}: {t.item():.3f} ms/call", flush=True)
comm.close()
