"""Kernel timeline of the headline aggregate step (torch.profiler / CUPTI).

    torchrun --nproc-per-node N tools/timeline.py
Prints, for rank 0, every GPU kernel of 3 consecutive steps with its start
offset and duration (us) relative to the first kernel, plus the idle gaps.
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1810_11112_b200 as P  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
dev = torch.device("cuda", local)
comm = P.Communicator(rank, world, local, staging_bytes=256 << 20, pool_bytes=64 << 20, blocking=False)
HOST = os.environ.get("HOST") == "1"     # pinned host gradients (the e2e path)
gs = bench.make_grads("resnet50_like", rank, None if HOST else dev, pinned=HOST) if HOST else \
    bench.make_grads("resnet50_like", rank, dev)
if HOST:
    comm.blocking = True
if os.environ.get("REG") == "1":
    P.register_gradients(gs, comm)
group = P.GroupSpec(world)
out = None
for _ in range(5):
    out = P.aggregate(gs, group, comm, out=out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
import time  # noqa: E402
t0w = time.perf_counter()
for _ in range(10):
    out = P.aggregate(gs, group, comm, out=out)
torch.cuda.synchronize()
if rank == 0:
    print(f"wall per aggregate(): {(time.perf_counter() - t0w) / 10 * 1e3:.3f} ms", flush=True)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        out = P.aggregate(gs, group, comm, out=out)
    torch.cuda.synchronize()
if rank == 0:
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = t0
    if HOST:    # memcpy-heavy: one line per run of same-named events
        runs = []
        for e in evs:
            nm = e.name[:40]
            if runs and runs[-1][0] == nm:
                runs[-1][2] = max(runs[-1][2], e.time_range.end)
                runs[-1][3] += 1
            else:
                runs.append([nm, e.time_range.start, e.time_range.end, 1])
        for nm, a, b, k in runs:
            print(f"{a - t0:10.1f} .. {b - t0:10.1f}  x{k:3d}  {nm}")
    else:
        for e in evs:
            s, d = e.time_range.start - t0, e.time_range.elapsed_us()
            gap = e.time_range.start - prev_end
            print(f"{s:10.1f} +{d:8.1f}  gap {gap:7.1f}  {e.name[:70]}")
            prev_end = max(prev_end, e.time_range.end)
comm.close()
if world > 1:
    dist.destroy_process_group()
