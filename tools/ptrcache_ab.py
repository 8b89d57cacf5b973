"""Pointer-cache A/B (PAPER §V-B; reference registry.py:104-131): small-message
allreduce latency under no_cache / lazy_cache / intercept_cache.

Every cm_allreduce classifies its send and recv buffers through the
communicator's pointer cache; no_cache pays one cuPointerGetAttributes per
buffer per call (the CUDA-aware-MPI baseline the paper measures), lazy_cache
one per new address, intercept_cache none (the buffers are registered). The
host-side latency of an eager call and the device drain rate are reported
per size, with the driver queries per call and their measured wall time.

    torchrun --nproc-per-node N tools/ptrcache_ab.py [--out FILE]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from paper_1810_11112_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2000)
ap.add_argument("--out", default=None)
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=64 << 20, pool_bytes=16 << 20, blocking=False)
g = P.GroupSpec(world)
sizes = [4, 64, 1024, 16384, 131072]
rows = []


def bar():
    dist.barrier()


for nbytes in sizes:
    n = max(1, nbytes // 4)
    x = torch.full((n,), float(rank + 1), device="cuda")
    y = torch.empty_like(x)
    for pol in ("no_cache", "lazy_cache", "intercept_cache"):
        comm.set_policy(pol)
        if pol == "intercept_cache":
            comm.register(x)
            comm.register(y)
        stream = torch.cuda.current_stream().cuda_stream
        st = L.Stats()

        def call():
            L.check(L.lib.cm_allreduce(comm._h, x.data_ptr(), y.data_ptr(), n, 0, 0, 0, 131072, 0, stream,
                                       C.byref(st)))
        for _ in range(50):
            call()
        torch.cuda.synchronize()
        bar()
        q0 = comm.registry_stats()
        host = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            t0 = time.perf_counter_ns()
            call()
            host.append(time.perf_counter_ns() - t0)
        e1.record()
        torch.cuda.synchronize()
        comm.poll()
        q1 = comm.registry_stats()
        dev_us = e0.elapsed_time(e1) / args.iters * 1e3
        assert bool(torch.all(y == float(sum(r + 1 for r in range(world))))), (pol, nbytes)
        row = {"bytes": nbytes, "policy": pol, "p": world,
               "host_us_median": statistics.median(host) / 1e3,
               "host_us_mean": statistics.mean(host) / 1e3,
               "device_us_per_call": dev_us,
               "driver_queries_per_call": (q1["driver_queries"] - q0["driver_queries"]) / args.iters,
               "query_ns_per_call": (q1["query_time_ns"] - q0["query_time_ns"]) / args.iters}
        vals = [None] * world
        dist.all_gather_object(vals, row)
        if rank == 0:
            agg = dict(row)
            for k in ("host_us_median", "host_us_mean", "device_us_per_call", "query_ns_per_call"):
                agg[k] = round(max(v[k] for v in vals), 3)
            rows.append(agg)
            print(json.dumps(agg), flush=True)
comm.set_policy("lazy_cache")
if rank == 0:
    lines = [f"# tools/ptrcache_ab.py: p={world}, {args.iters} eager cm_allreduce calls per row (fp32 sum, "
             f"auto algorithm), max over ranks",
             "# host_us: wall time of one C-ABI call (enqueue incl. pointer-cache classification of send+recv); "
             "device_us: back-to-back drain rate",
             f"{'bytes':>8} {'policy':>16} {'host_us_med':>11} {'host_us_mean':>12} {'device_us':>9} "
             f"{'queries/call':>12} {'query_ns/call':>13}"]
    for r in rows:
        lines.append(f"{r['bytes']:>8} {r['policy']:>16} {r['host_us_median']:>11.2f} {r['host_us_mean']:>12.2f} "
                     f"{r['device_us_per_call']:>9.2f} {r['driver_queries_per_call']:>12.2f} "
                     f"{r['query_ns_per_call']:>13.0f}")
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(txt + "\n")
comm.close()
dist.destroy_process_group()
