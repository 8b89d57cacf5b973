"""Host cost of one small allreduce through each layer (diagnostics):

* `ctypes`: cm_allreduce called directly through the ctypes binding;
* `fast-call`: the same entry point through the CPython module `_cmfast`
  (csrc/pyfast.cpp) that the façade uses when it is built;
* `allreduce()`: the reference-API façade (collectives.allreduce), non-blocking;
* `allreduce(blocking)`: the same with the default blocking semantics
  (each call waits for its kernel and raises device-side errors).

Per layer: host microseconds per call (median over 2000 calls, eager, the
device drains concurrently) and the device drain rate. torchrun, p ranks.
"""
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

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=16 << 20, pool_bytes=16 << 20, blocking=False)
g = P.GroupSpec(world)
x = torch.full((256,), float(rank + 1), device="cuda")
y = torch.empty_like(x)
t = P.Tensor("x", "float32", x)
st = L.Stats()
s = torch.cuda.current_stream().cuda_stream


def direct():
    L.check(L.lib.cm_allreduce(comm._h, x.data_ptr(), y.data_ptr(), 256, 0, 0, 0, 131072, 0, s, C.byref(st)))


def fastcall():
    status, *_ = L.fast.allreduce(comm._hv, x.data_ptr(), y.data_ptr(), 256, 0, 0, 0, 131072, 0, s)
    L.check(status)


def facade():
    P.allreduce(t, P.ReduceOp.SUM, g, comm)


def facade_out():
    P.allreduce(t, P.ReduceOp.SUM, g, comm, out=y)


print(f"rank {rank}: fast-call module {'loaded' if L.fast else 'MISSING'}", flush=True)
rows = {}
for name, fn, blocking in (("ctypes", direct, False), ("fast-call", fastcall, False), ("allreduce()", facade, False),
                           ("allreduce(out=)", facade_out, False), ("allreduce(blocking)", facade, True)):
    comm.blocking = blocking
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    host = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2000):
        t0 = time.perf_counter_ns()
        fn()
        host.append(time.perf_counter_ns() - t0)
    e1.record()
    torch.cuda.synchronize()
    rows[name] = {"host_us_median": statistics.median(host) / 1e3, "device_us_per_call": e0.elapsed_time(e1) / 2000 * 1e3}
comm.blocking = True
vals = [None] * world
dist.all_gather_object(vals, rows)
if rank == 0:
    for name in rows:
        print(f"p={world} {name:<22} host {max(v[name]['host_us_median'] for v in vals):6.2f} us/call, "
              f"device {max(v[name]['device_us_per_call'] for v in vals):6.2f} us/call", flush=True)
comm.close()
dist.destroy_process_group()
