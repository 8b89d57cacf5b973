"""NCCL comparator, timed directly (not through torch.distributed).

ncclAllReduce (fp32 sum) through ctypes on torch's bundled libnccl, next to
this framework's cm_allreduce on the same buffers, timed the same two ways:

* eager: K back-to-back calls from the host, CUDA events around them
  (device drain per call) and the host wall time per call;
* graph: the same K calls captured in one CUDA graph, replayed once.

Plain device buffers for both libraries (ours: automatic registration, so
after the first call peers read them in place). Run under torchrun, one
process per GPU; set NCCL_NVLS_ENABLE=0 for the non-NVLS variant and
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING to log algorithm / protocol.

    torchrun --nproc-per-node N tools/nccl_direct.py --out FILE.csv
"""
import argparse
import ctypes as C
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from paper_1810_11112_b200 import _lib as L  # noqa: E402


def load_nccl():
    import nvidia
    for base in nvidia.__path__:
        p = os.path.join(base, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(p):
            return C.CDLL(p)
    return C.CDLL("libnccl.so.2")


class UniqueId(C.Structure):
    _fields_ = [("internal", C.c_byte * 128)]


ap = argparse.ArgumentParser()
ap.add_argument("--min-bytes", type=int, default=4)
ap.add_argument("--max-bytes", type=int, default=1 << 30)
ap.add_argument("--out", default=None)
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
nccl = load_nccl()
ver = C.c_int()
nccl.ncclGetVersion(C.byref(ver))
uid = UniqueId()
if rank == 0:
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
obj = [bytes(uid.internal) if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
C.memmove(uid.internal, obj[0], 128)
ncomm = C.c_void_p()
assert nccl.ncclCommInitRank(C.byref(ncomm), world, uid, rank) == 0
comm = P.Communicator(staging_bytes=max(64 << 20, args.max_bytes + (8 << 20)), pool_bytes=16 << 20, blocking=False)
maxn = args.max_bytes // 4
x = torch.randn(maxn, device="cuda")
y = torch.empty_like(x)
st = L.Stats()
stream = torch.cuda.Stream()
rows = []


def timed(fn, iters, graph):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for _ in range(iters):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        dist.barrier()
        with torch.cuda.stream(stream):
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters * 1e3, None
    dist.barrier()
    with torch.cuda.stream(stream):
        e0.record()
        t0 = time.perf_counter()
        for _ in range(iters):
            fn()
        host = (time.perf_counter() - t0) / iters * 1e6
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3, host


nbytes = args.min_bytes
while nbytes <= args.max_bytes:
    n = max(1, nbytes // 4)
    iters = 200 if nbytes <= (1 << 20) else (40 if nbytes <= (64 << 20) else 8)
    for _ in range(10):              # mapping of the automatically registered buffers settles first
        L.check(L.lib.cm_allreduce(comm._h, x.data_ptr(), y.data_ptr(), n, 0, 0, 0, 131072, 0,
                                   stream.cuda_stream, C.byref(st)))
    torch.cuda.synchronize()
    dist.barrier()

    def ours():
        L.check(L.lib.cm_allreduce(comm._h, x.data_ptr(), y.data_ptr(), n, 0, 0, 0, 131072, 0,
                                   stream.cuda_stream, C.byref(st)))

    def theirs():
        assert nccl.ncclAllReduce(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_size_t(n), 7, 0,
                                  ncomm, C.c_void_p(stream.cuda_stream)) == 0   # ncclFloat32, ncclSum
    row = {"bytes": nbytes}
    for name, fn in (("ours", ours), ("nccl", theirs)):
        dev, host = timed(fn, iters, False)
        row[f"{name}_eager_us"], row[f"{name}_host_us"] = dev, host
        if nbytes <= (16 << 20):
            row[f"{name}_graph_us"], _ = timed(fn, iters, True)
    comm.poll()
    vals = [None] * world
    dist.all_gather_object(vals, row)
    if rank == 0:
        agg = {k: (max(v[k] for v in vals) if k != "bytes" else row[k]) for k in row}
        rows.append(agg)
        print(agg, flush=True)
    nbytes *= 2
if rank == 0 and args.out:
    keys = ["bytes", "ours_eager_us", "nccl_eager_us", "ours_graph_us", "nccl_graph_us", "ours_host_us",
            "nccl_host_us"]
    with open(args.out, "w") as fh:
        fh.write(f"# tools/nccl_direct.py p={world} nccl={ver.value} NCCL_NVLS_ENABLE="
                 f"{os.environ.get('NCCL_NVLS_ENABLE', 'default')} (max over ranks; us per call)\n")
        fh.write(",".join(keys) + ",ours_busbw_gbps,nccl_busbw_gbps\n")
        for r in rows:
            fac = 2 * (world - 1) / world
            fh.write(",".join(f"{r.get(k, ''):.3f}" if isinstance(r.get(k), float) else str(r.get(k, ""))
                              for k in keys))
            fh.write(f",{r['bytes'] * fac / (r['ours_eager_us'] * 1e-6) / 1e9:.1f}"
                     f",{r['bytes'] * fac / (r['nccl_eager_us'] * 1e-6) / 1e9:.1f}\n")
nccl.ncclCommDestroy(ncomm)
comm.close()
dist.destroy_process_group()
