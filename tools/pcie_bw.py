"""Host<->device copy ceilings on this box (diagnostics for the e2e number).

    python tools/pcie_bw.py                       # one GPU
    torchrun --nproc-per-node 4 tools/pcie_bw.py  # all ranks copying at once

Prints GB/s per GPU for H2D alone, D2H alone and both directions at once
(two streams), pinned host memory, 101.76 MB (the C5 gradient set).
"""
import os

import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", 0))
world = int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
S = int(os.environ.get("BYTES", 101_760_000))
hsrc = torch.empty(S, dtype=torch.uint8).pin_memory()
hdst = torch.empty(S, dtype=torch.uint8).pin_memory()
d1 = torch.empty(S, dtype=torch.uint8, device="cuda")
d2 = torch.empty(S, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, it=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def h2d():
    d1.copy_(hsrc, non_blocking=True)


def d2h():
    hdst.copy_(d2, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(hsrc, non_blocking=True)
    with torch.cuda.stream(s2):
        hdst.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def pipelined(piece):
    """H2D piece k -> event -> D2H piece k of the same bytes (the single-rank
    host pipeline's shape), pieces of `piece` bytes."""
    def fn():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for a in range(0, S, piece):
            b = min(S, a + piece)
            with torch.cuda.stream(s1):
                d1[a:b].copy_(hsrc[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                hdst[a:b].copy_(d1[a:b], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    return fn


res = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("pipe8M", pipelined(8 << 20)),
                 ("pipe2M", pipelined(2 << 20)), ("pipe32M", pipelined(32 << 20))):
    ms = timed(fn)
    res[name] = (ms, S / (ms * 1e-3) / 1e9)
line = f"rank {rank}/{world}: " + " ".join(f"{k} {ms:.3f} ms ({gb:.1f} GB/s)" for k, (ms, gb) in res.items())
print(line, flush=True)

# ---- member-wise (C5: 53 x 1.92 MB separate pinned tensors) DMA vs SM-driven copies
import ctypes as C  # noqa: E402
import sys  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_11112_b200 import _lib as L  # noqa: E402

M, E = 53, 480_000 * 4
hm = [torch.empty(E, dtype=torch.uint8).pin_memory() for _ in range(M)]
hout = torch.empty(M * E, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(M * E, dtype=torch.uint8, device="cuda")
dsrc = torch.empty(M * E, dtype=torch.uint8, device="cuda")


def kcopy(srcs, dsts, sizes, stream):
    n = len(srcs)
    L.check(L.lib.cm_batched_copy(n, (C.c_void_p * n)(*srcs), (C.c_void_p * n)(*dsts),
                                  (C.c_int64 * n)(*sizes), stream.cuda_stream))


def dma_members():
    for i, h in enumerate(hm):
        dbuf[i * E:(i + 1) * E].copy_(h, non_blocking=True)


def k_members(stream=None):
    s = stream or torch.cuda.current_stream()
    kcopy([h.data_ptr() for h in hm], [dbuf.data_ptr() + i * E for i in range(M)], [E] * M, s)


def dma_out():
    hout.copy_(dsrc, non_blocking=True)


def k_out(stream=None):
    s = stream or torch.cuda.current_stream()
    kcopy([dsrc.data_ptr()], [hout.data_ptr()], [M * E], s)


def pair(a, b):
    def run():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            a(s1) if a in (k_members, k_out) else a()
        with torch.cuda.stream(s2):
            b(s2) if b in (k_members, k_out) else b()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    return run


res = {}
for name, fn in (("dma_members", dma_members), ("kernel_members", k_members), ("dma_out", dma_out),
                 ("kernel_out", k_out), ("dma_members+dma_out", pair(dma_members, dma_out)),
                 ("kernel_members+dma_out", pair(k_members, dma_out)),
                 ("dma_members+kernel_out", pair(dma_members, k_out)),
                 ("kernel_members+kernel_out", pair(k_members, k_out))):
    ms = timed(fn)
    res[name] = ms
print(f"rank {rank}/{world} member-wise 53 x 1.92 MB: " + " | ".join(f"{k} {v:.3f} ms" for k, v in res.items()),
      flush=True)

# ---- host -> host through the SMs (one kernel reads pinned host memory over
# PCIe and writes pinned host memory: both directions at once, no staging and
# no H2D -> D2H dependency)
hflat_in = torch.empty(M * E, dtype=torch.uint8).pin_memory()
res = {}
for name, fn in (("kernel_h2h_members", lambda: kcopy([h.data_ptr() for h in hm],
                                                      [hout.data_ptr() + i * E for i in range(M)], [E] * M,
                                                      torch.cuda.current_stream())),
                 ("kernel_h2h_flat", lambda: kcopy([hflat_in.data_ptr()], [hout.data_ptr()], [M * E],
                                                   torch.cuda.current_stream()))):
    ms = timed(fn)
    res[name] = ms
print(f"rank {rank}/{world} host->host kernel, {M * E / 1e6:.2f} MB: " +
      " | ".join(f"{k} {v:.3f} ms ({M * E / (v * 1e-3) / 1e9:.1f} GB/s each way)" for k, v in res.items()), flush=True)
