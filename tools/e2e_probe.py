"""Where the single-rank e2e step goes: host time of one aggregate() call on
pinned host gradients (enqueue only, non-blocking) vs the blocking step, and
the copy floors measured in the same process.

    python tools/e2e_probe.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1810_11112_b200 as P  # noqa: E402

torch.cuda.set_device(0)
comm = P.Communicator(0, 1, 0, staging_bytes=256 << 20, pool_bytes=64 << 20, blocking=False)
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    comm.set_param(k, int(v))
group = P.GroupSpec(1)
cfg = P.FusionConfig(64 << 20)
hgs = bench.make_grads("resnet50_like", 0, None, "float32", pinned=True)
r = None
for _ in range(3):
    r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
torch.cuda.synchronize()
K = 20
enq = []
t0 = time.perf_counter()
for _ in range(K):
    a = time.perf_counter()
    r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
    enq.append(time.perf_counter() - a)
    torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K
# device span of one step on the caller's stream (the copy streams join it)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
spans = []
for _ in range(K):
    e0.record()
    r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
    e1.record()
    torch.cuda.synchronize()
    spans.append(e0.elapsed_time(e1))
comm.blocking = True
t0 = time.perf_counter()
for _ in range(K):
    r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
blocking = (time.perf_counter() - t0) / K
enq.sort()
spans.sort()
print(f"params {sys.argv[1:]}: blocking step {blocking * 1e3:.3f} ms | non-blocking enqueue median "
      f"{enq[K // 2] * 1e6:.0f} us, +sync wall {wall * 1e3:.3f} ms | device span median {spans[K // 2]:.3f} ms "
      f"(min {spans[0]:.3f})", flush=True)
