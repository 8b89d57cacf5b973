"""Single-GPU driver of the collective kernels (VirtualGroup) for ncu / timing.

    python tools/virtual_ar.py --p 4 --n 16777216 --algo ring_rsa --iters 5
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--algo", default="ring_rsa")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--dtype", default="float32")
a = ap.parse_args()
torch.cuda.set_device(0)
vg = P.VirtualGroup(a.p, 0, staging_bytes=max(64 << 20, a.n * 4 + (1 << 20)))
dt = P.DTYPES[a.dtype]
xs = [P.Tensor(f"r{r}", a.dtype, torch.randn(a.n, device="cuda").to(dt)) for r in range(a.p)]
for _ in range(a.iters):
    res = P.allreduce_group(xs, P.ReduceOp.SUM, vg, algo=a.algo)
torch.cuda.synchronize()
print("ok", a.p, a.n, a.algo, res[0][0].payload[:2].tolist())
