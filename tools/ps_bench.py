"""Parameter-server step timing (paramserver.py:171-271 workload) on one GPU.

p virtual ranks (every rank a worker and a PS), the resnet50_like gradient
set (53 x 480,000 float32), lr 0.1. Prints one JSON line with the median
wall time per ``run_ps_step_group`` call (pack + fuse + ``cm_ps_step`` +
synchronize); parity of the kernel is covered by tests/test_ps.py.

    python tools/ps_bench.py --p 4                    # current libcm.so, virtual ranks
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ps_bench.py   # real NVLink ranks
    CM_LIB=.../libcm_ps_scalar.so python tools/ps_bench.py --p 4   # A/B build

Kernel-only durations come from an ncu launch list of the same command.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--dtype", choices=("float32", "float64"), default="float32")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L

    n_layers, count = 53, 480_000
    names = [f"layer{i:03d}" for i in range(n_layers)]
    rng = np.random.default_rng(0)
    params = {nm: rng.standard_normal(count).astype(a.dtype) for nm in names}
    grads = [{nm: rng.standard_normal(count).astype(a.dtype) for nm in names} for _ in range(a.p)]
    staging = max(256 << 20, 2 * n_layers * count * np.dtype(a.dtype).itemsize + (8 << 20))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        rank, local = int(os.environ["RANK"]), int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        a.p = world
        comm = P.Communicator(staging_bytes=staging, pool_bytes=64 << 20, timeout_s=10.0)
        topo = P.PsTopology.create(range(world), range(world), names)
        pt = [P.Tensor(nm, a.dtype, torch.from_numpy(params[nm]).cuda()) for nm in names]
        my_g = [P.Tensor(nm, a.dtype, torch.from_numpy(grads[rank % len(grads)][nm]).cuda()) for nm in names]
        step = lambda: P.run_ps_step(rank, comm, topo, my_g, pt, 0.1)
        res0 = step()
        for _ in range(2):
            step()
        digest = hashlib.sha256(b"".join(t.to_bytes() for t in res0)).hexdigest()[:16]
        ts = []
        for _ in range(a.iters):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            dt = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            ts.append(float(dt.item()))
        comm.close()
        if rank != 0:
            return
    else:
        vg = P.VirtualGroup(a.p, 0, staging_bytes=staging, timeout_s=10.0)
        topo = P.PsTopology.create(range(a.p), range(a.p), names)
        pt = [P.Tensor(nm, a.dtype, torch.from_numpy(params[nm]).cuda()) for nm in names]
        gper = [[P.Tensor(nm, a.dtype, torch.from_numpy(grads[r][nm]).cuda()) for nm in names]
                for r in range(a.p)]
        res = None
        for _ in range(3):
            res = P.run_ps_step_group(vg, topo, gper, [pt] * a.p, 0.1)
        # the step is deterministic: both builds must give identical parameters
        digest = hashlib.sha256(b"".join(t.to_bytes() for t in res[0])).hexdigest()[:16]
        ts = []
        for _ in range(a.iters):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.run_ps_step_group(vg, topo, gper, [pt] * a.p, 0.1)
            ts.append((time.perf_counter() - t0) * 1e3)
        vg.close()
    print(json.dumps({"tool": "ps_bench", "lib": os.path.basename(L.LIB_PATH), "p": a.p, "ranks": "real (one process per GPU)" if world > 1 else "virtual (one GPU)",
                      "dtype": a.dtype, "elements": n_layers * count, "ms_per_call_median": round(statistics.median(ts), 4),
                      "rank0_params_sha256_16": digest}))


if __name__ == "__main__":
    main()
