"""Host cost of OverlappedAggregator.ready() per gradient (diagnostics): the
backward loop of a training step is often host-bound, so every microsecond
spent in ready() lands on the step. p = 1 communicator, C5 schema (53 x
480,000 fp32, 16 MiB fusion threshold -> 7 groups), median over steps.

    python tools/ready_overhead.py
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402

torch.cuda.set_device(0)
comm = P.Communicator(rank=0, size=1, device=0, staging_bytes=256 << 20, pool_bytes=2 << 20, blocking=False)
names = [f"layer{i:04d}" for i in range(53)]
grads = [torch.randn(480_000, device="cuda") for _ in names]
ov = P.OverlappedAggregator([(nm, 480_000, "float32") for nm in names], comm, cfg=P.FusionConfig(16 << 20))
per_ready, per_launch, per_step = [], [], []
for step in range(30):
    t_step = time.perf_counter_ns()
    for nm, g in zip(reversed(names), reversed(grads)):
        t0 = time.perf_counter_ns()
        before = ov._next
        ov.ready(nm, g)
        dt = time.perf_counter_ns() - t0
        (per_launch if ov._next != before else per_ready).append(dt / 1e3)
    ov.finish()
    per_step.append((time.perf_counter_ns() - t_step) / 1e3)
    torch.cuda.synchronize()
print(f"ready() without a launch: median {statistics.median(per_ready):.2f} us; "
      f"with a group launch: median {statistics.median(per_launch):.2f} us; "
      f"host per step (53 ready + finish): median {statistics.median(per_step[3:]):.1f} us", flush=True)
comm.close()
