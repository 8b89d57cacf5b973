"""Timeline of one single-rank host-gradient aggregate() step (torch.profiler,
CUPTI): when the first H2D starts after the call begins, the copies' busy
time per direction, and when the last D2H ends before the call returns.

    python tools/e2e_trace.py [knob=value ...]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1810_11112_b200 as P  # noqa: E402

torch.cuda.set_device(0)
comm = P.Communicator(0, 1, 0, staging_bytes=256 << 20, pool_bytes=64 << 20, blocking=True)
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    comm.set_param(k, int(v))
group, cfg = P.GroupSpec(1), P.FusionConfig(64 << 20)
hgs = bench.make_grads("resnet50_like", 0, None, "float32", pinned=True)
r = None
for _ in range(5):
    r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        with torch.profiler.record_function(f"step{i}"):
            r = P.aggregate(hgs, group, comm, cfg=cfg, out=r)
evs = prof.events()
for i in range(3):
    st = [e for e in evs if e.name == f"step{i}" and e.device_type.name == "CPU"][0]
    t0, t1 = st.time_range.start, st.time_range.end
    cps = sorted([e for e in evs if e.device_type.name == "CUDA" and "Memcpy" in e.name
                  and t0 <= e.time_range.start <= t1], key=lambda e: e.time_range.start)
    h = [e for e in cps if "HtoD" in e.name]
    d = [e for e in cps if "DtoH" in e.name]
    busy = lambda xs: sum(e.time_range.end - e.time_range.start for e in xs)
    print(f"step{i}: call {t1 - t0:.0f} us | first H2D at +{h[0].time_range.start - t0:.0f} us | "
          f"H2D {len(h)} copies busy {busy(h):.0f} us, last ends +{h[-1].time_range.end - t0:.0f} | "
          f"D2H {len(d)} copies busy {busy(d):.0f} us, first starts +{d[0].time_range.start - t0:.0f}, "
          f"last ends +{d[-1].time_range.end - t0:.0f} | return after last D2H {t1 - d[-1].time_range.end:.0f} us",
          flush=True)
    if i == 0:
        print("  H2D:", " ".join(f"{e.time_range.start - t0:.0f}-{e.time_range.end - t0:.0f}" for e in h))
        print("  D2H:", " ".join(f"{e.time_range.start - t0:.0f}-{e.time_range.end - t0:.0f}" for e in d))
