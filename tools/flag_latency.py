"""NVLink flag latency (diagnostics): one-thread ping-pong round trip between
ranks 0 and 1, and the start-barrier pattern (every CTA publishes one
release-store flag to every peer and waits for all of theirs) at several grid
sizes. torchrun --nproc-per-node N tools/flag_latency.py"""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from paper_1810_11112_b200 import _lib as L  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=16 << 20, pool_bytes=16 << 20)
s = torch.cuda.current_stream().cuda_stream
iters = 2000
out = []
for mode, ctas in ((10, 1), (11, 1), (11, 148), (12, 1), (12, 148), (13, 1), (13, 148)):
    ms = C.c_double()
    dist.barrier()
    L.check(L.lib.cm_bench_p2p(comm._h, mode, iters, ctas, 3, s, C.byref(ms)))
    out.append((mode, ctas, ms.value / iters * 1e3))
if rank == 0:
    for mode, ctas, us in out:
        what = "ping-pong round trip (ranks 0,1)" if mode == 10 else f"all-to-all flag barrier ({"release/acquire" if mode == 11 else "relaxed"}), {ctas} CTAs"
        print(f"p={world} {what}: {us:.2f} us", flush=True)
comm.close()
dist.destroy_process_group()
