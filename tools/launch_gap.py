"""Back-to-back launch cost of empty kernels (diagnostics, cm_bench_p2p):
the CollParams parameter block (mode 2, 0 bytes) vs a 4-byte parameter
(mode 16) vs the same with large dynamic shared memory (mode 17), on 148 and
296 CTAs of 512 threads. us per launch, CUDA events over 500 launches (host
bound for empty kernels). Then the device-side gap between consecutive 20 us
spin kernels (modes 18/19: %globaltimer stamps, median).

    torchrun --nproc-per-node 2 tools/launch_gap.py
"""
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
comm = P.Communicator(staging_bytes=16 << 20, pool_bytes=2 << 20, blocking=False)
s = torch.cuda.current_stream().cuda_stream
for ctas in (1, 148, 296):
    for mode, nbytes, what in ((2, 0, "CollParams param block"), (16, 0, "4-byte param"),
                               (17, 100 << 10, "4-byte param + 100 KiB dyn smem"),
                               (17, 200 << 10, "4-byte param + 200 KiB dyn smem")):
        if mode == 17 and ctas > 148:
            continue
        ms = C.c_double()
        L.check(L.lib.cm_bench_p2p(comm._h, mode, nbytes, ctas, 500, s, C.byref(ms)))
        if rank == 0:
            print(f"ctas={ctas:4d} {what:<34} {ms.value * 1e3:6.2f} us/launch", flush=True)
# device-side gap: 20 us spin kernels (the host stays ahead), CTA 0's end stamp
# of launch i to its start stamp of launch i + 1 (median)
for ctas in (1, 148):
    for mode, nbytes, what in ((18, 0, "spin, CollParams param block"), (19, 0, "spin, 20-byte params"),
                               (20, 0, "spin, CollParams, PDL launch"),
                               (20, 160 << 10, "spin, PDL, 160 KiB smem (1 CTA/SM)"),
                               (21, 0, "spin, PDL, one remote store"), (22, 0, "spin, PDL, one remote load"),
                               (24, 0, "spin, PDL, one remote ld.cg")):
        ms = C.c_double()
        L.check(L.lib.cm_bench_p2p(comm._h, mode, nbytes, ctas, 200, s, C.byref(ms)))
        if rank == 0:
            print(f"ctas={ctas:4d} {what:<34} device gap {ms.value * 1e3:6.2f} us", flush=True)
comm.close()
dist.destroy_process_group()
