"""All-to-all NVLink pull vs push bandwidth (cm_bench_p2p) per GPU.

    torchrun --nproc-per-node N tools/p2p_bw.py
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
comm = P.Communicator(staging_bytes=int(os.environ.get("STAGING", 1 << 30)), pool_bytes=2 << 20, blocking=False)
SIZES = [int(x) for x in os.environ.get("SIZES", str(64 << 20)).split(",")]
for ctas in [int(x) for x in os.environ.get("CTAS", "148,296").split(",")]:
    names = {2: "pull-concurrent", 3: "push-concurrent", 4: "pull-TMA-bulk", 5: "pull+local-add (RS-like)",
             6: "p2-anatomy remote-only 1 store", 7: "p2-anatomy remote+local 1 store",
             8: "p2-anatomy remote+local 2 stores", 9: "p2-anatomy remote-first then local, 2 stores",
             14: "copy-engine pull", 15: "copy-engine push"}
    for mode in [int(x) for x in os.environ.get("MODES", "2,4,5,3").split(",")]:
        name = names[mode]
        for nb in SIZES:
            per = nb // (world - 1)
            per -= per % 16
            ms = C.c_double()
            dist.barrier()
            L.check(L.lib.cm_bench_p2p(comm._h, mode, per, ctas, 20, torch.cuda.current_stream().cuda_stream,
                                       C.byref(ms)))
            t = torch.tensor([ms.value], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gbs = per * (world - 1) / (t.item() * 1e-3) / 1e9
            if rank == 0:
                print(f"p={world} ctas={ctas} {name} {nb >> 20} MiB/rank-round: {gbs:.1f} GB/s per GPU "
                      f"per direction", flush=True)
comm.close()
dist.destroy_process_group()
