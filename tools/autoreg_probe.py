"""Automatic-registration probe (2+ ranks): plain torch tensors through
allreduce; prints the auto-registration counters per call. Run with torchrun
(one process per GPU, or several processes sharing one GPU)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from oracle import collectives as OC  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=256 << 20, pool_bytes=64 << 20, timeout_s=20.0)
g = P.GroupSpec(world)
n = int(os.environ.get("N", 3_000_017))
x = torch.empty(n, device="cuda")
for it in range(int(os.environ.get("ITERS", 6))):
    xs = [np.random.default_rng([it, r]).standard_normal(n).astype(np.float32) for r in range(world)]
    x.copy_(torch.from_numpy(xs[rank]))
    out, _ = P.allreduce(P.Tensor("x", "float32", x), P.ReduceOp.SUM, g, comm, algo="ring_rsa")
    ok = out.to_bytes() == OC.allreduce(xs, "sum", "ring_rsa", "float32").tobytes()
    print(f"rank {rank} it {it} ok={ok} published={comm.get_param('auto_published')} "
          f"mapped={comm.get_param('auto_mapped')} zc={comm.get_param('auto_zero_copy_calls')}", flush=True)
comm.close()
dist.destroy_process_group()
