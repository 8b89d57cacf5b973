"""Real-mode (one process per GPU) reproduction of one large copy-in allreduce."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, torch.distributed as dist
import paper_1810_11112_b200 as P
from oracle import collectives as OC
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
comm = P.Communicator(staging_bytes=256 << 20, pool_bytes=64 << 20, timeout_s=60.0)
for n in [int(v) for v in os.environ.get("N", "262145,4194304,5000011,20000003").split(",")]:
    rng = np.random.default_rng([21, n])
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    for algo in os.environ.get("ALGOS", "ring_rsa,rhd_rsa,flat").split(","):
        for chunk in (8192, 1):
            comm.set_param("stream_chunk", chunk)
            print(f"rank {rank} {algo} n={n} chunk={chunk} ...", flush=True)
            out, _ = P.allreduce(P.Tensor("x", "float32", torch.from_numpy(xs[rank]).cuda()), P.ReduceOp.SUM,
                                 P.GroupSpec(world), comm, algo=algo)
            ok = out.to_bytes() == OC.allreduce(xs, "sum", algo, "float32").tobytes()
            print(f"rank {rank} {algo} n={n} chunk={chunk}: {'ok' if ok else 'MISMATCH'}", flush=True)
comm.close()
dist.destroy_process_group()
