"""Host-side cost of one small allreduce submission (the paper's small-message
latency concern, §8 pointer-cache row), one process per GPU:

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/host_overhead.py

Times N back-to-back host calls WITHOUT synchronising in between (so the
figure is the host's submission cost per call once the launch queue is the
bottleneck) for: an empty C-ABI call (cm_comm_poll), a bare torch kernel
launch (x.add_(1)), and cm_allreduce on 4 B / 4 KiB / 64 KiB through a
plain (unregistered) buffer and through a registered one.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    import torch
    import torch.distributed as dist
    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = P.Communicator(staging_bytes=64 << 20, pool_bytes=64 << 20, timeout_s=10.0, blocking=False)
    st = L.Stats()
    stream = torch.cuda.current_stream().cuda_stream
    plain = torch.randn(1 << 16, device="cuda")
    plain_out = torch.empty_like(plain)
    reg = comm.empty(1 << 16, "float32")
    reg_out = comm.empty(1 << 16, "float32")
    reg.normal_()
    x = torch.zeros(1, device="cuda")
    n_calls = 2000

    def host_us(fn):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_calls):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        return (t1 - t0) / n_calls * 1e6, (t2 - t0) / n_calls * 1e6

    rows = {}
    rows["cm_comm_poll (empty C-ABI call)"] = host_us(lambda: L.check(L.lib.cm_comm_poll(comm._h)))
    rows["torch add_ (one kernel launch)"] = host_us(lambda: x.add_(1))
    for nb in (4, 4096, 65536):
        n = nb // 4
        for tag, s, d in (("plain", plain, plain_out), ("registered", reg, reg_out)):
            rows[f"cm_allreduce {nb} B {tag}"] = host_us(
                lambda s=s, d=d, n=n: L.check(L.lib.cm_allreduce(comm._h, s.data_ptr(), d.data_ptr(), n, 0, 0,
                                                                  L.ALGO["rhd_rsa"], 131072, 0, stream,
                                                                  C.byref(st))))
    comm.close()
    if rank == 0:
        for k, (sub, tot) in rows.items():
            print(json.dumps({"call": k, "p": world, "host_submit_us": round(sub, 3),
                              "submit_plus_drain_us": round(tot, 3)}))


if __name__ == "__main__":
    main()
