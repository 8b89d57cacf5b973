import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1810_11112_b200 as P
from oracle import collectives as OC
torch.cuda.set_device(0)
g = P.VirtualGroup(4, 0, staging_bytes=128 << 20)
for n in (16_320_000, 6_000_007):
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(4)]
    want = OC.allreduce(xs, "sum", "ring_rsa", "float32")
    for chunk in (1024, 8192, 1):
        for avg in (False, True):
            g.set_param("stream_chunk", chunk)
            res = P.allreduce_group([P.Tensor("x", "float32", torch.from_numpy(x).cuda()) for x in xs],
                                    P.ReduceOp.SUM, g, algo="ring_rsa", average=avg)
            w = want / np.float32(4) if avg else want
            for r, (t, _) in enumerate(res):
                got = t.numpy()
                bad = np.nonzero(got.view(np.uint32) != w.astype(np.float32).view(np.uint32))[0]
                if len(bad):
                    print(f"n={n} chunk={chunk} avg={avg} rank={r}: {len(bad)} bad, first {bad[:5]}, last {bad[-3:]}")
                    break
            else:
                print(f"n={n} chunk={chunk} avg={avg}: ok")
