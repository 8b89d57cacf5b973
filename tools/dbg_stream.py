import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1810_11112_b200 as P
from oracle import collectives as OC
torch.cuda.set_device(0)
p = int(os.environ.get("P", 4))
g = P.VirtualGroup(p, 0, staging_bytes=128 << 20)
for n in [int(v) for v in os.environ.get("NS", "20000003,16320000,6000007").split(",")]:
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    for algo in ("ring_rsa", "rhd_rsa"):
        want = OC.allreduce(xs, "sum", algo, "float32")
        for chunk in (8192, 1):
            g.set_param("stream_chunk", chunk)
            try:
                res = P.allreduce_group([P.Tensor("x", "float32", torch.from_numpy(x).cuda()) for x in xs],
                                        P.ReduceOp.SUM, g, algo=algo)
            except Exception as exc:
                print(f"n={n} {algo} chunk={chunk}: EXC {exc}", flush=True)
                sys.exit(1)
            bad = [r for r, (t, _) in enumerate(res) if t.to_bytes() != want.tobytes()]
            print(f"n={n} {algo} chunk={chunk}: {'ok' if not bad else 'BAD ranks ' + str(bad)}", flush=True)
