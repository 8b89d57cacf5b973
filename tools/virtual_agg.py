"""The headline aggregate kernel configuration (registered C5 resnet50_like
gradients, one multi-buffer two-shot launch with the fused mean) on p virtual
ranks of one GPU, a few iterations — the target of the ncu capture behind
bench.py's `virtual` block.

    python tools/virtual_agg.py --p 4 [--iters 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11112_b200 as P  # noqa: E402
from tests.golden import inputs as I  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
layers = I.MODELS["resnet50_like"]
S = sum(layers) * 4
vg = P.VirtualGroup(a.p, 0, staging_bytes=S + (8 << 20))
sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(x).cuda())
                            for nm, x in I.synth_gradients(0, 0, layers, r))) for r in range(a.p)]
P.register_gradients_group(sets, vg)
for _ in range(a.iters):
    P.aggregate_group(sets, vg)
torch.cuda.synchronize()
print(f"virtual aggregate p={a.p}: {vg.launches} launches")
