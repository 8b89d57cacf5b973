"""Golden sweep CSVs from the UNMODIFIED reference cost model (simcost.py),
for the restatement in paper_1810_11112_b200/costmodel.py. Run in the build
container (needs /root/reference):

    python tests/golden/gen_sweep.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import reference  # noqa: E402

CASES = [
    {"models": ["mobilenet_like", "resnet50_like", "nasnet_like"],
     "strategies": ["horovod_allreduce", "baidu_ring", "ps_pull"], "p_list": [1, 2, 3, 4, 8, 16],
     "cost": {}, "threshold": 67108864},
    {"models": ["resnet50_like", "nasnet_like"], "strategies": ["horovod_allreduce", "ps_pull"],
     "p_list": [2, 5, 8], "cost": {"alpha": 3e-6, "beta": 1.5e-12, "gamma": 4.6e-13,
                                   "driver_query_delay": 1e-6, "parallel_channels": 3},
     "threshold": 16777216},
]


def main():
    ref = reference.load()
    from collectium import simcost
    out = []
    for c in CASES:
        costs = simcost.CostModel.from_dict(c["cost"])
        reports = simcost.sweep(c["models"], c["strategies"], c["p_list"], costs, c["threshold"])
        out.append(dict(c, csv=simcost.sweep_csv_rows(reports)))
    for n, p, algo in [(8, 2, "auto"), (131071, 4, "auto"), (131072, 4, "auto"), (1 << 20, 3, "rhd_rsa"),
                       (1 << 30, 8, "ring_rsa"), (12345, 6, "flat"), (0, 5, "ring_rsa")]:
        out.append({"predict": [algo, n, p],
                    "seconds": simcost.predict_allreduce_time(algo, n, p, simcost.CostModel())})
    json.dump(out, open(os.path.join(HERE, "sweep.json"), "w"), indent=1)
    print("wrote", len(out), "cases", ref.__name__)


if __name__ == "__main__":
    main()


def ps_cases():
    """Parameter-server steps run by the unmodified reference on its simulated
    network (paramserver.py:274-298): co-located and split topologies."""
    import numpy as np
    ref = reference.load()
    from collectium import paramserver as PS
    from collectium.core import Tensor
    cases = []
    specs = [((0, 1, 2, 3), (0, 1, 2, 3), "float32", [5, 1, 1000, 37, 64, 3, 129]),
             ((0, 1, 2), (0, 1, 2), "float64", [7, 100, 2, 33]),
             ((0, 1, 2, 3), (1, 3), "float32", [16, 9, 250, 4, 1]),
             ((1, 2, 3), (0,), "float32", [8, 12, 1001])]
    for workers, ps, dtype, sizes in specs:
        names = [f"w{i:02d}" for i in range(len(sizes))]
        rng = np.random.default_rng([len(workers), len(ps), len(sizes)])
        params = [Tensor(nm, dtype, rng.standard_normal(n).astype(dtype)) for nm, n in zip(names, sizes)]
        grads = [[Tensor(nm, dtype, rng.standard_normal(n).astype(dtype)) for nm, n in zip(names, sizes)]
                 for _ in workers]
        topo = PS.PsTopology.create(workers, ps, names)
        res, _ = PS.ps_training_step(topo, grads, params, 0.05)
        cases.append({"workers": list(workers), "ps": list(ps), "dtype": dtype, "sizes": sizes, "lr": 0.05,
                      "seed": [len(workers), len(ps), len(sizes)],
                      "sha": {t.name: __import__("hashlib").sha256(t.to_bytes()).hexdigest() for t in res[0]},
                      "same_on_all_workers": all([t.to_bytes() for t in r] == [t.to_bytes() for t in res[0]]
                                                 for r in res)})
    json.dump(cases, open(os.path.join(HERE, "ps.json"), "w"), indent=1)
    print("wrote", len(cases), "ps cases", ref.__name__)


if __name__ == "__main__" and "--ps" in sys.argv:
    ps_cases()
