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
