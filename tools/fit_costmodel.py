"""Fit the reference's alpha-beta-gamma model (simcost.py:62-93) to this
framework's measured ring_rsa latencies -> paper_1810_11112_b200/costmodel.json.

    python tools/fit_costmodel.py profiles/r01_sweep_p2.csv profiles/r01_sweep_p4.csv

alpha: the small-message plateau (median of sizes <= 4 KiB) over the ring's
2(p-1) messages; beta: the slope between the two largest sizes over the
2(p-1)/p bytes per GPU; gamma: the reduction's HBM traffic (3 bytes moved per
reduced byte at MEASURED_PEAKS hbm_gbs). Also records predicted-vs-measured
errors over the whole sweep.
"""
import csv
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_11112_b200 import costmodel as CM  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
gamma = 3.0 / (peaks["hbm_gbs"] * 1e9)
fits = {}
for path in sys.argv[1:]:
    rows = list(csv.DictReader(open(path)))
    p = int(rows[0]["p"])
    pts = sorted((int(r["message_bytes"]), float(r["ring_rsa_us"]) * 1e-6) for r in rows)
    small = [t for n, t in pts if n <= 4096]
    alpha = statistics.median(small) / (2 * (p - 1))
    (n1, t1), (n2, t2) = pts[-2], pts[-1]
    frac = (p - 1) / p
    beta = ((t2 - t1) - frac * (n2 - n1) * gamma) / (2 * frac * (n2 - n1))
    m = CM.CostModel(alpha=alpha, beta=beta, gamma=gamma)
    errs = [(n, CM.predict_allreduce_time("ring_rsa", n, p, m) / t - 1) for n, t in pts]
    fits[str(p)] = {"alpha": alpha, "beta": beta, "gamma": gamma,
                    "bus_gbps_asymptotic": round(1 / beta / 1e9, 1),
                    "max_abs_rel_err": round(max(abs(e) for _, e in errs), 3),
                    "rel_err_by_size": {str(n): round(e, 3) for n, e in errs},
                    "source": os.path.relpath(path, ROOT)}
    print(f"p={p}: alpha {alpha * 1e6:.2f} us, beta {beta * 1e12:.3f} ps/B "
          f"({1 / beta / 1e9:.0f} GB/s), gamma {gamma * 1e12:.3f} ps/B, "
          f"max |rel err| {fits[str(p)]['max_abs_rel_err']:.2f}")
out = {"fits": fits, "how": "tools/fit_costmodel.py on bench.py --mode sweep ring_rsa eager latencies "
                            "(CUDA events, max over ranks); the reference defaults are alpha 25 us, "
                            "beta 2 ns/B, gamma 1 ns/B (simcost.py:27-29)"}
json.dump(out, open(os.path.join(ROOT, "paper_1810_11112_b200", "costmodel.json"), "w"), indent=1)
