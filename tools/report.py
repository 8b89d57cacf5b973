"""Render BASELINE.md §5 rows from the committed sweep/refsweep CSVs.

    python tools/report.py profiles/r01
"""
import csv
import sys

SIZES = [8, 1024, 65536, 1048576, 16777216, 67108864, 268435456, 1073741824]
PEAK = 770.0


def load(path):
    try:
        return {int(r["message_bytes"]): r for r in csv.DictReader(open(path))}
    except OSError:
        return {}


def f(r, k):
    v = r.get(k, "")
    return float(v) if v not in ("", None) else None


def switch_for(p):
    import json
    try:
        return int(json.load(open("paper_1810_11112_b200/tuning.json"))["switch_bytes"][str(p)])
    except (OSError, KeyError, ValueError):
        return 131072


def main(prefix):
    print("| p | Bytes | dtype | Algo (auto) | This framework µs (graph / eager) | busBW GB/s | Roofline frac | "
          "NCCL µs (graph / eager) | NCCL busBW | Reference CPU ms (32-core host) | Parity |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in (2, 4):
        sw = load(f"{prefix}_sweep_p{p}.csv")
        ref = load(f"{prefix}_refsweep_p{p}.csv")
        for b in SIZES:
            r = sw.get(b)
            if r is None:
                continue
            algo = "rhd_rsa" if b < switch_for(p) else "ring_rsa"
            eager = min(x for x in (f(r, "rhd_rsa_us"), f(r, "rhd_rsa_zc_us"), f(r, "ring_rsa_us"),
                                    f(r, "ring_rsa_zc_us")) if x)
            graph = min([x for x in (f(r, "rhd_rsa_graph_us"), f(r, "ring_rsa_graph_us")) if x] or [None]) \
                if f(r, "rhd_rsa_graph_us") else None
            best = min(x for x in (eager, graph) if x)
            bus = b * 2 * (p - 1) / p / (best * 1e-6) / 1e9
            ng, ne = f(r, "nccl_graph_us"), f(r, "nccl_us")
            nb = b * 2 * (p - 1) / p / (min(x for x in (ng, ne) if x) * 1e-6) / 1e9
            refms = f"{float(ref[b]['mean_ms']):.3f}" if b in ref else "–"
            gtxt = f"{graph:.1f} / {eager:.1f}" if graph else f"– / {eager:.1f}"
            ntxt = f"{ng:.1f} / {ne:.1f}" if ng else f"– / {ne:.1f}"
            print(f"| {p} | {b} | fp32 | {algo} | {gtxt} | {bus:.1f} | {bus / PEAK:.3f} | {ntxt} | {nb:.1f} | "
                  f"{refms} | bit-exact (tests) |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01")
