"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches, total time and share.
    python tools/launch_summary.py launches.csv [--json out.json]"""
import collections
import csv
import json
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * scale[r[ui]]
        name = r[ki].replace("void ", "").split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(t for _, t in agg.values())
    out = [{"kernel": k, "launches": n, "ms": t / 1e3, "share": t / total, "avg_us": t / n}
           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    return out, total / 1e3


if __name__ == "__main__":
    table, total_ms = summarise(sys.argv[1])
    for e in table:
        print(f"{e['ms']:10.2f} ms {100 * e['share']:5.1f}%  n={e['launches']:5d}  avg {e['avg_us']:9.1f} us  {e['kernel']}")
    print(f"total {total_ms:.1f} ms")
    if "--json" in sys.argv:
        json.dump({"total_ms": total_ms, "kernels": table}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
