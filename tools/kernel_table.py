"""Per-kernel evidence table from an ncu --csv launch capture (SpeedOfLight
section + DRAM bytes, SM clock, tensor / MUFU activity per launch):
    python tools/kernel_table.py capture.csv [hbm_peak_gbs] > table.json
For every kernel name: launches, mean device time, share of the captured
time, DRAM bytes per launch and the GB/s they imply, tensor-pipe and MUFU
activity. The launches are cold-cache and serialised under ncu, so shares
and per-launch figures are compared, not absolute step times."""
import collections
import csv
import json
import re
import sys


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def short(name):
    name = re.sub(r"\(.*$", "", name)                 # drop the argument list
    name = name.replace("(anonymous namespace)::", "").replace("bp::", "")
    return name.replace("void ", "").strip()


def main():
    path = sys.argv[1]
    hbm_peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6550.1
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per_launch = collections.defaultdict(dict)
    names = {}
    for r in rows:
        lid = r["ID"]
        names[lid] = short(r["Kernel Name"])
        unit = r.get("Metric Unit", "")
        v = num(r["Metric Value"])
        m = r["Metric Name"]
        if v is None:
            continue
        if m == "Duration" or m == "gpu__time_duration.sum":
            v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
            per_launch[lid]["us"] = v
        elif m == "dram__bytes_read.sum":
            per_launch[lid]["rd"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif m == "dram__bytes_write.sum":
            per_launch[lid]["wr"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif m == "sm__cycles_elapsed.avg.per_second":
            per_launch[lid]["ghz"] = v * {"Ghz": 1, "GHz": 1, "Mhz": 1e-3, "MHz": 1e-3, "hz": 1e-9}.get(unit, 1)
        elif m == "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active":
            per_launch[lid]["tensor"] = v
        elif m == "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active":
            per_launch[lid]["xu"] = v
        elif m in ("Compute (SM) Throughput", "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
            per_launch[lid]["sm_pct"] = v
        elif m in ("Memory Throughput", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"):
            per_launch[lid]["dram_pct"] = v
    agg = collections.defaultdict(list)
    for lid, d in per_launch.items():
        if "us" in d:
            agg[names[lid]].append(d)
    total_us = sum(d["us"] for ds in agg.values() for d in ds)
    out = []
    for name, ds in agg.items():
        n = len(ds)
        us = sum(d["us"] for d in ds) / n
        b = sum(d.get("rd", 0) + d.get("wr", 0) for d in ds) / n

        def mean(k):
            v = [d[k] for d in ds if k in d]
            return sum(v) / len(v) if v else None
        gbs = b / (us * 1e-6) / 1e9 if us > 0 else None
        out.append({"kernel": name, "launches": n, "us_per_launch": us, "share": n * us / total_us,
                    "dram_mb_per_launch": b / 1e6, "dram_gbs": gbs,
                    "dram_frac_of_hbm": gbs / hbm_peak if gbs else None,
                    "tensor_active_pct": mean("tensor"), "mufu_pct": mean("xu"),
                    "sm_throughput_pct": mean("sm_pct"), "memory_throughput_pct": mean("dram_pct"),
                    "sm_ghz": mean("ghz")})
    out.sort(key=lambda x: -x["share"])
    json.dump({"capture": path.split("/")[-1], "hbm_peak_gbs": hbm_peak, "launches": len(per_launch),
               "captured_us": total_us, "kernels": out}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
