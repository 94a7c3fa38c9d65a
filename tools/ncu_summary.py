"""Key metrics of an ncu --set full capture (.ncu-rep) as JSON: duration,
clock, tensor / MUFU / issue utilisation, DRAM bytes, registers, and the
top warp-stall reasons from the SASS source page.
    python tools/ncu_summary.py capture.ncu-rep [label] > summary.json"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "tensor_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_realtime_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "mufu_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
}


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h, units, v = raw[0], raw[1], raw[2]
    out = {"capture": rep.split("/")[-1], "label": sys.argv[2] if len(sys.argv) > 2 else "",
           "kernel": v[h.index("Kernel Name")]}
    for k, m in KEYS.items():
        if m in h:
            i = h.index(m)
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if k == "duration_us" and u in ("msecond", "ms"):
                val *= 1e3
            if k == "duration_us" and u in ("nsecond", "ns"):
                val /= 1e3
            if k.endswith("_mb") and u in ("Gbyte", "GB"):
                val *= 1e3
            if k.endswith("_mb") and u in ("Kbyte", "KB"):
                val /= 1e3
            if k == "sm_clock_ghz" and u in ("Mhz", "MHz", "cycle/usecond"):
                val /= 1e3
            out[k] = val
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    sh = src[1]
    cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    for r in src[2:]:
        for c in cols:
            try:
                agg[c] += int(r[sh.index(c)] or 0)
            except (ValueError, IndexError):
                pass
    tot = sum(agg.values()) or 1
    out["stall_share"] = {c: round(n / tot, 4) for c, n in agg.most_common(6)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
