"""Device timeline of one video through the CUPTI activity trace
(torch.profiler, CUDA activities only; the kernels are this repo's, launched
by libbp_cuda.so): kernel busy time, the idle gaps between consecutive
kernels on the compute stream, and the gap distribution.
    python tools/timeline_gaps.py [workload] > out.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_21070_b200 as bp  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "wan13-81"]
cfg = bp.PipelineConfig(devices=1, precision="bf16", layers=w["layers"], hidden=w["hidden"], heads=w["heads"],
                        ffn=w["ffn"], channels=w["channels"], height=w["height"], width=w["width"],
                        context_len=w["context_len"], num_b=w["num_b"], num_c=w["num_c"], steps=w["steps"],
                        blocks=w["blocks"])
p = bp.Pipeline(cfg)
p.run_device()
p.run_device()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    p.run_device()
    torch.cuda.synchronize()
kern = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "memcpy" not in e.name.lower() and \
            "memset" not in e.name.lower():
        kern.append((e.time_range.start, e.time_range.end, e.name))
kern.sort()
start, end = kern[0][0], max(k[1] for k in kern)
busy = 0.0
gaps = []
cur_s, cur_e = kern[0][0], kern[0][1]
for s, e, _ in kern[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append(s - cur_e)
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
gaps.sort()
n = len(gaps)
out = {"workload": w["name"], "kernels": len(kern), "span_ms": (end - start) / 1e3, "busy_ms": busy / 1e3,
       "idle_ms": (end - start - busy) / 1e3, "idle_frac": 1 - busy / (end - start), "gaps": n,
       "gap_us_p50": gaps[n // 2] if n else 0, "gap_us_p90": gaps[int(n * 0.9)] if n else 0,
       "gap_us_max": gaps[-1] if n else 0, "gaps_over_10us_ms": sum(g for g in gaps if g > 10) / 1e3,
       "gpu_ms_reported": p.stats()["gpu_ms"],
       "note": "CUPTI activity timestamps (torch.profiler, CUDA only); overlapping kernels (PDL) are merged; "
               "a gap is device time with none of this process's kernels running"}
print(json.dumps(out))
