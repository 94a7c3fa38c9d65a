"""Runs the bench workload (Wan2.1-1.3B-shape, 81 frames 480p, bf16) for a
given number of videos, for ncu launch lists / kernel captures:
    ncu ... python tools/profile_pass.py [videos]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2505_21070_b200 as bp  # noqa: E402

w = bench.WORKLOADS["wan13-81"]
cfg = bp.PipelineConfig(devices=1, precision="bf16", layers=w["layers"], hidden=w["hidden"], heads=w["heads"],
                        ffn=w["ffn"], channels=w["channels"], height=w["height"], width=w["width"],
                        context_len=w["context_len"], num_b=w["num_b"], num_c=w["num_c"], steps=w["steps"],
                        blocks=w["blocks"])
p = bp.Pipeline(cfg)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    p.run_device()
print("gpu_ms", p.stats()["gpu_ms"])
