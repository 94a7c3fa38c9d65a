#!/usr/bin/env python
"""Benchmark of the block-wise denoising path (DualParal) on B200.

A "step" is one whole video generation: noise pool build, all T + B - 1
denoising rounds of the layer pipeline, emission of every clean block. The
N=1 workload is BASELINE configs[1] (Wan2.1-1.3B-shape DiT, 81 frames 480p:
21 latent frames -> 3 blocks of 8 + 4 context frames, T = 50, 150 passes);
N>1 runs configs[2] (301 frames, 9 blocks) on the NCCL layer pipeline.
Weights are random-init of that architecture, latents are the reference's
synthetic noise pool; inputs larger than L2 (18720 x 1536 activations).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "s per 1025-frame video & frames/s at 1/2/4/8 B200; peak HBM GB/GPU"

WAN13 = dict(layers=30, hidden=1536, heads=12, ffn=8960, channels=64, height=30, width=52, context_len=512,
             num_b=8, num_c=8, steps=50)
WORKLOADS = {
    1: dict(WAN13, blocks=3, frames=81, name="Wan2.1-1.3B-shape 81f 480p (BASELINE configs[1])"),
    "multi": dict(WAN13, blocks=9, frames=301, name="Wan2.1-1.3B-shape 301f 480p (BASELINE configs[2])"),
    # wiring checks only (the mid parity config: 4 layers, h 256, 3 blocks x 6 steps)
    "tiny": dict(layers=8, hidden=256, heads=2, ffn=1024, channels=64, height=4, width=6, context_len=16,
                 num_b=8, num_c=8, steps=6, blocks=3, frames=41, name="8-layer mid parity shape (wiring check only)"),
    # the paper's headline video length (BASELINE configs[3] names 8 GPUs);
    # selectable at any N, e.g. N = 1 for the single-GPU reference point
    "wan13-1025": dict(WAN13, blocks=32, frames=1025, name="Wan2.1-1.3B-shape 1025f 480p (BASELINE configs[3] video)"),
}
# BASELINE configs[4] (14B, 1025 frames 720p, 8 GPUs): the 8-stage layer split
# on one GPU through the loopback transport, over a bounded sample of the
# schedule (2 blocks x 2 denoising steps = 4 passes at full 720p width).
WAN14 = dict(layers=40, hidden=5120, heads=40, ffn=13824, channels=64, height=45, width=80, context_len=512,
             num_b=8, num_c=8, steps=2, blocks=2, frames=None, devices=8,
             name="Wan2.1-14B-shape 720p, 8-stage split on 1 GPU (BASELINE configs[4] sample: 2 blocks x 2 steps)")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def pipeline_roofline(flops_video, n, peak_tflops, link_bytes_video, s_video, sched=None, layers=None):
    """Whole-pipeline roofline of one video: compute at the sustained bf16
    peak on N GPUs vs the busiest stage boundary's bytes over one NVLink
    direction (900 GB/s); frac = that ideal time / the measured time. With
    the schedule, also the schedule-aware bound: the makespan in
    slots (EventLog) x one slot of the largest stage at peak."""
    compute_s = flops_video / (n * peak_tflops * 1e12)
    nvlink_s = link_bytes_video / 900e9 if n > 1 else 0.0
    ideal = max(compute_s, nvlink_s)
    out = {"bound": "tensor" if compute_s >= nvlink_s else "nvlink", "compute_s": compute_s, "nvlink_s": nvlink_s,
           "ideal_s": ideal, "measured_s": s_video, "frac": ideal / s_video if s_video > 0 else None,
           "link_bytes_per_video": link_bytes_video, "peak_tflops": peak_tflops, "nvlink_gbs": 900.0}
    if sched is not None and layers:
        slots = int(sched.events[:, 0].max() - sched.events[:, 0].min()) + 1 if len(sched.events) else 0
        largest = max(e - b for b, e in sched.partition)
        slot_s = flops_video / sched.npasses * (largest / layers) / (peak_tflops * 1e12)
        out.update({"makespan_slots": slots, "largest_stage_layers": largest,
                    "schedule_aware_s": slots * slot_s,
                    "schedule_aware_frac": slots * slot_s / s_video if s_video > 0 else None})
    out["note"] = ("N = 1: no stage boundary, every stage on one GPU" if n == 1 else
                   f"N = {n}: busiest stage boundary over one NVLink direction")
    return out


def pass_flops(w, tokens, prefix, reference_algorithm=False):
    """Algorithmic FLOPs of one forward through all layers:
    4 S C h + L [8 S h^2 + 4 S Skv h + 4 S h^2 + 4 S Lc h + 4 S h F] (+ head),
    cross K/V hoisted. reference_algorithm adds what the reference recomputes
    every pass: ctx@Ck,Cv (model.cpp:216-217) and the captured K,V rows
    (model.cpp:321-322)."""
    S, h, F, C, Lc, L = tokens, w["hidden"], w.get("ffn") or 4 * w["hidden"], w["channels"], w["context_len"], w["layers"]
    skv = S + prefix
    per_layer = 2 * S * h * 3 * h + 2 * S * h * h + 4 * S * skv * h + 4 * S * h * h + 4 * S * Lc * h + 4 * S * h * F
    if reference_algorithm:
        per_layer += 4 * Lc * h * h + 4 * S * h * h
    return 2 * S * C * h + L * per_layer + 2 * S * h * C


def video_flops(w, sched, reference_algorithm=False):
    tpf = w["height"] * w["width"]
    S = (w["num_b"] + w["num_c"] // 2) * tpf
    P = (w["num_c"] // 2) * tpf
    n_prefix = sched.npasses - sched.rounds  # every pass except each round's tail pass
    return (n_prefix * pass_flops(w, S, P, reference_algorithm) +
            sched.rounds * pass_flops(w, S, 0, reference_algorithm)), n_prefix


def self_attn_flops(w, sched):
    tpf = w["height"] * w["width"]
    S = (w["num_b"] + w["num_c"] // 2) * tpf
    P = (w["num_c"] // 2) * tpf
    n_prefix = sched.npasses - sched.rounds
    return w["layers"] * (n_prefix * 4 * S * (S + P) * w["hidden"] + sched.rounds * 4 * S * S * w["hidden"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = str(gpu_index)
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [l.split(", ") for l in self.lines if l.split(", ")[0] == self.gpu]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def cpu_baseline(w, sched, threads=None, tokens_per_sample=16):
    """Times the UNMODIFIED reference forward_chunk (oracle/_ref) on a bounded
    sample: one Wan-width layer (h, heads, Lc, C) over `tokens_per_sample`
    tokens, `threads` independent samples in parallel, then extrapolates the
    video time as reference-algorithm FLOPs / measured FLOP rate."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import ref
    import paper_2505_21070_b200 as bp

    if not ref.available():
        return None
    threads = threads or min(os.cpu_count() or 1, 16)
    side = int(math.isqrt(tokens_per_sample))
    cfg = bp.PipelineConfig(layers=1, hidden=w["hidden"], heads=w["heads"], channels=w["channels"], height=side,
                            width=tokens_per_sample // side, context_len=w["context_len"], devices=1)
    chunks = [ref.RefChunk(cfg, 1, 0, 1, 3) for _ in range(threads)]
    rng = np.random.default_rng(0)
    payload = rng.standard_normal((tokens_per_sample, w["channels"]))

    def one(ch):
        ch.forward(payload, [10], [0], mode="off")

    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        list(ex.map(one, chunks))
        dt = time.perf_counter() - t0
    # the sample's own reference-algorithm FLOPs (reference FFN width 4h)
    wr = dict(w, layers=1, ffn=4 * w["hidden"])
    f_sample = pass_flops(wr, tokens_per_sample, 0, reference_algorithm=True)
    rate = threads * f_sample / dt  # FLOP/s over `threads` cores
    f_video, _ = video_flops(w, sched, reference_algorithm=True)
    sec_video = f_video / rate
    return {"value": w["frames"] / sec_video, "unit": "frames/s", "cores": threads, "kind": "reference",
            "sample": (f"{threads} x reference forward_chunk, 1 layer at h={w['hidden']} heads={w['heads']} "
                       f"Lc={w['context_len']} C={w['channels']}, {tokens_per_sample} tokens, fp64; "
                       f"{rate / 1e9 / threads:.3f} GFLOP/s/core over {dt:.1f} s, extrapolated to "
                       f"{f_video:.3e} reference FLOP per video"),
            "s_per_video_extrapolated": sec_video}


def run_wan14b(args):
    """Memory / feature-cache stress leg for configs[4]: all eight stages of
    the 14B layer split (5 layers each) resident on one GPU, S = 43200 tokens,
    Skv = 57600 on prefix passes. Reports seconds per pass, model TFLOP/s,
    peak HBM, and the configs[4] video time this rate implies on 8 GPUs
    (labelled a projection: schedule-aware makespan 1656 slots of one
    5-layer stage)."""
    import paper_2505_21070_b200 as bp
    w = WAN14
    cfg = bp.PipelineConfig(devices=w["devices"], precision="bf16", layers=w["layers"], hidden=w["hidden"],
                            heads=w["heads"], ffn=w["ffn"], channels=w["channels"], height=w["height"],
                            width=w["width"], context_len=w["context_len"], num_b=w["num_b"], num_c=w["num_c"],
                            steps=w["steps"], blocks=w["blocks"], transport="loopback")
    sched = bp.Schedule(cfg)
    fl_sample, n_prefix = video_flops(w, sched)
    t0 = time.perf_counter()
    pipe = bp.Pipeline(cfg)
    build_s = time.perf_counter() - t0
    for _ in range(max(1, args.warmup)):
        pipe.run_device()
    ms = []
    with ClockSampler(0) as clk:
        for _ in range(max(1, args.steps)):
            pipe.run_device()
            ms.append(pipe.stats()["gpu_ms"])
    st = pipe.stats()
    s_sample = statistics.mean(ms) / 1e3
    rate = fl_sample / s_sample
    # configs[4]: 32 blocks x 50 steps = 1600 passes; 8 even stages; makespan
    # T*B + N(N-1) = 1656 slots, one slot = one stage pass
    full = dict(w, steps=50, blocks=32)
    tpf = w["height"] * w["width"]
    S, P = (w["num_b"] + w["num_c"] // 2) * tpf, (w["num_c"] // 2) * tpf
    f_pass = pass_flops(full, S, P)
    slots = 50 * 32 + 8 * 7
    proj = slots * (f_pass / 8) / rate
    peaks, _ = load_peaks()
    print(json.dumps({
        "metric": "s per pass, Wan2.1-14B-shape 720p (configs[4] sample)", "value": s_sample / sched.npasses,
        "unit": "s/pass", "higher_is_better": False, "n_gpus": 1, "steps": max(1, args.steps),
        "warmup": max(1, args.warmup), "dtype": "bf16", "data": "synthetic (random-init 14B-shape weights)",
        "config": {"workload": w["name"], "layers": w["layers"], "hidden": w["hidden"], "heads": w["heads"],
                   "ffn": w["ffn"], "latent_grid": [w["height"], w["width"], w["channels"]],
                   "tokens_per_pass": S, "prefix_tokens": P, "passes": sched.npasses, "prefix_passes": n_prefix,
                   "stages": w["devices"]},
        "s_per_sample": s_sample, "model_tflops": rate / 1e12,
        "frac_of_sustained_peak": rate / 1e12 / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
        "peak_hbm_gb": st["peak_bytes"] / 1e9,
        "peak_hbm_note": "all eight 5-layer stages (weights, workspaces, KV caches) resident on this one GPU",
        "build_s": build_s,
        "projected_cfg4_8gpu_s_per_video": {"value": proj, "slots": slots, "flop_per_pass": f_pass,
                                            "note": "projection from this measured rate: 1656 slots x one 5-layer "
                                                    "stage pass; not a multi-GPU measurement"},
        "gpu_launches": st["kernel_launches"], "clocks": clk.summary()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1 stage-boundary transport: NCCL send/recv or CUDA-IPC peer copies")
    ap.add_argument("--workload", default="auto", choices=["auto", "wan14b", "wan13-301", "wan13-1025", "tiny"],
                    help="auto: configs[1] at N=1, configs[2] at N>1; wan13-301 / wan13-1025: those videos at "
                         "any N; wan14b: the configs[4] sample leg")
    args = ap.parse_args()
    if args.workload == "wan14b":
        return run_wan14b(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BP_BENCH_ONE_GPU") == "1" and world > 1:
        # wiring check of the N > 1 path on a single GPU: every rank on device
        # 0, NCCL told the ranks are separate hosts (socket transport); the
        # numbers are time-sliced and mean nothing
        local = 0
        os.environ["NCCL_HOSTID"] = f"blockpipe-bench-rank-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    n = max(args.gpus, world)
    if args.workload == "wan13-301":
        w = WORKLOADS["multi"]
    elif args.workload in ("wan13-1025", "tiny"):
        w = WORKLOADS[args.workload]
    else:
        w = WORKLOADS[1] if n == 1 else WORKLOADS["multi"]

    import paper_2505_21070_b200 as bp

    cfg = bp.PipelineConfig(devices=n, precision="bf16", layers=w["layers"], hidden=w["hidden"], heads=w["heads"],
                            ffn=w["ffn"], channels=w["channels"], height=w["height"], width=w["width"],
                            context_len=w["context_len"], num_b=w["num_b"], num_c=w["num_c"], steps=w["steps"],
                            blocks=w["blocks"], uneven_split=True,
                            transport=args.transport if n > 1 else "loopback")
    sched = bp.Schedule(cfg)
    fl_video, n_prefix = video_flops(w, sched)
    config = {"workload": w["name"], "layers": w["layers"], "hidden": w["hidden"], "heads": w["heads"],
              "ffn": w["ffn"], "latent_grid": [w["height"], w["width"], w["channels"]], "context_len": w["context_len"],
              "num_b": w["num_b"], "num_c": w["num_c"], "steps": w["steps"], "blocks": w["blocks"],
              "frames": w["frames"], "passes": sched.npasses, "prefix_passes": n_prefix,
              "parallelism": f"layer-pipeline x{n}" + (f" ({args.transport})" if n > 1 else ""), "l2": "inputs larger than L2 (18720x1536 activations per pass)"}

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        cb = None
        for _ in range(args.warmup):
            pass  # the reference has no warm-up state; each step is a fresh bounded sample
        t_all = time.perf_counter()
        for _ in range(args.steps):
            cb = cpu_baseline(w, sched)
            if cb is None:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbp_ref.so not built"}))
                return
            vals.append(cb["value"])
        value = statistics.mean(vals)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * (time.perf_counter() - t_all) / max(1, args.steps),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference random-init weights, coordinated noise pool)", "config": config,
            "cpu_baseline": cb, "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}))
        return

    dist = None
    ids = None
    exchange = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")

        def exchange(h):  # IPC transport: every rank's 64-byte handle, rank order
            got = [None] * world
            dist.all_gather_object(got, h)
            return got

        if args.transport == "nccl":
            obj = [None]
            if rank == 0:
                from paper_2505_21070_b200._lib import lib
                import ctypes
                buf = bytearray()
                for _ in range(n):
                    b = (ctypes.c_uint8 * 128)()
                    assert lib.bp_nccl_unique_id(b) == 0
                    buf += bytes(b)
                obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0)
            ids = obj[0]

    t_build = time.perf_counter()
    pipe = bp.Pipeline(cfg, rank=rank, world=world, device=local, nccl_ids=ids, ipc_exchange=exchange)
    build_s = time.perf_counter() - t_build

    def barrier():
        if dist is not None:
            dist.barrier()

    n_warm = max(3, args.warmup) if args.workload == "auto" else max(1, args.warmup)
    for _ in range(n_warm):
        pipe.run_device()
    barrier()
    lib_launch = []
    gpu_ms = []
    prof = {"attn_ms": 0.0, "gemm_ms": 0.0, "cross_ms": 0.0, "ln_ms": 0.0, "attn_launches": 0, "gemm_launches": 0,
            "ln_launches": 0}
    from paper_2505_21070_b200._lib import lib
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            pipe.run_device()
            st = pipe.stats()
            gpu_ms.append(st["gpu_ms"])
            lib_launch.append(st["kernel_launches"])
    barrier()
    # one more video, untimed, with CUDA events around every class of launches
    # (self-attention, cross-attention, GEMMs, LayerNorm) for the rooflines and
    # the breakdown; the timed steps above carry no profiling events
    lib.bp_pipeline_set_profiling(pipe._h, 1)
    pipe.run_device()
    st = pipe.stats()
    for k in prof:
        prof[k] = st[k]
    prof_video_s = st["gpu_ms"] / 1e3
    lib.bp_pipeline_set_profiling(pipe._h, 0)
    barrier()
    ms = statistics.mean(gpu_ms)
    if dist is not None:
        import torch
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stats = pipe.stats()
    link_bytes = float(stats["boundary_bytes"])  # this rank's stage-boundary bytes of the last video
    if dist is not None:
        import torch
        t = torch.tensor([link_bytes], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # busiest stage-boundary link
        link_bytes = float(t.item())

    # e2e: the public API with host buffers. Rank 0 hands the engine the
    # reference's noise pool from pinned host memory (bp_pipeline_set_pool;
    # uploaded host->device inside every run) and receives every emitted
    # block's latents back in host memory; wall clock per step, max over ranks.
    pool = None
    if rank == 0:
        m = w["num_b"] + w["num_c"] // 2
        pool = bp.pinned_empty((m, w["height"], w["width"], w["channels"]))
        pool[...] = bp.build_pool(w["num_b"], w["num_c"], (w["height"], w["width"], w["channels"]),
                                  bp.derive_seed(cfg.seed_noise, [0]), device=local)
        pipe.set_pool(pool)
    e2e_vals = []
    h2d = d2h = 0
    for _ in range(max(1, min(args.steps, 2))):
        barrier()
        t0 = time.perf_counter()
        blocks = pipe.run()
        barrier()
        dt = time.perf_counter() - t0
        if dist is not None:
            import torch
            tt = torch.tensor([dt], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_vals.append(w["frames"] / dt)
        est = pipe.stats()
        h2d, d2h = est["h2d_bytes"], est["d2h_bytes"]
    if pool is not None:
        pipe.set_pool(None)

    if rank != 0:
        return
    peaks, peak_kind = load_peaks()
    attn_fl = self_attn_flops(w, sched)
    attn_s = prof["attn_ms"] / 1e3
    achieved = attn_fl / attn_s / 1e12 if attn_s > 0 else None
    peak = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "attn_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    cpu = None if args.no_cpu_baseline else cpu_baseline(w, sched)
    s_video = ms / 1e3
    tokens_per_pass = (w["num_b"] + w["num_c"] // 2) * w["height"] * w["width"]
    out = {
        "metric": METRIC, "value": w["frames"] / s_video, "unit": "frames/s", "n_gpus": n, "steps": args.steps,
        "warmup": n_warm, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if n > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init Wan2.1-1.3B-shape weights, reference coordinated noise pool)",
        "config": config,
        "s_per_video": s_video, "latent_frames_per_s": sum(b["frames"] for b in sched.blocks) / s_video,
        "peak_hbm_gb": stats["peak_bytes"] / 1e9,
        "model_tflops": fl_video / s_video / 1e12,
        "roofline": {"bound": "tensor", "kernel": "k_attn_pp2 (self-attention, tcgen05 ping-pong on a cta_group::2 pair)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_kind": f"{peak_kind} sustained (kernel timed inside a long step)",
                     "timing": "CUDA events around every launch of the class, in one extra video right after the timed steps (events inside the timed steps would perturb launch overlap)",
                     "share_of_step": attn_s / prof_video_s,
                     "gemm_tflops": None if prof["gemm_ms"] <= 0 else
                     (fl_video - self_attn_flops(w, sched)) / (prof["gemm_ms"] / 1e3) / 1e12,
                     "whole_step_frac": fl_video / s_video / 1e12 / peak},
        # north_star: the elementwise path against HBM bandwidth -- the
        # LayerNorm kernel (fp32 residual row in, bf16 operand row out: 6 B per
        # element algorithmic), device time from CUDA events in the timed steps
        "elementwise_roofline": None if prof["ln_ms"] <= 0 else {
            "bound": "hbm", "kernel": "k_ln_bf16_reg (LayerNorm + affine, fp32 -> bf16)",
            "achieved": prof["ln_launches"] * tokens_per_pass * w["hidden"] * 6 / (prof["ln_ms"] / 1e3) / 1e9,
            "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": prof["ln_launches"] * tokens_per_pass * w["hidden"] * 6 / (prof["ln_ms"] / 1e3) / 1e9 / peaks["hbm_gbs"],
            "bytes_per_launch": tokens_per_pass * w["hidden"] * 6, "share_of_step": prof["ln_ms"] / 1e3 / prof_video_s,
            "note": "event windows around each launch include the launch gap; ncu kernel time is lower "
                    "(profiles/r01b_summary.md)"},
        # where the device time of a step goes (CUDA events around each class of
        # launches on the compute stream; "rest" = embedding, capture copies,
        # head, Euler steps, gathers and the gaps between launches)
        "step_breakdown_s": {
            "video_s_with_events": prof_video_s,
            "self_attention": prof["attn_ms"] / 1e3, "cross_attention": prof["cross_ms"] / 1e3,
            "gemm": prof["gemm_ms"] / 1e3, "layernorm": prof["ln_ms"] / 1e3,
            "rest": prof_video_s - (prof["attn_ms"] + prof["cross_ms"] + prof["gemm_ms"] + prof["ln_ms"]) / 1e3},
        "cpu_baseline": cpu,
        "e2e": {"value": statistics.mean(e2e_vals), "unit": "frames/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "wall clock per video through bp_pipeline_run: the noise pool uploaded from pinned host "
                        "memory (bp_pipeline_set_pool) and every emitted block copied back to host"},
        # north_star: the slower of compute at peak and stage-boundary bytes over
        # NVLink (900 GB/s per direction) bounds the whole pipeline
        "pipeline_roofline": pipeline_roofline(fl_video, n, peak, link_bytes, s_video, sched, w["layers"]),
        "gpu_launches": int(statistics.mean(lib_launch)),
        "clocks": clk.summary(),
        "build_s": build_s,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
