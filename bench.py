#!/usr/bin/env python
"""Benchmark of the block-wise denoising path (DualParal) on B200.

A "step" is one whole video generation: noise pool build, all T + B - 1
denoising rounds of the layer pipeline, emission of every clean block. Every
N runs the same workload, BASELINE configs[2] (Wan2.1-1.3B-shape DiT, 301
frames 480p: 76 latent frames -> 9 blocks of 8 + 4 context frames, T = 50,
450 passes), so a 1 -> 8 GPU curve is strong scaling of one video.
Weights are random-init of that architecture, latents are the reference's
synthetic noise pool; inputs larger than L2 (18720 x 1536 activations).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (the
unmodified reference library compiled into oracle/_ref) on this host; it
never imports this repo's package or loads its CUDA library.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "s per 1025-frame video & frames/s at 1/2/4/8 B200; peak HBM GB/GPU"

WAN13 = dict(layers=30, hidden=1536, heads=12, ffn=8960, channels=64, height=30, width=52, context_len=512,
             num_b=8, num_c=8, steps=50)
WORKLOADS = {
    "wan13-301": dict(WAN13, blocks=9, frames=301, name="Wan2.1-1.3B-shape 301f 480p (BASELINE configs[2])"),
    "wan13-81": dict(WAN13, blocks=3, frames=81, name="Wan2.1-1.3B-shape 81f 480p (BASELINE configs[1])"),
    # the paper's headline video length (BASELINE configs[3] names 8 GPUs)
    "wan13-1025": dict(WAN13, blocks=32, frames=1025, name="Wan2.1-1.3B-shape 1025f 480p (BASELINE configs[3] video)"),
    # wiring checks only (8 layers at the mid parity shape, 3 blocks x 6 steps)
    "tiny": dict(layers=8, hidden=256, heads=2, ffn=1024, channels=64, height=4, width=6, context_len=16,
                 num_b=8, num_c=8, steps=6, blocks=3, frames=41, name="8-layer mid parity shape (wiring check only)"),
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


# ---- the reference's CPU implementation (oracle/_ref: the UNMODIFIED reference
# library), used by --impl reference and by the cpu_baseline leg ---------------------
REF_DEFAULTS = dict(devices=2, order="reverse", cache="on", threaded=True, num_b=2, num_c=4, steps=8, blocks=6,
                    retain_clean_context=True, layers=4, hidden=16, heads=2, channels=2, height=2, width=2,
                    context_len=4, strategy="coordinated", seed_model=1, seed_noise=2, seed_context=3,
                    fault_inject=False, record_trace=False, check_cache=False)  # engine.hpp:24-38, model.hpp:21-28


def ref_config(**kw):
    """A PipelineConfig as the reference spells it (no import of this repo's package)."""
    return SimpleNamespace(**dict(REF_DEFAULTS, **kw))


def ref_schedule(w, n):
    """Passes and rounds of the workload's schedule from the reference's own
    run_pipeline (engine.cpp:255-497), run at a schedule-only width (1 x 1
    latent grid, h 8): they depend on T, Block_num, num_b, num_c and N only."""
    from oracle import ref
    cfg = ref_config(devices=n, layers=n, hidden=8, heads=2, channels=1, height=1, width=1, context_len=2,
                     num_b=w["num_b"], num_c=w["num_c"], steps=w["steps"], blocks=w["blocks"], threaded=False)
    out = ref.run(cfg)
    passes = len(out["events"]) // n
    return SimpleNamespace(npasses=passes, rounds=int(out["rounds"]))


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except Exception:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    return {"nproc": cores, "cpu_model": model, "glibc": "-".join(platform.libc_ver())}


def reference_legs(include_mid):
    """End-to-end reference run_pipeline legs: configs[0]
    (tiny DiT, 2 layers, d 128, 4 heads, 4 blocks x 10 steps) best of 5, single-
    threaded (1 device) and threaded (2 device threads + coordinator,
    engine.cpp:280-285); optionally the mid parity config (4 layers, h 256,
    4 x 6 grid, C 64, 3 blocks x 6 steps) once each, 1 and 4 devices."""
    from oracle import ref

    def best(cfg, reps):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            ref.run(cfg)
            ts.append(time.perf_counter() - t0)
        return min(ts)

    cfg1 = dict(layers=2, hidden=128, heads=4, steps=10, blocks=4)
    legs = {"configs0_single_thread_s": best(ref_config(**cfg1, devices=1, threaded=False), 5),
            "configs0_threaded_2dev_s": best(ref_config(**cfg1, devices=2, threaded=True), 5),
            "configs0_note": "reference run_pipeline end to end, best of 5 (wall clock)"}
    if include_mid:
        mid = dict(layers=4, hidden=256, heads=2, channels=64, height=4, width=6, context_len=16, num_b=8, num_c=8,
                   steps=6, blocks=3)
        legs["mid_single_thread_s"] = best(ref_config(**mid, devices=1, threaded=False), 1)
        legs["mid_threaded_4dev_s"] = best(ref_config(**mid, devices=4, threaded=True), 1)
        legs["mid_note"] = "mid parity config (SURVEY Appendix A), reference run_pipeline end to end, once"
    return legs


class RefSample:
    """The bounded sample of the workload on the reference: the UNMODIFIED
    reference forward_chunk of one Wan-width layer (h, heads, Lc, C) over
    `tokens` tokens, `threads` chunks in parallel (one per host core). The
    chunks (weights drawn by the reference, model.cpp:87-128) are built once;
    each call times one forward per chunk and extrapolates the video time as
    reference-algorithm FLOPs / measured FLOP rate."""

    def __init__(self, w, sched, threads=None, tokens=16):
        from oracle import ref
        self.w, self.sched, self.tokens = w, sched, tokens
        self.threads = threads or min(host_info()["nproc"], 16)
        side = int(math.isqrt(tokens))
        cfg = ref_config(layers=1, hidden=w["hidden"], heads=w["heads"], channels=w["channels"], height=side,
                         width=tokens // side, context_len=w["context_len"], devices=1)
        self.chunks = [ref.RefChunk(cfg, 1, 0, 1, 3) for _ in range(self.threads)]
        import numpy as np
        self.payload = np.random.default_rng(0).standard_normal((tokens, w["channels"]))

    def measure(self):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(self.threads) as ex:
            t0 = time.perf_counter()
            list(ex.map(lambda ch: ch.forward(self.payload, [10], [0], mode="off"), self.chunks))
            dt = time.perf_counter() - t0
        w = self.w
        # the sample's own reference-algorithm FLOPs (reference FFN width 4h)
        f_sample = pass_flops(dict(w, layers=1, ffn=4 * w["hidden"]), self.tokens, 0, reference_algorithm=True)
        rate = self.threads * f_sample / dt  # FLOP/s over `threads` cores
        f_video, _ = video_flops(w, self.sched, reference_algorithm=True)
        sec_video = f_video / rate
        return {"value": w["frames"] / sec_video, "unit": "frames/s", "cores": self.threads, "kind": "reference",
                "sample": (f"{self.threads} x reference forward_chunk, 1 layer at h={w['hidden']} heads={w['heads']} "
                           f"Lc={w['context_len']} C={w['channels']}, {self.tokens} tokens, fp64; "
                           f"{rate / 1e9 / self.threads:.3f} GFLOP/s/core over {dt:.1f} s, extrapolated to "
                           f"{f_video:.3e} reference FLOP per video ({self.sched.npasses} passes, "
                           f"{self.sched.rounds} rounds from the reference's own schedule)"),
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


def reference_arm(args, w, n, rank):
    """--impl reference: the reference's CPU implementation on this host
    (rank 0 only; other ranks exit without work). Each step is one bounded
    sample of the workload (RefSample, ~10-15 s); measured end-to-end legs
    of the reference's own CPU configs are reported beside it."""
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbp_ref.so not built"}))
        return
    sched = ref_schedule(w, n)
    sample = RefSample(w, sched)
    legs = reference_legs(include_mid=not args.quick_reference)
    for _ in range(args.warmup):
        pass  # the reference keeps no state between samples: nothing to warm
    vals, ms = [], []
    cb = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = sample.measure()
        ms.append(1000 * (time.perf_counter() - t0))
        vals.append(cb["value"])
    value = statistics.mean(vals)
    cb = dict(cb, value=value, measured_legs=legs, host=host_info())
    try:  # evidence that this arm ran the reference library only (no repo CUDA library mapped)
        with open("/proc/self/maps") as f:
            cb["repo_libraries_loaded"] = sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")
                                                  and ln.split()[-1].startswith(ROOT)})
    except Exception:
        pass
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(ms),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference random-init weights, coordinated noise pool)",
        "config": workload_config(w, n, sched, args),
        "cpu_baseline": cb, "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                                     "d2h_bytes_per_step": 0}}))


def workload_config(w, n, sched, args):
    return {"workload": w["name"], "layers": w["layers"], "hidden": w["hidden"], "heads": w["heads"],
            "ffn": w["ffn"], "latent_grid": [w["height"], w["width"], w["channels"]], "context_len": w["context_len"],
            "num_b": w["num_b"], "num_c": w["num_c"], "steps": w["steps"], "blocks": w["blocks"],
            "frames": w["frames"], "passes": sched.npasses, "prefix_passes": sched.npasses - sched.rounds,
            "parallelism": f"layer-pipeline x{n}" + (f" ({args.transport})" if n > 1 else ""),
            "l2": "inputs larger than L2 (18720x1536 activations per pass)",
            **({"block": "wan (optional non-parity Wan2.1-style block)"} if getattr(args, "block", "reference") == "wan"
               else {})}


def attn_isolated_roofline(device, w, sched, peaks):
    """The dominant kernel timed alone (the burst peak is its denominator):
    20 back-to-back k_attn_pp2 launches at the workload's prefix-pass shape
    (q = S, kv = P + S), CUDA events on the launching stream, through the
    kernel self-test library (same objects as libbp_cuda.so). Inside the step
    the same kernel runs under the power cap and is judged against the
    sustained peak (roofline.frac)."""
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from kernels import load_testlib
    tpf = w["height"] * w["width"]
    S, P = (w["num_b"] + w["num_c"] // 2) * tpf, (w["num_c"] // 2) * tpf
    dh = w["hidden"] // w["heads"]
    ms = ctypes.c_double()
    if load_testlib().bp_bench_attn(device, S, w["heads"], dh, P, S, 20, ctypes.byref(ms)) != 0:
        return None
    tf = 4 * S * (P + S) * w["hidden"] / (ms.value * 1e-3) / 1e12
    return {"achieved": tf, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": tf / peaks["bf16_tflops"],
            "peak_kind": "measured burst (kernel timed alone)", "us_per_launch": ms.value * 1e3,
            "shape": f"q {S} x kv {P}+{S}, {w['heads']} heads, dh {dh}",
            "timing": "20 back-to-back launches after the timed videos, CUDA events on the launching stream"}


def ln_kernel_roofline(device, tokens, hidden, peaks):
    """LayerNorm (the elementwise path's largest kernel) from kernel time:
    back-to-back launches on [tokens, hidden] fp32 -> bf16 (larger than L2),
    CUDA events on the launching stream, through the kernel self-test library
    (built from the same objects as libbp_cuda.so)."""
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from kernels import load_testlib
    ms = ctypes.c_double()
    if load_testlib().bp_bench_ln(device, tokens, hidden, 20, ctypes.byref(ms)) != 0:
        return None
    bytes_launch = tokens * hidden * 6 + 2 * hidden * 4  # x read (fp32) + y written (bf16) + g, b
    gbs = bytes_launch / (ms.value * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "k_ln_bf16_reg (LayerNorm + affine, fp32 -> bf16)", "achieved": gbs,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"], "bytes_per_launch": bytes_launch,
            "us_per_launch": ms.value * 1e3,
            "timing": "kernel time: 20 back-to-back launches on device-resident [tokens, hidden] (inputs > L2), "
                      "CUDA events on the launching stream"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick-reference", action="store_true",
                    help="reference arm without the mid-config end-to-end legs (~2 min of CPU)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1 stage-boundary transport: NCCL send/recv or CUDA-IPC peer copies")
    ap.add_argument("--workload", default="wan13-301", choices=["wan13-301", "wan13-81", "wan13-1025", "tiny",
                                                                "wan14b"],
                    help="wan13-301 (default, every N): configs[2]; wan13-81: configs[1]; wan13-1025: the "
                         "configs[3] video at any N; wan14b: the configs[4] sample leg")
    ap.add_argument("--block", default="reference", choices=["reference", "wan"],
                    help="reference (the parity block, default) or wan: the optional non-parity Wan2.1-style block "
                         "(adaLN modulation, RMSNorm + 3D RoPE on Q/K, gated residuals; a labelled extra)")
    args = ap.parse_args()
    if args.workload == "wan14b":
        return run_wan14b(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(args.gpus, world)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, w, n, rank)

    if os.environ.get("BP_BENCH_ONE_GPU") == "1" and world > 1:
        # wiring check of the N > 1 path on a single GPU: every rank on device
        # 0, NCCL told the ranks are separate hosts (socket transport); the
        # numbers are time-sliced and mean nothing
        local = 0
        os.environ["NCCL_HOSTID"] = f"blockpipe-bench-rank-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

    import paper_2505_21070_b200 as bp

    cfg = bp.PipelineConfig(devices=n, precision="bf16", layers=w["layers"], hidden=w["hidden"], heads=w["heads"],
                            ffn=w["ffn"], channels=w["channels"], height=w["height"], width=w["width"],
                            context_len=w["context_len"], num_b=w["num_b"], num_c=w["num_c"], steps=w["steps"],
                            blocks=w["blocks"], uneven_split=True, block=args.block,
                            transport=args.transport if n > 1 else "loopback")
    sched = bp.Schedule(cfg)
    fl_video, n_prefix = video_flops(w, sched)
    config = workload_config(w, n, sched, args)

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
                obj = [bp.nccl_unique_ids(n)]
            dist.broadcast_object_list(obj, src=0)
            ids = obj[0]

    t_build = time.perf_counter()
    pipe = bp.Pipeline(cfg, rank=rank, world=world, device=local, nccl_ids=ids, ipc_exchange=exchange)
    build_s = time.perf_counter() - t_build

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        import torch
        t = torch.tensor([float(v)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up videos (untimed); the last one carries CUDA events around every
    # class of launches (self-attention, cross-attention, GEMMs, LayerNorm) for
    # the roofline and the breakdown -- the timed videos carry none
    n_warm = max(3, args.warmup)
    for i in range(n_warm):
        pipe.set_profiling(i == n_warm - 1)
        pipe.run_device()
        if i == n_warm - 1:
            prof = pipe.stats()
    pipe.set_profiling(False)
    barrier()
    lib_launch, gpu_ms = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            pipe.run_device()
            st = pipe.stats()
            gpu_ms.append(st["gpu_ms"])
            lib_launch.append(st["kernel_launches"])
    barrier()
    ms = max_over_ranks(statistics.mean(gpu_ms))
    stats = pipe.stats()
    link_bytes = max_over_ranks(stats["boundary_bytes"])  # busiest stage-boundary link of one video

    # e2e: the public API with host buffers. Rank 0 hands the engine the
    # reference's noise pool from pinned host memory (bp_pipeline_set_pool;
    # uploaded host->device inside the run) and receives every emitted block's
    # latents back in host memory; wall clock of the video, max over ranks.
    pool = None
    if rank == 0:
        m = w["num_b"] + w["num_c"] // 2
        pool = bp.pinned_empty((m, w["height"], w["width"], w["channels"]))
        pool[...] = bp.build_pool(w["num_b"], w["num_c"], (w["height"], w["width"], w["channels"]),
                                  bp.derive_seed(cfg.seed_noise, [0]), device=local)
        pipe.set_pool(pool)
    barrier()
    t0 = time.perf_counter()
    pipe.run()
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    est = pipe.stats()
    h2d, d2h = est["h2d_bytes"], est["d2h_bytes"]
    if pool is not None:
        pipe.set_pool(None)
    if dist is not None:  # no collectives after this point
        dist.destroy_process_group()

    if rank != 0:
        return
    peaks, peak_kind = load_peaks()
    prof_video_s = prof["gpu_ms"] / 1e3
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
    cpu = None
    if n == 1 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            cpu = RefSample(w, sched).measure()
            cpu["measured_legs"] = reference_legs(include_mid=False)
            cpu["host"] = host_info()
    s_video = ms / 1e3
    tokens_per_pass = (w["num_b"] + w["num_c"] // 2) * w["height"] * w["width"]
    out = {
        "metric": METRIC, "value": w["frames"] / s_video, "unit": "frames/s", "n_gpus": n, "steps": args.steps,
        "warmup": n_warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init Wan2.1-1.3B-shape weights, reference coordinated noise pool)",
        "config": config,
        "s_per_video": s_video, "latent_frames_per_s": sum(b["frames"] for b in sched.blocks) / s_video,
        "peak_hbm_gb": stats["peak_bytes"] / 1e9,
        "model_tflops": fl_video / s_video / 1e12,
        "roofline": {"bound": "tensor", "kernel": "k_attn_pp2 (self-attention, tcgen05 ping-pong on a cta_group::2 pair)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_kind": f"{peak_kind} sustained (kernel timed inside a long step)",
                     "frac_of_burst": (achieved / peaks["bf16_tflops"]) if achieved else None,
                     "timing": "CUDA events around every launch of the class in the last warm-up video (events "
                               "inside the timed videos would perturb launch overlap)",
                     "share_of_step": attn_s / prof_video_s,
                     "gemm_tflops": None if prof["gemm_ms"] <= 0 else
                     (fl_video - attn_fl) / (prof["gemm_ms"] / 1e3) / 1e12,
                     "whole_step_frac": fl_video / s_video / 1e12 / peak,
                     "isolated": attn_isolated_roofline(local, w, sched, peaks)},
        # north_star: the elementwise path against HBM bandwidth, from kernel time
        "elementwise_roofline": ln_kernel_roofline(local, tokens_per_pass, w["hidden"], peaks),
        # where the device time of a video goes (CUDA events around each class of
        # launches on the compute stream; "rest" = embedding, capture copies,
        # head, Euler steps, gathers and the gaps between launches)
        "step_breakdown_s": {
            "video_s_with_events": prof_video_s,
            "self_attention": prof["attn_ms"] / 1e3, "cross_attention": prof["cross_ms"] / 1e3,
            "gemm": prof["gemm_ms"] / 1e3, "layernorm": prof["ln_ms"] / 1e3,
            "rest": prof_video_s - (prof["attn_ms"] + prof["cross_ms"] + prof["gemm_ms"] + prof["ln_ms"]) / 1e3},
        "cpu_baseline": cpu,
        "e2e": {"value": w["frames"] / e2e_s, "unit": "frames/s", "s_per_video": e2e_s,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "wall clock of one video through bp_pipeline_run: the noise pool uploaded from pinned host "
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
