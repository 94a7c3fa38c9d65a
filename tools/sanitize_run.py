"""Small launches of every kept device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck) runs (tests/test_gpu_sanitizer.py):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [part]

part: "kernels" (tcgen05 GEMM epilogues, pair / single-CTA attention with and
without a prefix segment, LayerNorm, through the kernel self-test library),
"pipeline" (a bf16 and an fp32 two-stage loopback run of the mid config:
embedding, capture copies, fp32 flash attention and tile GEMM, Euler steps;
and a bf16 run of the optional Wan block),
or "all" (default). Shapes are small: the sanitizer instruments every access.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from kernels import attn, attn_cross, gemm, load_testlib, to_bf16_bits  # noqa: E402


def kernels():
    lib = load_testlib()
    rng = np.random.default_rng(0)
    for epi in (0, 1, 2, 3):  # k_gemm_pair<epi, cg2>: bf16 store, erf-GELU, fp32 residual (TMA reduce-add), fp32 store
        M, N, K = 300, 512, 128
        A = to_bf16_bits(rng.standard_normal((M, K)))
        W = to_bf16_bits(rng.standard_normal((N, K)) / 10)
        C0 = np.zeros((M, N), dtype=np.uint16) if epi in (0, 1) else np.zeros((M, N), dtype=np.float32)
        gemm(lib, A, W, C0, epi)
    H = 2 * 128
    for rows, n0, n1 in ((300, 200, 300), (257, 0, 129)):  # k_attn_pp2 with / without the prefix segment
        q = to_bf16_bits(rng.standard_normal((rows, H)))
        k1, v1 = to_bf16_bits(rng.standard_normal((n1, H))), to_bf16_bits(rng.standard_normal((n1, H)))
        k0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
        v0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
        attn(lib, q, k0, v0, k1, v1, 2, 128, 0.088)
    q = to_bf16_bits(rng.standard_normal((300, H)))
    kc, vc = to_bf16_bits(rng.standard_normal((512, H))), to_bf16_bits(rng.standard_normal((512, H)))
    attn_cross(lib, q, kc, vc, 2, 128, 0.088)  # k_attn_ps (cross-attention, persistent)
    import ctypes
    ms = ctypes.c_double()
    assert lib.bp_bench_ln(0, 300, 1536, 1, ctypes.byref(ms)) == 0  # k_ln_bf16_reg


def pipeline():
    import paper_2505_21070_b200 as bp
    base = dict(devices=2, layers=2, hidden=256, heads=2, channels=64, height=4, width=6, context_len=16, num_b=8,
                num_c=8, steps=2, blocks=2, mode="single")
    for prec in ("bf16", "f32"):
        out = bp.run_pipeline(dict(base, precision=prec))
        assert all(np.isfinite(b["frames"]).all() for b in out["blocks"])
    # the optional Wan block (dh = 128: modulated LayerNorm, the q/k RMSNorm +
    # 3D RoPE kernel, gated-residual and tanh-GELU GEMM epilogues)
    out = bp.run_pipeline(dict(base, precision="bf16", block="wan"))
    assert all(np.isfinite(b["frames"]).all() for b in out["blocks"])


if __name__ == "__main__":
    part = sys.argv[1] if len(sys.argv) > 1 else "all"
    if part in ("kernels", "all"):
        kernels()
    if part in ("pipeline", "all"):
        pipeline()
    print("sanitize_run ok")
