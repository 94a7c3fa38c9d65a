"""Kernel micro-benchmarks through the self-test hooks (include/bp_cuda_test.h),
used for A/B runs and ncu captures:
    python tools/bench_kernels.py attn|gemm|all [iters]
Attention: the stage's kernels (self-attention: the cta_group::2 pair
kernel k_attn_pp2; "cross": the persistent cross-attention kernel k_attn_ps)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from kernels import load_testlib  # noqa: E402

lib = load_testlib()

what = sys.argv[1] if len(sys.argv) > 1 else "attn"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
only = sys.argv[3] if len(sys.argv) > 3 else ""  # substring filter on the case tag
ms = ctypes.c_double()
impl = "default"
if what in ("attn", "all"):
    # (rows, heads, dh, prefix n0, block n1): prefix pass, plain pass, cross-attention
    for rows, n0, n1, tag in ((18720, 6240, 18720, "self+prefix"), (18720, 0, 18720, "self"),
                              (18720, 0, 512, "cross")):
        if only not in tag:
            continue
        # bp_bench_attn times the attention launcher of the current implementation
        # id: 4 = the self-attention pair kernel, 2 = the cross-attention kernel
        lib.bp_set_kernel_impl(3, 2 if tag == "cross" else 4)
        assert lib.bp_bench_attn(0, rows, 12, 128, n0, n1, iters, ctypes.byref(ms)) == 0
        lib.bp_set_kernel_impl(3, 4)
        tf = 4 * rows * (n0 + n1) * 1536 / ms.value / 1e9
        print(f"attn impl={impl} {tag:12s} ms {ms.value:.4f} TF {tf:.1f}")
if what in ("gemm", "all"):
    for m, n, k, epi, tag in ((18720, 4608, 1536, 0, "qkv bf16"), (18720, 1536, 1536, 2, "o resid"),
                              (18720, 8960, 1536, 1, "ffn1 gelu"), (18720, 1536, 8960, 2, "ffn2 resid"),
                              (18720, 1536, 8960, 6, "ffn2 resid-out (fused send)")):
        if only not in tag:
            continue
        assert lib.bp_bench_gemm(0, m, n, k, epi, iters, ctypes.byref(ms)) == 0
        print(f"gemm {tag:10s} {m}x{n}x{k} ms {ms.value:.4f} TF {2 * m * n * k / ms.value / 1e9:.1f}")
if what in ("wan", "all"):
    # the Wan block's Q/K RMSNorm + 3D RoPE (bf16, in place on the QKV buffer):
    # algorithmic bytes = q and k read once and written once
    rows, h = 18720, 1536
    assert lib.bp_bench_wan_qk(0, rows, h, 12, 30, 52, iters, ctypes.byref(ms)) == 0
    gb = 4 * rows * h * 2 / 1e9
    print(f"wan qk-norm+rope {rows}x{h} ms {ms.value:.4f} GB/s {gb / ms.value * 1e3:.0f}")
    assert lib.bp_bench_ln(0, rows, h, iters, ctypes.byref(ms)) == 0
    print(f"ln (modulated form shares it) {rows}x{h} ms {ms.value:.4f} GB/s {rows * h * 6 / ms.value / 1e6:.0f}")
