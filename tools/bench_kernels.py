"""Kernel micro-benchmarks through the self-test hooks (include/bp_cuda_test.h),
used for ncu captures: python tools/bench_kernels.py attn|gemm [iters]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21070_b200._lib import lib  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "attn"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ms = ctypes.c_double()
if what == "attn":
    assert lib.bp_bench_attn(0, 18720, 12, 128, 6240, 18720, iters, ctypes.byref(ms)) == 0
    print("attn ms", ms.value, "TF", 4 * 18720 * 24960 * 1536 / ms.value / 1e9)
else:
    assert lib.bp_bench_gemm(0, 18720, 1536, 1536, 2, iters, ctypes.byref(ms)) == 0
    print("gemm ms", ms.value)
