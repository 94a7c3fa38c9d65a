"""One production-shape attention launch series of one variant (for ncu):
    python tools/attn_one.py IMPL [n0] [iters] [n1]
(IMPL 2 with n0 0 and n1 512 is the cross-attention launch)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from kernels import load_testlib  # noqa: E402

lib = load_testlib()
impl = int(sys.argv[1])
n0 = int(sys.argv[2]) if len(sys.argv) > 2 else 6240
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n1 = int(sys.argv[4]) if len(sys.argv) > 4 else 18720
lib.bp_set_kernel_impl(3, impl)
ms = ctypes.c_double()
assert lib.bp_bench_attn(0, 18720, 12, 128, n0, n1, iters, ctypes.byref(ms)) == 0, lib.bp_last_error()
print(f"impl {impl} n0 {n0} n1 {n1}: {4 * 18720 * (n0 + n1) * 1536 / ms.value / 1e9:.0f} TF/s")
