"""A/B of attention kernel variants (bp_set_kernel_impl attention ids):
correctness against fp64 numpy on a few shapes, then isolated timing at the
production shape, variants interleaved over several rounds.
    python tools/attn_ab.py 4,5,6 [rounds] [iters]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from kernels import attn, from_bf16_bits, load_testlib, ref_attn, to_bf16_bits  # noqa: E402

lib = load_testlib()
impls = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4").split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
GEMM = 3

for impl in impls:
    lib.bp_set_kernel_impl(GEMM, impl)
    worst = 0.0
    for rows, n0, n1, heads in ((1000, 300, 1000, 2), (257, 65, 129, 1), (512, 0, 640, 2), (300, 128, 64, 1)):
        rng = np.random.default_rng(rows + n0 + n1)
        dh = 128
        H = heads * dh
        q = to_bf16_bits(rng.standard_normal((rows, H)))
        k1 = to_bf16_bits(rng.standard_normal((n1, H)) * 1.5)
        v1 = to_bf16_bits(rng.standard_normal((n1, H)))
        k0 = to_bf16_bits(rng.standard_normal((n0, H)) * 1.5) if n0 else None
        v0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
        kk = from_bf16_bits(np.concatenate([k0, k1]) if n0 else k1)
        vv = from_bf16_bits(np.concatenate([v0, v1]) if n0 else v1)
        want = ref_attn(from_bf16_bits(q), kk, vv, heads, dh, 1 / np.sqrt(dh))
        got = from_bf16_bits(attn(lib, q, k0, v0, k1, v1, heads, dh, 1 / np.sqrt(dh))).astype(np.float64)
        worst = max(worst, np.linalg.norm(got - want) / np.linalg.norm(want))
    print(f"impl {impl}: worst rel-L2 {worst:.2e} {'OK' if worst < 1e-2 else 'FAIL'}", flush=True)

ms = ctypes.c_double()
res = {i: [] for i in impls}
for r in range(rounds):
    for impl in impls:
        lib.bp_set_kernel_impl(GEMM, impl)
        for rows, n0, n1 in ((18720, 6240, 18720), (18720, 0, 18720)):
            assert lib.bp_bench_attn(0, rows, 12, 128, n0, n1, iters, ctypes.byref(ms)) == 0, lib.bp_last_error()
            res[impl].append((n0, 4 * rows * (n0 + n1) * 1536 / ms.value / 1e9))
for impl in impls:
    pre = [t for n0, t in res[impl] if n0]
    nop = [t for n0, t in res[impl] if not n0]
    print(f"impl {impl}: self+prefix TF {np.median(pre):.0f} (max {max(pre):.0f})  self TF {np.median(nop):.0f}"
          f" (max {max(nop):.0f})", flush=True)
