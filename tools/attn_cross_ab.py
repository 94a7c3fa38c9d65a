"""The cross-attention launch (q 18720 x kv 512, 12 heads) by attention
implementation id (IMPLS, default 2 = k_attn_ps, the persistent cross kernel;
4 = the pair kernel): correctness vs fp64 numpy on ragged and exact-multiple
shapes, then interleaved timing.   IMPLS=2,4 python tools/attn_cross_ab.py [rounds] [iters]
Round 2: the one-item-per-CTA k_attn_pp it replaced ran at 821 TF/s on the
same box, k_attn_ps with direct stores 823-830, with the TMA-store epilogue
through the item's Q buffer 947-969."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from kernels import attn, from_bf16_bits, load_testlib, ref_attn, to_bf16_bits  # noqa: E402

lib = load_testlib()
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
IMPLS = [int(v) for v in os.environ.get("IMPLS", "2,4").split(",")]
for impl in IMPLS:
    lib.bp_set_kernel_impl(3, impl)
    worst = 0.0
    for rows, n0, n1, heads in ((1000, 0, 512, 3), (257, 0, 64, 2), (300, 0, 100, 1), (5000, 0, 512, 2),
                                (129, 65, 127, 1), (600, 128, 256, 2), (2048, 0, 1, 1)):
        rng = np.random.default_rng(rows + n1)
        dh, H = 128, heads * 128
        q = to_bf16_bits(rng.standard_normal((rows, H)))
        k1, v1 = to_bf16_bits(rng.standard_normal((n1, H))), to_bf16_bits(rng.standard_normal((n1, H)))
        k0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
        v0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
        kk = from_bf16_bits(np.concatenate([k0, k1]) if n0 else k1)
        vv = from_bf16_bits(np.concatenate([v0, v1]) if n0 else v1)
        want = ref_attn(from_bf16_bits(q), kk, vv, heads, dh, 1 / np.sqrt(dh))
        got = from_bf16_bits(attn(lib, q, k0, v0, k1, v1, heads, dh, 1 / np.sqrt(dh))).astype(np.float64)
        r = np.linalg.norm(got - want) / np.linalg.norm(want)
        worst = max(worst, r)
        if r > 1e-2:
            print(f"impl {impl} FAIL rows {rows} n0 {n0} n1 {n1} heads {heads}: {r:.3e}", flush=True)
    print(f"impl {impl}: worst rel-L2 {worst:.2e}", flush=True)
ms = ctypes.c_double()
res = {i: [] for i in IMPLS}
for _ in range(rounds):
    for impl in IMPLS:
        lib.bp_set_kernel_impl(3, impl)
        assert lib.bp_bench_attn(0, 18720, 12, 128, 0, 512, iters, ctypes.byref(ms)) == 0, lib.bp_last_error()
        res[impl].append(4 * 18720 * 512 * 1536 / ms.value / 1e9)
for impl in IMPLS:
    print(f"impl {impl}: cross-attention TF/s median {np.median(res[impl]):.0f} max {max(res[impl]):.0f}", flush=True)
lib.bp_set_kernel_impl(3, 4)
