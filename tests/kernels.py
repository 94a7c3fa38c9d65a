"""Helpers for kernel-level GPU tests (bf16 packing, self-test wrappers)."""
import ctypes as C

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTLIB_PATH = os.environ.get("BP_TESTLIB_PATH") or os.path.join(ROOT, "paper_2505_21070_b200", "lib", "libbp_cuda_test.so")

i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
# kernel-level self-test hooks (include/bp_cuda_test.h), served by the test
# library built from the product's objects plus selftest.cu
TEST_SIGS = {
    "bp_last_error": (C.c_char_p, []),
    "bp_set_kernel_impl": (i32, [i32, i32]),
    "bp_selftest_gemm": (i32, [i32, i32, i32, i32, i32, C.c_void_p, i64, C.c_void_p, C.c_void_p, i64]),
    "bp_selftest_gemm_gated": (i32, [i32, i32, i32, i32, C.c_void_p, i64, C.c_void_p, C.c_void_p, i64, C.c_void_p,
                                     i32, i32]),
    "bp_selftest_attn": (i32, [i32, i64, i32, i32, C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_void_p,
                               C.c_void_p, i64, C.c_float, C.c_void_p]),
    "bp_selftest_attn_cross": (i32, [i32, i64, i32, i32, C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_float,
                                     C.c_void_p]),
    "bp_bench_gemm": (i32, [i32, i32, i32, i32, i32, i32, C.POINTER(f64)]),
    "bp_bench_attn": (i32, [i32, i64, i32, i32, i64, i64, i32, C.POINTER(f64)]),
    "bp_bench_ln": (i32, [i32, i64, i32, i32, C.POINTER(f64)]),
    "bp_bench_wan_qk": (i32, [i32, i64, i32, i32, i32, i32, i32, C.POINTER(f64)]),
}
_testlib = None


def load_testlib():
    global _testlib
    if _testlib is None:
        L = C.CDLL(TESTLIB_PATH)
        for name, (res, args) in TEST_SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _testlib = L
    return _testlib


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def gemm(lib, A_bits, W_bits, C_init, epi, lda=None):
    M, K = A_bits.shape[0], W_bits.shape[1]
    N = W_bits.shape[0]
    lda = lda or A_bits.shape[1]
    Cb = np.ascontiguousarray(C_init).copy()
    st = lib.bp_selftest_gemm(0, M, N, K, epi, A_bits.ctypes.data, lda, W_bits.ctypes.data, Cb.ctypes.data, N)
    assert st == 0, lib.bp_last_error()
    return Cb


def attn_cross(lib, q, k1, v1, heads, dh, scale):
    """The stage's cross-attention launcher (one key segment)."""
    rows = q.shape[0]
    out = np.zeros((rows, heads * dh), dtype=np.uint16)
    st = lib.bp_selftest_attn_cross(0, rows, heads, dh, q.ctypes.data, k1.ctypes.data, v1.ctypes.data, k1.shape[0],
                                    C.c_float(scale), out.ctypes.data)
    assert st == 0, lib.bp_last_error()
    return out


def attn(lib, q, k0, v0, k1, v1, heads, dh, scale):
    rows = q.shape[0]
    out = np.zeros((rows, heads * dh), dtype=np.uint16)
    n0 = 0 if k0 is None else k0.shape[0]
    z = np.zeros((1, heads * dh), dtype=np.uint16)
    st = lib.bp_selftest_attn(0, rows, heads, dh, q.ctypes.data, (k0 if n0 else z).ctypes.data,
                              (v0 if n0 else z).ctypes.data, n0, k1.ctypes.data, v1.ctypes.data, k1.shape[0],
                              C.c_float(scale), out.ctypes.data)
    assert st == 0, lib.bp_last_error()
    return out


def ref_attn(q, k, v, heads, dh, scale):
    out = np.zeros((q.shape[0], heads * dh))
    for hd in range(heads):
        sl = slice(hd * dh, (hd + 1) * dh)
        s = (q[:, sl].astype(np.float64) @ k[:, sl].T.astype(np.float64)) * scale
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, sl] = p @ v[:, sl].astype(np.float64)
    return out


# the library's default implementations (kernels_bf16.cu), restored after A/B tests
DEFAULT_ATTN_IMPL = 4
DEFAULT_GEMM_IMPL = 3
