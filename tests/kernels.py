"""Helpers for kernel-level GPU tests (bf16 packing, self-test wrappers)."""
import ctypes as C

import os

import numpy as np


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


# the library's default attention implementation (kernels_bf16.cu), restored after A/B tests
DEFAULT_ATTN_IMPL = int(os.environ.get("BP_ATTN_IMPL", "4"))
DEFAULT_GEMM_IMPL = int(os.environ.get("BP_GEMM_IMPL", "3"))
