"""Drop-in for the reference's pybind11 module ``_blockpipe``
(P/python/bindings.cpp:76-161) over the B200 engine, so code written against
the reference (e.g. P/tests/python/test_smoke.py) runs unchanged:

    import _blockpipe as bp          # repo-root shim re-exports this module

Same function names, argument names, defaults and return shapes. The compute
entries (matmul, softmax_rows, layer_norm, RandomSource.next_normal,
run_pipeline, serial_oracle) run on the GPU through the C-ABI; there is no CPU
fallback. Integer-only host logic (splitmix64 draws, permutations, the static
schedule, closed-form analytics) runs on the host like in the reference.
"""
from __future__ import annotations

import ctypes as C
from typing import Any, Dict, List, Optional

import numpy as np

from . import api, errors
from ._lib import check, f64, lib, u64
from .operator import bubble_ratio, bubble_size, method_cost  # noqa: F401  (bindings.cpp:96-137)

__all__ = ["matmul", "softmax_rows", "layer_norm", "RandomSource", "bubble_size", "bubble_ratio",
           "method_cost", "run_pipeline", "serial_oracle", "coordinated_noise_ids"]

_MASK = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


def _f64_2d(a: Any, what: str) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise errors.DimensionError(f"{what} expects a 2-d array, got shape {arr.shape}")
    return arr


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(f64))


def matmul(a: Any, b: Any) -> np.ndarray:
    """matmul (tensor.cpp:84-109) on the GPU: ascending-k, unfused multiply-add,
    bit-identical to the reference's loop."""
    a, b = _f64_2d(a, "matmul"), _f64_2d(b, "matmul")
    if a.shape[1] != b.shape[0]:
        raise errors.DimensionError(f"matmul inner dimensions disagree: {list(a.shape)} vs {list(b.shape)}")
    out = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
    check(lib.bp_matmul(0, _p(a), _p(b), a.shape[0], a.shape[1], b.shape[1], _p(out)))
    return out


def softmax_rows(x: Any) -> np.ndarray:
    """softmax_rows (tensor.cpp:111-126) on the GPU."""
    x = _f64_2d(x, "softmax_rows")
    out = np.empty_like(x)
    check(lib.bp_softmax_rows(0, _p(x), x.shape[0], x.shape[1], _p(out)))
    return out


def layer_norm(x: Any, eps: float = 1e-5) -> np.ndarray:
    """layer_norm (tensor.cpp:128-146, no affine) on the GPU."""
    x = _f64_2d(x, "layer_norm")
    out = np.empty_like(x)
    check(lib.bp_layer_norm(0, _p(x), x.shape[0], x.shape[1], float(eps), _p(out)))
    return out


class RandomSource:
    """RandomSource (rng.hpp:28-45): splitmix64 stream. Integer draws are
    host-side; next_normal runs the bit-exact Box-Muller kernel (glibc
    log/cos port) on the GPU and advances the state by two draws."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + _PHI) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def next_normal(self) -> float:
        out = np.empty(1, dtype=np.float64)
        fin = u64()
        check(lib.bp_normals(0, self.state, 1, 1.0, _p(out), 0, C.byref(fin)))
        self.state = fin.value
        return float(out[0])

    def permutation(self, n: int) -> List[int]:
        p = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.next_u64() % (i + 1)
            p[i], p[j] = p[j], p[i]
        return p


def _run_to_dict(out: Dict[str, Any]) -> Dict[str, Any]:
    """run_to_dict (bindings.cpp:37-72) plus the extra keys of api.run_pipeline."""
    b = out["bubbles"]
    out["bubbles"] = {k: b[k] for k in ("busy_per_device", "idle_per_device", "warmup_idle", "steady_idle",
                                          "cooldown_idle", "ratio")}
    return out


def run_pipeline(config: Optional[Dict[str, Any]] = None) -> Dict[str, Any]:
    """bindings.cpp:139-141: run the pipeline (on the GPU) for a flat config dict."""
    return _run_to_dict(api.run_pipeline(dict(config or {})))


def serial_oracle(config: Optional[Dict[str, Any]] = None) -> Dict[str, Any]:
    """bindings.cpp:142-144: the same config on a single stage."""
    return _run_to_dict(api.serial_oracle(dict(config or {})))


def coordinated_noise_ids(num_b: int, num_c: int, appends: int, seed: int = 2) -> List[List[int]]:
    """bindings.cpp:146-160."""
    return api.coordinated_noise_ids(num_b, num_c, appends, seed)
