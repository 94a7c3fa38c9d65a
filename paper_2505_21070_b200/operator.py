"""Operator surface: artifacts, run config, analytics and the
CLI, through the C-ABI of include/bp_operator.h (lib/libblockpipe_b200.so).

Mirrors P/include/blockpipe/{artifacts,run_config,analytics,cli}.hpp:
``run_and_write_artifacts`` (artifacts.cpp:130-143), ``config_echo``
(run_config.cpp:114-141), ``bubble_size``/``bubble_ratio`` (analytics.cpp:13-31),
``method_cost`` (analytics.cpp:67-117) and ``cli_main`` (cli.cpp:312-544).
Errors raise the reference exception types (ConfigError for exit code 2,
IoError for 3, BlockpipeError otherwise).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Any, Dict, List, Optional, Sequence, Tuple

from . import errors
from ._lib import LIB_PATH, lib as _cuda_lib  # noqa: F401  (loads libbp_cuda.so first)

OP_LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "libblockpipe_b200.so")
if not os.path.exists(OP_LIB_PATH):
    raise ImportError(f"{OP_LIB_PATH} is missing: build with __graft_entry__.build()")
_op = C.CDLL(OP_LIB_PATH)

i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
SINK = C.CFUNCTYPE(None, C.c_void_p, i32, C.POINTER(C.c_char), i64)


class CostParams(C.Structure):
    _fields_ = [("frames", i64), ("height", i64), ("width", i64), ("hidden", i64), ("channels", i64),
                ("layers", i64), ("devices", i64), ("num_b", i64), ("num_c", i64),
                ("model_mem", f64), ("kv_mem", f64), ("ring_refinement", i32), ("bytes_per_scalar", i32)]


class CostRow(C.Structure):
    _fields_ = [("comm_scalars", f64), ("comm_overlap", i32), ("model_mem", f64), ("kv_mem", f64),
                ("comm_bytes", f64)]


_op.bp_operator_last_error.restype = C.c_char_p
_op.bp_cli_main.argtypes = [i32, C.POINTER(C.c_char_p), SINK, C.c_void_p]
_op.bp_cli_main.restype = i32
_op.bp_write_artifacts.argtypes = [C.c_char_p, i32, C.c_char_p, i64]
_op.bp_write_artifacts.restype = i32
_op.bp_config_echo.argtypes = [C.c_char_p, C.c_char_p, i64]
_op.bp_config_echo.restype = i64
_op.bp_bubble.argtypes = [i32, i32, i64, i32, C.POINTER(i64), C.POINTER(f64)]
_op.bp_bubble.restype = i32
_op.bp_cost_defaults.argtypes = [C.POINTER(CostParams)]
_op.bp_cost_defaults.restype = None
_op.bp_method_cost.argtypes = [C.c_char_p, C.POINTER(CostParams), C.POINTER(CostRow)]
_op.bp_method_cost.restype = i32

METHODS = ("ring-attention", "ulysses", "video-infinity", "fifo", "dualparal")
DTYPE_BYTES = {"f64": 8, "f32": 4, "bf16": 2, "fp8": 1}
BOUNDARY_BYTES = {"f64": 8, "f32": 4, "bf16": 4}  # stage-boundary activation element size per precision


def _check(code: int) -> None:
    if code == 0:
        return
    msg = _op.bp_operator_last_error().decode()
    if code == 2:
        raise errors.ConfigError(msg)
    if code == 3:
        raise errors.IoError(msg)
    raise errors.BlockpipeError(msg)


def _config_text(config: Optional[Dict[str, Any]]) -> bytes:
    return json.dumps(dict(config or {})).encode()


def run_and_write_artifacts(config: Optional[Dict[str, Any]] = None, plan_only: bool = False) -> str:
    """Run the GPU pipeline for a flat JSON config and write latents.bin,
    schedule.csv, transfers.json and summary.json into its out_dir (default
    "out"). plan_only writes the three schedule-derived files without device
    work. Returns the summary path."""
    buf = C.create_string_buffer(4096)
    _check(_op.bp_write_artifacts(_config_text(config), 1 if plan_only else 0, buf, len(buf)))
    return buf.value.decode()


def plan_and_write_artifacts(config: Optional[Dict[str, Any]] = None) -> str:
    return run_and_write_artifacts(config, plan_only=True)


def config_echo(config: Optional[Dict[str, Any]] = None) -> str:
    """The effective config as every artifact echoes it (dump(2) text)."""
    n = _op.bp_config_echo(_config_text(config), None, 0)
    if n < 0:
        _check(2)
    buf = C.create_string_buffer(int(n) + 1)
    _op.bp_config_echo(_config_text(config), buf, len(buf))
    return buf.value.decode()


def bubble_size(devices: int, steps: int, block_num: int, order: str = "reverse") -> int:
    size, ratio = i64(), f64()
    _check(_op.bp_bubble(devices, steps, block_num, _order(order), C.byref(size), C.byref(ratio)))
    return size.value


def bubble_ratio(devices: int, steps: int, block_num: int, order: str = "reverse") -> float:
    size, ratio = i64(), f64()
    _check(_op.bp_bubble(devices, steps, block_num, _order(order), C.byref(size), C.byref(ratio)))
    return ratio.value


def _order(order: str) -> int:
    if order not in ("reverse", "sequential"):
        raise errors.ConfigError(f"order must be reverse or sequential, got {order}")
    return 0 if order == "reverse" else 1


_COST_INT = ("frames", "height", "width", "hidden", "channels", "layers", "devices", "num_b", "num_c")


def method_cost(method: str, **kwargs: Any) -> Dict[str, Any]:
    """bindings.cpp:109-137 semantics: CostParams defaults overridden by
    kwargs; unknown keys raise. Extension: dtype="bf16" (or bytes_per_scalar)
    adds comm_bytes."""
    cp = CostParams()
    _op.bp_cost_defaults(C.byref(cp))
    bytes_key = False
    for k, v in kwargs.items():
        if k in _COST_INT:
            setattr(cp, k, int(v))
        elif k in ("model_mem", "kv_mem"):
            setattr(cp, k, float(v))
        elif k == "ring_refinement":
            cp.ring_refinement = 1 if v else 0
        elif k == "bytes_per_scalar":
            cp.bytes_per_scalar, bytes_key = int(v), True
        elif k == "dtype":
            if v not in DTYPE_BYTES:
                raise errors.ConfigError(f"dtype must be one of {sorted(DTYPE_BYTES)}")
            cp.bytes_per_scalar, bytes_key = DTYPE_BYTES[v], True
        else:
            raise ValueError(f"unknown cost parameter: {k}")
    row = CostRow()
    _check(_op.bp_method_cost(method.encode(), C.byref(cp), C.byref(row)))
    out = {"method": method, "comm_scalars": row.comm_scalars, "comm_overlap": bool(row.comm_overlap),
           "model_mem": row.model_mem, "kv_mem": row.kv_mem}
    if bytes_key:
        out["comm_bytes"] = row.comm_bytes
    return out


def traffic_report(ledger: Sequence[Dict[str, Any]], precision: str = "f64",
                   measured_bytes: Optional[int] = None) -> Dict[str, Any]:
    """Predicted device->device bytes of one run (ledger scalars x element
    size of the boundary activation) beside the engine's measured
    boundary_bytes. The bf16 path keeps its residual stream in fp32 and ships
    it as fp32, so an N-stage split stays bitwise equal to one stage."""
    scalars = sum(int(e["scalars"]) for e in ledger
                  if e["channel"].startswith("dev") and "->dev" in e["channel"])
    elem = BOUNDARY_BYTES[precision]
    return {"ledger_scalars": scalars, "predicted_bytes": scalars * elem,
            "measured_bytes": measured_bytes,
            "match": None if measured_bytes is None else measured_bytes == scalars * elem}


def cli_main(args: Sequence[str]) -> Tuple[int, str, str]:
    """Run the `blockpipe` CLI in-process. Returns (exit code, stdout, stderr)."""
    chunks: Dict[int, List[bytes]] = {1: [], 2: []}

    def _sink(_user, stream, text, n):
        chunks[int(stream)].append(C.string_at(text, n))

    sink = SINK(_sink)
    argv = (C.c_char_p * len(args))(*[a.encode() for a in args])
    code = _op.bp_cli_main(len(args), argv, sink, None)
    return int(code), b"".join(chunks[1]).decode(), b"".join(chunks[2]).decode()
