"""ctypes binding of the C-ABI in include/bp_cuda.h (lib/libbp_cuda.so).

There is no Python or CPU fallback: if the shared library is missing this
module raises ImportError, and every compute entry point raises CudaError
when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# BP_LIB_PATH points at an alternative build (A/B kernel experiments only)
LIB_PATH = os.environ.get("BP_LIB_PATH") or os.path.join(_HERE, "lib", "libbp_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). The blockpipe-b200 path has no CPU fallback.")

def _prefer_bundled_nccl() -> None:
    """NCCL is dlopen'ed lazily by the library; point it at torch's bundled
    libnccl (if installed) so one process never mixes two NCCL builds."""
    if "BP_NCCL_LIB" in os.environ:
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        if spec and spec.submodule_search_locations:
            cand = os.path.join(list(spec.submodule_search_locations)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["BP_NCCL_LIB"] = cand
    except Exception:
        pass


_prefer_bundled_nccl()
lib = C.CDLL(LIB_PATH)

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


class ModelDesc(C.Structure):
    _fields_ = [("layers", i32), ("hidden", i32), ("heads", i32), ("channels", i32),
                ("height", i32), ("width", i32), ("context_len", i32), ("ffn", i32), ("block", i32)]


class PipelineDesc(C.Structure):
    _fields_ = [("devices", i32), ("order", i32), ("cache_mode", i32),
                ("num_b", i32), ("num_c", i32), ("steps", i32), ("block_num", i32),
                ("retain_clean_context", i32), ("strategy", i32), ("model", ModelDesc),
                ("seed_model", u64), ("seed_noise", u64), ("seed_context", u64),
                ("fault_inject_ulp", i32), ("record_trace", i32), ("check_cache", i32),
                ("precision", i32), ("transport", i32), ("uneven_split", i32),
                ("layer_split", i32 * 64)]


class ChunkIn(C.Structure):
    _fields_ = [("payload", P(f64)), ("rows", i64), ("cols", i64),
                ("frame_levels", P(i32)), ("frame_ids", P(i64)), ("nframes", i32),
                ("capture_frames", P(i32)), ("ncapture", i32), ("record_inputs", i32),
                ("mode", i32), ("use_prev", i32), ("prefix_k", P(f64)), ("prefix_v", P(f64)),
                ("prefix_rows", i64)]


class ChunkOut(C.Structure):
    _fields_ = [("payload", P(f64)), ("payload_capacity", i64), ("rows", i64), ("cols", i64),
                ("captured", i32), ("recorded", i32), ("captured_tokens", i64)]


class PipelineStats(C.Structure):
    _fields_ = [("gpu_ms", f64), ("passes", i64), ("kernel_launches", i64), ("peak_bytes", i64),
                ("boundary_bytes", i64), ("attn_ms", f64), ("gemm_ms", f64), ("cross_ms", f64),
                ("attn_launches", i64), ("gemm_launches", i64), ("cross_launches", i64),
                ("ln_ms", f64), ("ln_launches", i64), ("h2d_bytes", i64), ("d2h_bytes", i64),
                ("boundary_copies", i64), ("registered_buffers", i64), ("fused_sends", i64)]


EMIT_FN = C.CFUNCTYPE(None, C.c_void_p, i64, i64, P(f64), P(i32), i32, P(i64))

_SIGS = {
    "bp_last_error": (C.c_char_p, []),
    "bp_version": (C.c_char_p, []),
    "bp_derive_seed": (u64, [u64, P(u64), i32]),
    "bp_normals": (i32, [i32, u64, i64, f64, P(f64), i32, P(u64)]),
    "bp_noise_pool": (i32, [i32, i32, i32, P(i64), u64, P(f64), i32]),
    "bp_stage_create": (i32, [i32, P(ModelDesc), u64, u64, i32, i32, i32, P(C.c_void_p)]),
    "bp_stage_destroy": (i32, [C.c_void_p]),
    "bp_forward_chunk": (i32, [C.c_void_p, P(ChunkIn), P(ChunkOut)]),
    "bp_stage_cache_rows": (i32, [C.c_void_p, i32, i32, P(f64), P(i64)]),
    "bp_stage_cache_bump_ulp": (i32, [C.c_void_p, i32, i32, i64]),
    "bp_stage_recorded_rows": (i32, [C.c_void_p, i32, P(f64), P(i64)]),
    "bp_stage_set_context": (i32, [C.c_void_p, P(f64), i64, i64]),
    "bp_stage_cache_audit": (i32, [C.c_void_p, C.c_char_p, i32]),
    "bp_scheduler_step": (i32, [i32, P(f64), P(f64), i64, i32, i32, P(f64)]),
    "bp_matmul": (i32, [i32, P(f64), P(f64), i64, i64, i64, P(f64)]),
    "bp_elementwise": (i32, [i32, i32, P(f64), P(f64), i64, f64, P(f64)]),
    "bp_gather_block": (i32, [i32, P(f64), i32, i64, P(i32), i32, P(f64), i32]),
    "bp_noise_draw": (i32, [i32, i32, i32, i32, i32, P(i64), P(f64), i32, P(i32), i32, P(u64), P(f64), P(i32),
                            P(i32), P(i32), i32]),
    "bp_softmax_rows": (i32, [i32, P(f64), i64, i64, P(f64)]),
    "bp_layer_norm": (i32, [i32, P(f64), i64, i64, f64, P(f64)]),
    "bp_schedule_create": (i32, [P(PipelineDesc), P(C.c_void_p)]),
    "bp_schedule_destroy": (None, [C.c_void_p]),
    "bp_schedule_rounds": (i64, [C.c_void_p]),
    "bp_schedule_npasses": (i64, [C.c_void_p]),
    "bp_schedule_nevents": (i64, [C.c_void_p]),
    "bp_schedule_events": (None, [C.c_void_p, P(i64)]),
    "bp_schedule_nledger": (i64, [C.c_void_p]),
    "bp_schedule_ledger": (None, [C.c_void_p, i64, C.c_char_p, P(i64), P(i64), P(i64)]),
    "bp_schedule_nsnapshots": (i64, [C.c_void_p]),
    "bp_schedule_snapshot": (i32, [C.c_void_p, i64, P(i64), P(i64), P(i32)]),
    "bp_schedule_nblocks": (i64, [C.c_void_p]),
    "bp_schedule_block": (i32, [C.c_void_p, i64, P(i64), P(i64), P(i32), P(i64)]),
    "bp_schedule_partition": (None, [C.c_void_p, P(i32), P(i32)]),
    "bp_schedule_rank_program": (i64, [C.c_void_p, i32, P(i64), i64]),
    "bp_schedule_pass": (i32, [C.c_void_p, i64, P(i64), P(i32), P(i64), P(i32)]),
    "bp_schedule_block_meta": (None, [C.c_void_p, i64, P(i64)]),
    "bp_nccl_unique_id": (i32, [P(C.c_uint8)]),
    "bp_pipeline_create": (i32, [P(PipelineDesc), i32, i32, i32, P(C.c_uint8), P(C.c_void_p)]),
    "bp_pipeline_destroy": (i32, [C.c_void_p]),
    "bp_ipc_handle": (i32, [C.c_void_p, P(C.c_uint8)]),
    "bp_bootstrap_nccl_ids": (i32, [C.c_char_p, i32, i32, i32, P(C.c_uint8)]),
    "bp_bootstrap_ipc": (i32, [C.c_void_p, C.c_char_p, i32, i32, i32]),
    "bp_ipc_connect": (i32, [C.c_void_p, P(C.c_uint8)]),
    "bp_ipc_counters": (i32, [C.c_void_p, P(C.c_uint32)]),
    "bp_pipeline_run": (i32, [C.c_void_p, EMIT_FN, C.c_void_p]),
    "bp_pipeline_get_stats": (i32, [C.c_void_p, P(PipelineStats)]),
    "bp_pipeline_set_profiling": (i32, [C.c_void_p, i32]),
    "bp_pipeline_ntrace": (i64, [C.c_void_p]),
    "bp_pipeline_trace": (i32, [C.c_void_p, i64, P(i64), P(i64), P(i64), P(i64), P(f64)]),
    "bp_pipeline_block": (i32, [C.c_void_p, i64, P(P(f64)), P(i64)]),
    "bp_pipeline_set_pool": (i32, [C.c_void_p, P(f64), i64]),
    "bp_host_alloc": (i32, [i64, P(C.c_void_p)]),
    "bp_host_free": (i32, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def check(status: int) -> None:
    """Raises the blockpipe exception matching a bp_status (errors.hpp:11-41)."""
    if status != 0:
        msg = lib.bp_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)
