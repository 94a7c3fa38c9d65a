"""TEST INFRASTRUCTURE ONLY (oracle). ctypes driver of the unmodified
reference library compiled into oracle/_ref/libbp_ref.so (oracle/Makefile,
oracle/ref_shim.cpp). Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Any, Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libbp_ref.so")
RNG_LIB = os.path.join(HERE, "_ref", "libbp_oracle_rng.so")

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


class RefCfg(C.Structure):
    _fields_ = [("devices", i32), ("order", i32), ("cache_mode", i32), ("threaded", i32),
                ("num_b", i32), ("num_c", i32), ("steps", i32), ("block_num", i32),
                ("retain_clean_context", i32), ("layers", i32), ("hidden", i32), ("heads", i32),
                ("channels", i32), ("height", i32), ("width", i32), ("context_len", i32),
                ("strategy", i32), ("seed_model", u64), ("seed_noise", u64), ("seed_context", u64),
                ("fault_inject_ulp", i32), ("record_trace", i32), ("check_cache", i32)]


def available() -> bool:
    return os.path.exists(REF_LIB)


_lib = None
_rng = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(REF_LIB)
        L.bpref_last_error.restype = C.c_char_p
        L.bpref_derive_seed.restype = u64
        L.bpref_derive_seed.argtypes = [u64, P(u64), C.c_int]
        L.bpref_u64.argtypes = [u64, i64, P(u64)]
        L.bpref_normals.argtypes = [u64, i64, f64, P(f64)]
        L.bpref_permutation.argtypes = [u64, C.c_int, P(C.c_int)]
        L.bpref_pool.argtypes = [C.c_int, C.c_int, i64, i64, i64, u64, P(f64)]
        L.bpref_build_layer.argtypes = [P(RefCfg), u64, C.c_int, P(f64)]
        L.bpref_build_context.argtypes = [P(RefCfg), u64, P(f64)]
        L.bpref_chunk_create.restype = C.c_void_p
        L.bpref_chunk_create.argtypes = [P(RefCfg), u64, C.c_int, C.c_int, u64]
        L.bpref_chunk_destroy.argtypes = [C.c_void_p]
        L.bpref_chunk_forward.argtypes = [C.c_void_p, P(f64), i64, i64, P(C.c_int), P(i64), C.c_int,
                                          P(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int, P(f64), P(i64)]
        L.bpref_chunk_cache.argtypes = [C.c_void_p, C.c_int, C.c_int, P(f64), P(i64)]
        L.bpref_run.restype = C.c_void_p
        L.bpref_run.argtypes = [P(RefCfg), C.c_int]
        for n in ("bpref_run_free",):
            getattr(L, n).argtypes = [C.c_void_p]
        for n in ("bpref_run_rounds", "bpref_run_nblocks", "bpref_run_nevents", "bpref_run_nledger",
                  "bpref_run_nsnap", "bpref_run_ntrace"):
            getattr(L, n).restype = i64
            getattr(L, n).argtypes = [C.c_void_p]
        L.bpref_run_block_info.argtypes = [C.c_void_p, i64, P(i64), P(i64), P(i64)]
        L.bpref_run_block_data.argtypes = [C.c_void_p, i64, P(f64), P(C.c_int), P(i64)]
        L.bpref_run_events.argtypes = [C.c_void_p, P(i64)]
        L.bpref_run_ledger.argtypes = [C.c_void_p, i64, C.c_char_p, P(i64), P(i64), P(i64)]
        L.bpref_run_snap.argtypes = [C.c_void_p, i64, P(i64), P(i64), P(C.c_int)]
        L.bpref_run_trace_info.argtypes = [C.c_void_p, i64, P(i64), P(i64), P(i64), P(i64)]
        L.bpref_run_trace_data.argtypes = [C.c_void_p, i64, P(f64)]
        L.bpref_run_bubbles.argtypes = [C.c_void_p, P(i64), P(f64)]
        L.bpref_bubble.argtypes = [C.c_int, C.c_int, i64, C.c_int, P(i64), P(f64)]
        L.bpref_method_cost.argtypes = [C.c_char_p, P(i64), P(f64), C.c_int, P(f64)]
        L.bpref_noise_walk.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, u64, C.c_int, P(C.c_int),
                                       P(C.c_int)]
        L.bpref_noise_walk_frames.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, P(i64), u64, C.c_int,
                                              P(C.c_int), P(C.c_int), P(f64), P(i64)]
        _lib = L
    return _lib


def rng_lib():
    global _rng
    if _rng is None:
        R = C.CDLL(RNG_LIB)
        R.bpo_normals.restype = u64
        R.bpo_normals.argtypes = [u64, i64, f64, P(f64)]
        R.bpo_derive_seed.restype = u64
        R.bpo_derive_seed.argtypes = [u64, P(u64), C.c_int]
        _rng = R
    return _rng


ORDER = {"reverse": 0, "sequential": 1}
CACHE = {"off": 0, "on": 1, "recompute": 2}
STRAT = {"coordinated": 0, "complete-shuffle": 1, "subset": 2, "fresh": 3, "repeat": 4}
ERR = {1: "ConfigError", 2: "DimensionError", 3: "CacheError", 4: "SchedulerError", 5: "QueueError",
       6: "SchedulingError", 7: "PartitionError", 9: "Error"}


class RefError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def _raise():
    L = lib()
    raise RefError(ERR.get(L.bpref_last_error_kind(), "Error"), L.bpref_last_error().decode())


def ref_cfg(cfg) -> RefCfg:
    """cfg: paper_2505_21070_b200.PipelineConfig (or anything with the same fields)."""
    return RefCfg(cfg.devices, ORDER[cfg.order], CACHE[cfg.cache], int(cfg.threaded), cfg.num_b, cfg.num_c,
                  cfg.steps, cfg.blocks, int(cfg.retain_clean_context), cfg.layers, cfg.hidden, cfg.heads,
                  cfg.channels, cfg.height, cfg.width, cfg.context_len, STRAT[cfg.strategy], cfg.seed_model,
                  cfg.seed_noise, cfg.seed_context, int(cfg.fault_inject), int(cfg.record_trace),
                  int(cfg.check_cache))


def run(cfg, serial: bool = False) -> Dict[str, Any]:
    """The reference's run_pipeline / serial_oracle, converted to numpy."""
    L = lib()
    rc = ref_cfg(cfg)
    h = L.bpref_run(C.byref(rc), int(serial))
    if not h:
        _raise()
    try:
        out: Dict[str, Any] = {"rounds": L.bpref_run_rounds(h)}
        blocks = []
        for i in range(L.bpref_run_nblocks(h)):
            bid, fr, nid = i64(), i64(), i64()
            L.bpref_run_block_info(h, i, C.byref(bid), C.byref(fr), C.byref(nid))
            frames = np.empty((fr.value, cfg.height, cfg.width, cfg.channels))
            ids = np.zeros(max(nid.value, 1), dtype=np.intc)
            fids = np.zeros(fr.value, dtype=np.int64)
            L.bpref_run_block_data(h, i, frames.ctypes.data_as(P(f64)), ids.ctypes.data_as(P(C.c_int)),
                                   fids.ctypes.data_as(P(i64)))
            blocks.append({"block_id": bid.value, "frames": frames, "noise_ids": ids[:nid.value].tolist(),
                           "frame_ids": fids.tolist()})
        out["blocks"] = blocks
        ne = L.bpref_run_nevents(h)
        ev = np.zeros((max(ne, 1), 6), dtype=np.int64)
        L.bpref_run_events(h, ev.ctypes.data_as(P(i64)))
        out["events"] = ev[:ne]
        ledger = []
        for i in range(L.bpref_run_nledger(h)):
            ch = C.create_string_buffer(32)
            r, p, s = i64(), i64(), i64()
            L.bpref_run_ledger(h, i, ch, C.byref(r), C.byref(p), C.byref(s))
            ledger.append({"channel": ch.value.decode(), "round": r.value, "passes": p.value, "scalars": s.value})
        out["ledger"] = ledger
        snaps = []
        for i in range(L.bpref_run_nsnap(h)):
            r = i64()
            ids = np.zeros(64, dtype=np.int64)
            lv = np.zeros(64, dtype=np.intc)
            n = L.bpref_run_snap(h, i, C.byref(r), ids.ctypes.data_as(P(i64)), lv.ctypes.data_as(P(C.c_int)))
            snaps.append({"round": r.value, "block_ids": ids[:n].tolist(), "levels": lv[:n].tolist()})
        out["queue_snapshots"] = snaps
        trace = []
        for i in range(L.bpref_run_ntrace(h)):
            r, b, rows, cols = i64(), i64(), i64(), i64()
            L.bpref_run_trace_info(h, i, C.byref(r), C.byref(b), C.byref(rows), C.byref(cols))
            eps = np.empty((rows.value, cols.value))
            L.bpref_run_trace_data(h, i, eps.ctypes.data_as(P(f64)))
            trace.append({"round": r.value, "block_id": b.value, "eps": eps})
        out["trace"] = trace
        st = np.zeros(7, dtype=np.int64)
        ratio = f64()
        L.bpref_run_bubbles(h, st.ctypes.data_as(P(i64)), C.byref(ratio))
        out["bubbles"] = dict(zip(("first_slot", "last_slot", "busy_per_device", "idle_per_device",
                                   "warmup_idle", "steady_idle", "cooldown_idle"), st.tolist()),
                              ratio=ratio.value)
        return out
    finally:
        L.bpref_run_free(h)


def pool(num_b: int, num_c: int, shape, seed: int) -> np.ndarray:
    L = lib()
    m = num_b + num_c // 2
    out = np.empty((m, *shape))
    if L.bpref_pool(num_b, num_c, shape[0], shape[1], shape[2], seed, out.ctypes.data_as(P(f64))):
        _raise()
    return out


def normals(seed: int, n: int, sigma: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    lib().bpref_normals(seed, n, sigma, out.ctypes.data_as(P(f64)))
    return out


class RefChunk:
    """A reference ModelChunk + the DeviceWorker-style single-entry cache."""

    def __init__(self, cfg, seed: int, begin: int, end: int, context_seed: int):
        L = lib()
        rc = ref_cfg(cfg)
        self.cfg = cfg
        self.h = L.bpref_chunk_create(C.byref(rc), seed, begin, end, context_seed)
        if not self.h:
            _raise()
        self.last = end == cfg.layers

    def forward(self, payload, levels, frame_ids, capture=(), mode="off", use_prev=0, record_inputs=False):
        L = lib()
        payload = np.ascontiguousarray(payload, dtype=np.float64)
        lv = np.ascontiguousarray(levels, dtype=np.intc)
        fi = np.ascontiguousarray(frame_ids, dtype=np.int64)
        cf = np.ascontiguousarray(capture, dtype=np.intc)
        cols = self.cfg.channels if self.last else self.cfg.hidden
        out = np.empty((payload.shape[0], cols))
        oc = i64()
        if L.bpref_chunk_forward(self.h, payload.ctypes.data_as(P(f64)), payload.shape[0], payload.shape[1],
                                 lv.ctypes.data_as(P(C.c_int)), fi.ctypes.data_as(P(i64)), len(lv),
                                 cf.ctypes.data_as(P(C.c_int)), len(cf), CACHE[mode], use_prev,
                                 int(record_inputs), out.ctypes.data_as(P(f64)), C.byref(oc)):
            _raise()
        return out

    def cache(self, layer: int, which: int) -> np.ndarray:
        L = lib()
        rows = i64()
        if L.bpref_chunk_cache(self.h, layer, which, None, C.byref(rows)):
            _raise()
        out = np.empty((rows.value, self.cfg.hidden))
        L.bpref_chunk_cache(self.h, layer, which, out.ctypes.data_as(P(f64)), C.byref(rows))
        return out

    def __del__(self):
        try:
            lib().bpref_chunk_destroy(self.h)
        except Exception:
            pass


def fnv1a64(arrays) -> str:
    """FNV-1a-64 over the raw bytes of fp64 arrays, in order."""
    h = 0xCBF29CE484222325
    for a in arrays:
        for byte in np.ascontiguousarray(a, dtype=np.float64).tobytes():
            h ^= byte
            h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# ---- analytics.hpp / noise-demo (operator surface goldens) -----------------------------
def _ck(rc: int) -> None:
    if rc != 0:
        _raise()


def bubble(n: int, t: int, blocks: int, order: str = "reverse"):
    """(bubble_size, bubble_ratio) (analytics.cpp:13-31)."""
    size, ratio = i64(), f64()
    _ck(lib().bpref_bubble(n, t, blocks, 1 if order == "sequential" else 0, C.byref(size), C.byref(ratio)))
    return size.value, ratio.value


COST_KEYS = ("frames", "height", "width", "hidden", "channels", "layers", "devices", "num_b", "num_c")
COST_DEFAULTS = dict(frames=16, height=4, width=4, hidden=8, channels=4, layers=8, devices=2, num_b=8,
                     num_c=8, model_mem=1.0, kv_mem=1.0, ring_refinement=False)


def method_cost(method: str, **kw) -> Dict[str, Any]:
    """method_cost (analytics.cpp:67-117) with CostParams defaults (analytics.hpp:31-47)."""
    p = dict(COST_DEFAULTS, **kw)
    ints = (i64 * 9)(*[int(p[k]) for k in COST_KEYS])
    mem = (f64 * 2)(float(p["model_mem"]), float(p["kv_mem"]))
    out = (f64 * 4)()
    _ck(lib().bpref_method_cost(method.encode(), ints, mem, 1 if p["ring_refinement"] else 0, out))
    return {"method": method, "comm_scalars": out[0], "comm_overlap": bool(out[1]), "model_mem": out[2],
            "kv_mem": out[3]}


def noise_walk(strategy: str, appends: int, num_b: int, num_c: int, seed: int):
    """Noise ids per block as cli.cpp:499-529 (noise-demo) draws them."""
    cap = num_b + num_c // 2
    ids = (C.c_int * ((appends + 1) * cap))()
    counts = (C.c_int * (appends + 1))()
    _ck(lib().bpref_noise_walk(strategy.encode(), appends, num_b, num_c, seed, cap, ids, counts))
    return [[ids[r * cap + k] for k in range(counts[r])] for r in range(appends + 1)]


def noise_walk_frames(strategy: str, appends: int, num_b: int, num_c: int, shape, seed: int):
    """The reference's draw_first_block + `appends` draw_next_block calls:
    [(noise_ids, frames [f, H, W, C])] per draw."""
    cap = num_b + num_c // 2
    per = int(np.prod(shape))
    ids = (C.c_int * ((appends + 1) * cap))()
    counts = (C.c_int * (appends + 1))()
    frames = np.empty((appends + 1) * cap * per)
    sh = (i64 * 3)(*shape)
    nv = i64()
    _ck(lib().bpref_noise_walk_frames(strategy.encode(), appends, num_b, num_c, sh, seed, cap, ids, counts,
                                      frames.ctypes.data_as(P(f64)), C.byref(nv)))
    out, at = [], 0
    for r in range(appends + 1):
        f = cap if r == 0 else num_b
        out.append(([ids[r * cap + k] for k in range(counts[r])], frames[at:at + f * per].reshape((f,) + tuple(shape))))
        at += f * per
    return out


def permutation(seed: int, n: int) -> np.ndarray:
    """RandomSource(seed).permutation(n) (rng.cpp:41-49)."""
    out = (C.c_int * max(n, 1))()
    lib().bpref_permutation(seed, n, out)  # void
    return np.array(out[:n], dtype=np.int64)
