"""Python mirror of the reference's operator surface for the hot path
(engine.hpp, model.hpp, noise.hpp, rng.hpp and the pybind module
python/bindings.cpp:76-161), every call going through the C-ABI."""
from __future__ import annotations

import ctypes as C
from typing import Any, Callable, Dict, List, Optional, Sequence, Union

import numpy as np

from . import errors
from ._lib import (EMIT_FN, ChunkIn, ChunkOut, PipelineStats, check, i32, i64, lib, u64, f64)
from .config import CACHE, PRECISIONS, PipelineConfig

ConfigLike = Union[PipelineConfig, Dict[str, Any], None]

PHASES = ("warmup", "steady", "cooldown")


def _cfg(config: ConfigLike) -> PipelineConfig:
    if isinstance(config, PipelineConfig):
        return config
    return PipelineConfig.from_dict(config)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---- rng.hpp -----------------------------------------------------------------------
def derive_seed(base: int, tags: Sequence[int]) -> int:
    """derive_seed (rng.cpp:51-60), host-side."""
    arr = (u64 * max(1, len(tags)))(*tags)
    return int(lib.bp_derive_seed(base, arr, len(tags)))


def normals(state: int, n: int, sigma: float = 1.0, device: int = 0) -> np.ndarray:
    """RandomSource(state).normal_tensor({n}, sigma) drawn on the GPU (bit-exact)."""
    out = np.empty(n, dtype=np.float64)
    fin = u64()
    check(lib.bp_normals(device, state, n, sigma, _ptr(out, f64), 0, C.byref(fin)))
    return out


# ---- noise.hpp ------------------------------------------------------------------------
def build_pool(num_b: int, num_c: int, frame_shape: Sequence[int], noise_seed: int,
               device: int = 0) -> np.ndarray:
    """build_pool (noise.cpp:26-48) on the GPU: [M, H, W, C] fp64."""
    h, w, c = (int(v) for v in frame_shape)
    m = num_b + num_c // 2
    out = np.empty((m, h, w, c), dtype=np.float64)
    shape = (i64 * 3)(h, w, c)
    check(lib.bp_noise_pool(device, num_b, num_c, shape, noise_seed, _ptr(out, f64), 0))
    return out


def gather_block(pool: np.ndarray, ids: Sequence[int], device: int = 0) -> np.ndarray:
    """stack_entries (noise.cpp:12-22) on the GPU: pool [M, H, W, C] -> [len(ids), H, W, C]."""
    pool = np.ascontiguousarray(pool, dtype=np.float64)
    idx = np.ascontiguousarray(ids, dtype=np.int32)
    per = int(np.prod(pool.shape[1:]))
    out = np.empty((len(idx),) + pool.shape[1:], dtype=np.float64)
    check(lib.bp_gather_block(device, _ptr(pool, f64), pool.shape[0], per, _ptr(idx, i32), len(idx),
                              _ptr(out, f64), 0))
    return out


def _noise_draw(strategy: str, first: bool, pool: np.ndarray, num_b: int, num_c: int,
                tail_window_ids: Sequence[int], rng_state: int, device: int) -> Dict[str, Any]:
    from .config import STRATEGIES
    if strategy not in STRATEGIES:
        raise errors.ConfigError(f"unknown noise strategy: {strategy}")
    pool = np.ascontiguousarray(pool, dtype=np.float64)
    shape = (i64 * 3)(*pool.shape[1:])
    cap = pool.shape[0] if first else num_b
    frames = np.empty((cap,) + pool.shape[1:], dtype=np.float64)
    ids = np.zeros(max(cap, 1), dtype=np.int32)
    win = np.ascontiguousarray(tail_window_ids, dtype=np.int32)
    state = u64(rng_state)
    nf, ni = i32(), i32()
    check(lib.bp_noise_draw(device, STRATEGIES[strategy], int(first), num_b, num_c, shape, _ptr(pool, f64),
                            pool.shape[0], _ptr(win, i32), len(win), C.byref(state), _ptr(frames, f64),
                            _ptr(ids, i32), C.byref(nf), C.byref(ni), 0))
    return {"frames": frames[:nf.value], "noise_ids": ids[:ni.value].tolist(), "rng_state": int(state.value)}


def draw_first_block(strategy: str, pool: np.ndarray, num_b: int, num_c: int, rng_state: int,
                     device: int = 0) -> Dict[str, Any]:
    """draw_first_block (noise.cpp:135-152): NoiseDraw {frames, noise_ids} and
    the append RandomSource's state after the draw."""
    return _noise_draw(strategy, True, pool, num_b, num_c, (), rng_state, device)


def draw_next_block(strategy: str, pool: np.ndarray, num_b: int, num_c: int, tail_window_ids: Sequence[int],
                    rng_state: int, device: int = 0) -> Dict[str, Any]:
    """draw_next_block (noise.cpp:154-178); coordinated excludes tail_window_ids."""
    return _noise_draw(strategy, False, pool, num_b, num_c, tail_window_ids, rng_state, device)


def scheduler_step(x: np.ndarray, eps: np.ndarray, level: int, steps: int, device: int = 0) -> np.ndarray:
    """scheduler_step (model.cpp:338-345) on the GPU."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    eps = np.ascontiguousarray(eps, dtype=np.float64)
    if x.shape != eps.shape:
        raise errors.SchedulerError("x and eps shapes disagree")
    out = np.empty_like(x)
    check(lib.bp_scheduler_step(device, _ptr(x, f64), _ptr(eps, f64), x.size, level, steps, _ptr(out, f64)))
    return out


# ---- model.hpp -------------------------------------------------------------------------
class Stage:
    """A ModelChunk over layers [begin, end) resident on one GPU, with the
    per-device KV feature cache (model.hpp:50-101)."""

    def __init__(self, config: ConfigLike, seed: int, begin: int, end: int, context_seed: int,
                 precision: str = "f64", device: int = 0):
        cfg = _cfg(config)
        self.cfg = cfg
        self.begin, self.end = begin, end
        self._h = C.c_void_p()
        md = cfg.model_desc()
        check(lib.bp_stage_create(device, C.byref(md), seed, context_seed, begin, end,
                                  PRECISIONS[precision], C.byref(self._h)))

    def close(self):
        if self._h:
            lib.bp_stage_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward_chunk(self, payload: np.ndarray, frame_levels: Sequence[int], frame_ids: Sequence[int],
                      capture_frames: Sequence[int] = (), mode: str = "off", use_prev: int = 0,
                      record_inputs: bool = False) -> Dict[str, Any]:
        """forward_chunk (model.cpp:227-336). use_prev: 0 none, 1 the resident
        captured K/V of the previous call, 2 its recorded layer inputs."""
        payload = np.ascontiguousarray(payload, dtype=np.float64)
        if len(frame_levels) != len(frame_ids):
            raise errors.DimensionError("frame_ids and frame_levels disagree")
        lv = np.ascontiguousarray(frame_levels, dtype=np.int32)
        fi = np.ascontiguousarray(frame_ids, dtype=np.int64)
        cf = np.ascontiguousarray(capture_frames, dtype=np.int32)
        tpf = self.cfg.height * self.cfg.width
        rows = payload.shape[0]
        if rows != len(lv) * tpf:
            raise errors.DimensionError("payload rows do not match frames * tokens_per_frame")
        cin = ChunkIn(_ptr(payload, f64), rows, payload.shape[1] if payload.ndim > 1 else 1,
                      _ptr(lv, i32), _ptr(fi, i64), len(lv), _ptr(cf, i32), len(cf),
                      int(record_inputs), CACHE[mode], int(use_prev), None, None, 0)
        out_cols = self.cfg.channels if self.end == self.cfg.layers else self.cfg.hidden
        out = np.empty((rows, out_cols), dtype=np.float64)
        cout = ChunkOut(_ptr(out, f64), out.size, 0, 0, 0, 0, 0)
        check(lib.bp_forward_chunk(self._h, C.byref(cin), C.byref(cout)))
        return {"payload": out, "captured": bool(cout.captured), "recorded": bool(cout.recorded),
                "captured_tokens": int(cout.captured_tokens)}

    def cache_rows(self, layer: int, which: int) -> np.ndarray:
        rows = i64()
        check(lib.bp_stage_cache_rows(self._h, layer, which, None, C.byref(rows)))
        out = np.empty((rows.value, self.cfg.hidden), dtype=np.float64)
        check(lib.bp_stage_cache_rows(self._h, layer, which, _ptr(out, f64), C.byref(rows)))
        return out

    def bump_ulp(self, layer: int = 0, which: int = 1, index: int = 0) -> None:
        check(lib.bp_stage_cache_bump_ulp(self._h, layer, which, index))

    def audit(self) -> str:
        buf = C.create_string_buffer(512)
        check(lib.bp_stage_cache_audit(self._h, buf, 512))
        return buf.value.decode()


# ---- engine.hpp: schedule (host-only) ----------------------------------------------------
class Schedule:
    """The static schedule of run_pipeline: EventLog, TransferLedger,
    QueueSnapshots, emitted block ids / noise ids (host-only, no GPU)."""

    def __init__(self, config: ConfigLike):
        self.cfg = _cfg(config)
        self._h = C.c_void_p()
        desc = self.cfg.to_desc()
        check(lib.bp_schedule_create(C.byref(desc), C.byref(self._h)))
        h = self._h
        self.rounds = int(lib.bp_schedule_rounds(h))
        self.npasses = int(lib.bp_schedule_npasses(h))
        ne = int(lib.bp_schedule_nevents(h))
        ev = np.zeros((max(ne, 1), 6), dtype=np.int64)
        lib.bp_schedule_events(h, _ptr(ev, i64))
        self.events = ev[:ne]
        self.ledger = []
        for i in range(int(lib.bp_schedule_nledger(h))):
            ch = C.create_string_buffer(32)
            r, p, s = i64(), i64(), i64()
            lib.bp_schedule_ledger(h, i, ch, C.byref(r), C.byref(p), C.byref(s))
            self.ledger.append({"channel": ch.value.decode(), "round": r.value, "passes": p.value,
                                "scalars": s.value})
        self.snapshots = []
        for i in range(int(lib.bp_schedule_nsnapshots(h))):
            r = i64()
            n = lib.bp_schedule_snapshot(h, i, C.byref(r), None, None)
            ids = np.zeros(max(n, 1), dtype=np.int64)
            lv = np.zeros(max(n, 1), dtype=np.int32)
            lib.bp_schedule_snapshot(h, i, C.byref(r), _ptr(ids, i64), _ptr(lv, i32))
            self.snapshots.append({"round": r.value, "block_ids": ids[:n].tolist(), "levels": lv[:n].tolist()})
        self.blocks = []
        for i in range(int(lib.bp_schedule_nblocks(h))):
            bid, fr = i64(), i64()
            n = lib.bp_schedule_block(h, i, C.byref(bid), C.byref(fr), None, None)
            nid = np.zeros(max(n, 1), dtype=np.int32)
            fid = np.zeros(max(fr.value, 1), dtype=np.int64)
            lib.bp_schedule_block(h, i, C.byref(bid), C.byref(fr), _ptr(nid, i32), _ptr(fid, i64))
            self.blocks.append({"block_id": bid.value, "frames": fr.value, "noise_ids": nid[:n].tolist(),
                                "frame_ids": fid[:fr.value].tolist()})
        b = (i32 * self.cfg.devices)()
        e = (i32 * self.cfg.devices)()
        lib.bp_schedule_partition(h, b, e)
        self.partition = [(b[j], e[j]) for j in range(self.cfg.devices)]

    PASS_FIELDS = ("round", "block", "level", "version", "ctx", "ctx_block", "ctx_frames", "ctx_version",
                   "ctx_first_frame", "center_frames", "tokens", "center_tokens", "cached_context_id",
                   "ncapture", "earliest", "slot0", "completion", "finishes_block", "phase", "nframes")

    def rank_program(self, rank: int) -> List[tuple]:
        """The ordered ops the NCCL executor issues on `rank`: (kind, pass),
        kind 0 = stage forward (+ send), 1 = rank-0 eps receive + update."""
        n = int(lib.bp_schedule_rank_program(self._h, rank, None, 0))
        out = np.zeros(2 * max(n, 1), dtype=np.int64)
        lib.bp_schedule_rank_program(self._h, rank, _ptr(out, i64), n)
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(n)]

    def pass_record(self, i: int) -> Dict[str, Any]:
        rec = np.zeros(20, dtype=np.int64)
        lib.bp_schedule_pass(self._h, i, _ptr(rec, i64), None, None, None)
        d = dict(zip(self.PASS_FIELDS, rec.tolist()))
        lv = np.zeros(max(d["nframes"], 1), dtype=np.int32)
        fi = np.zeros(max(d["nframes"], 1), dtype=np.int64)
        cp = np.zeros(max(d["ncapture"], 1), dtype=np.int32)
        lib.bp_schedule_pass(self._h, i, _ptr(rec, i64), _ptr(lv, i32), _ptr(fi, i64), _ptr(cp, i32))
        d["frame_levels"] = lv[:d["nframes"]].tolist()
        d["frame_ids"] = fi[:d["nframes"]].tolist()
        d["capture_frames"] = cp[:d["ncapture"]].tolist()
        return d

    def block_meta(self, block_id: int) -> Dict[str, Any]:
        rec = np.zeros(4, dtype=np.int64)
        lib.bp_schedule_block_meta(self._h, block_id, _ptr(rec, i64))
        return {"frames": int(rec[0]), "append_round": int(rec[1]), "fresh": bool(rec[2]),
                "fresh_state": int(rec[3]) & ((1 << 64) - 1)}

    def __del__(self):
        try:
            if self._h:
                lib.bp_schedule_destroy(self._h)
        except Exception:
            pass


def measure_bubbles(events: np.ndarray, devices: int) -> Dict[str, Any]:
    """measure_bubbles (engine.cpp:505-555) over (slot, device, block, level, phase, round) rows."""
    st = {"first_slot": 0, "last_slot": 0, "busy_per_device": 0, "idle_per_device": 0,
          "warmup_idle": 0, "steady_idle": 0, "cooldown_idle": 0, "ratio": 0.0}
    if len(events) == 0:
        return st
    if devices < 1:
        raise errors.SchedulingError("malformed event log: no devices")
    if any(int(e[1]) < 0 or int(e[1]) >= devices for e in events):
        raise errors.SchedulingError("malformed event log: device out of range")
    # per-device events in log order, as engine.cpp:510-530 walks them
    per = [[(int(e[0]), int(e[4])) for e in events if int(e[1]) == d] for d in range(devices)]
    first, last = int(events[:, 0].min()), int(events[:, 0].max())
    busy = len(per[0])
    if any(len(v) != busy for v in per):
        raise errors.SchedulingError("malformed event log: devices saw different pass counts")
    if any(v[i][0] <= v[i - 1][0] for v in per for i in range(1, len(v))):
        raise errors.SchedulingError("malformed event log: duplicate slot on one device")
    st.update(first_slot=first, last_slot=last, busy_per_device=busy,
              idle_per_device=(last - first + 1) - busy)
    keys = ("warmup_idle", "steady_idle", "cooldown_idle")
    for v in per:
        nxt = 0
        for s in range(first, last + 1):
            while nxt < len(v) and v[nxt][0] < s:
                nxt += 1
            if nxt < len(v) and v[nxt][0] == s:
                continue
            st[keys[v[nxt][1] if nxt < len(v) else 2]] += 1
    idle = st["idle_per_device"] * devices
    st["ratio"] = 0.0 if idle <= 0 else idle / (idle + busy * devices)
    return st


def coordinated_noise_ids(num_b: int, num_c: int, appends: int, seed: int = 2) -> List[List[int]]:
    """bindings.cpp:146-160: ids of the first block and `appends` coordinated appends."""
    s = Schedule({"num_b": num_b, "num_c": num_c, "steps": 1, "blocks": appends + 1, "devices": 1,
                  "layers": 1, "hidden": 2, "heads": 1, "channels": 1, "height": 1, "width": 1,
                  "seed_noise": seed})
    return [b["noise_ids"] for b in s.blocks]


class _Pinned:
    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        check(lib.bp_host_alloc(nbytes, C.byref(self.ptr)))
        self.nbytes = nbytes

    def __del__(self):
        try:
            if self.ptr:
                lib.bp_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array over page-locked host memory (cudaMallocHost); the
    allocation lives as long as the array (its base buffer holds it)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape))
    nbytes = max(1, n * dt.itemsize)
    mem = _Pinned(nbytes)
    buf = (C.c_uint8 * nbytes).from_address(mem.ptr.value)
    buf._bp_pinned = mem
    return np.frombuffer(buf, dtype=dt, count=n).reshape(shape)


def nccl_unique_ids(world: int) -> bytes:
    """`world` NCCL unique ids (128 bytes each), one per pipeline channel, made
    on the rank that broadcasts them to the others (ncclGetUniqueId)."""
    buf = bytearray()
    for _ in range(world):
        b = (C.c_uint8 * 128)()
        check(lib.bp_nccl_unique_id(b))
        buf += bytes(b)
    return bytes(buf)


# ---- engine.hpp: the pipeline ---------------------------------------------------------------
class Pipeline:
    """run_pipeline (engine.cpp:255-497) on B200: build once, run many times."""

    def __init__(self, config: ConfigLike, rank: int = 0, world: int = 1, device: int = 0,
                 nccl_ids: Optional[bytes] = None,
                 ipc_exchange: Optional[Callable[[bytes], Sequence[bytes]]] = None,
                 bootstrap_dir: Optional[str] = None, bootstrap_timeout_ms: int = 120000):
        """Multi-process transports (one process per stage, world = devices):
        either bootstrap_dir -- a fresh directory every rank can see; the ranks
        rendezvous through files there (bp_bootstrap_nccl_ids /
        bp_bootstrap_ipc), no other runtime needed -- or the caller's own
        exchange: nccl_ids (world x 128-byte NCCL unique ids, transport
        "nccl") / ipc_exchange (all-gathers this rank's 64-byte IPC handle and
        returns every rank's in rank order, transport "ipc")."""
        self.cfg = _cfg(config)
        self._h = C.c_void_p()
        desc = self.cfg.to_desc()
        multi = world > 1 and self.cfg.transport in ("nccl", "ipc")
        if multi and bootstrap_dir is not None and self.cfg.transport == "nccl" and nccl_ids is None:
            got = (C.c_uint8 * (128 * world))()
            check(lib.bp_bootstrap_nccl_ids(bootstrap_dir.encode(), rank, world, bootstrap_timeout_ms, got))
            nccl_ids = bytes(got)
        ids = None
        if nccl_ids is not None:
            buf = (C.c_uint8 * len(nccl_ids)).from_buffer_copy(nccl_ids)
            ids = C.cast(buf, C.POINTER(C.c_uint8))
        check(lib.bp_pipeline_create(C.byref(desc), rank, world, device, ids, C.byref(self._h)))
        if self.cfg.transport == "ipc" and world > 1:
            if bootstrap_dir is not None and ipc_exchange is None:
                check(lib.bp_bootstrap_ipc(self._h, bootstrap_dir.encode(), rank, world, bootstrap_timeout_ms))
            else:
                if ipc_exchange is None:
                    raise errors.ConfigError("transport 'ipc' needs ipc_exchange or bootstrap_dir to share handles")
                mine = (C.c_uint8 * 64)()
                check(lib.bp_ipc_handle(self._h, mine))
                allh = b"".join(bytes(h) for h in ipc_exchange(bytes(mine)))
                if len(allh) != 64 * world:
                    raise errors.ConfigError("ipc_exchange must return one 64-byte handle per rank")
                hb = (C.c_uint8 * len(allh)).from_buffer_copy(allh)
                check(lib.bp_ipc_connect(self._h, hb))
        self.schedule = Schedule(self.cfg)

    def close(self):
        if self._h:
            lib.bp_pipeline_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, emit: Optional[Callable] = None, collect: bool = True) -> List[Dict[str, Any]]:
        """One whole generation. Returns the emitted blocks (EmittedBlock,
        engine.hpp:73-78) in emission order with host fp64 frames."""
        blocks: List[Dict[str, Any]] = []
        hwc = self.cfg.height * self.cfg.width * self.cfg.channels

        def _cb(user, block_id, frames, data, nids_p, nids, fids_p):
            arr = np.ctypeslib.as_array(data, shape=(frames * hwc,)).copy() if collect else None
            item = {"block_id": int(block_id),
                    "frames": None if arr is None else arr.reshape(frames, self.cfg.height, self.cfg.width,
                                                                 self.cfg.channels),
                    "noise_ids": [nids_p[k] for k in range(nids)],
                    "frame_ids": [fids_p[k] for k in range(frames)]}
            blocks.append(item)
            if emit is not None:
                emit(item)

        cb = EMIT_FN(_cb)
        check(lib.bp_pipeline_run(self._h, cb, None))
        return blocks

    def set_pool(self, pool: Optional[np.ndarray]) -> None:
        """Host-supplied noise pool (replaces build_pool(seed_noise),
        noise.cpp:26-48): M = num_b + num_c/2 entries in id order, fp64, the
        layout build_pool returns. Each later run uploads it host->device
        (pass a pinned_empty() array for a DMA-speed copy). None restores the
        seeded device pool."""
        if pool is None:
            self._pool = None
            check(lib.bp_pipeline_set_pool(self._h, C.cast(None, C.POINTER(f64)), 0))
            return
        if pool.dtype != np.float64 or not pool.flags["C_CONTIGUOUS"]:
            raise TypeError("pool must be a C-contiguous float64 array")
        self._pool = pool  # borrowed by the engine for every later run
        check(lib.bp_pipeline_set_pool(self._h, _ptr(pool, f64), pool.size))

    def set_profiling(self, on: bool) -> None:
        """CUDA events around every class of launches in later runs (the
        per-class device times appear in stats()); off for timed runs."""
        check(lib.bp_pipeline_set_profiling(self._h, int(bool(on))))

    def run_device(self) -> None:
        """One whole generation with the emitted latents left in HBM (no
        device->host copies); bp_pipeline_block exposes their device pointers."""
        check(lib.bp_pipeline_run(self._h, C.cast(None, EMIT_FN), None))

    def stats(self) -> Dict[str, Any]:
        s = PipelineStats()
        check(lib.bp_pipeline_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in PipelineStats._fields_}

    def trace(self) -> List[Dict[str, Any]]:
        out = []
        for i in range(int(lib.bp_pipeline_ntrace(self._h))):
            r, b, rows, cols = i64(), i64(), i64(), i64()
            check(lib.bp_pipeline_trace(self._h, i, C.byref(r), C.byref(b), C.byref(rows), C.byref(cols), None))
            eps = np.empty((rows.value, cols.value), dtype=np.float64)
            check(lib.bp_pipeline_trace(self._h, i, C.byref(r), C.byref(b), C.byref(rows), C.byref(cols),
                                        _ptr(eps, f64)))
            out.append({"round": r.value, "block_id": b.value, "eps": eps})
        return out


def run_pipeline(config: ConfigLike = None) -> Dict[str, Any]:
    """bindings.cpp:139-141 + run_to_dict (:37-72), plus the event log,
    snapshots and (when record_trace) the per-pass eps trace."""
    cfg = _cfg(config)
    p = Pipeline(cfg)
    try:
        blocks = p.run()
        sched = p.schedule
        out = {"blocks": blocks, "rounds": sched.rounds,
               "bubbles": measure_bubbles(sched.events, cfg.devices),
               "ledger": sched.ledger, "events": sched.events, "queue_snapshots": sched.snapshots,
               "stats": p.stats()}
        if cfg.record_trace:
            out["trace"] = p.trace()
        return out
    finally:
        p.close()


def serial_oracle(config: ConfigLike = None) -> Dict[str, Any]:
    """serial_oracle (engine.cpp:499-503): the same run on a single stage."""
    cfg = _cfg(config)
    cfg = PipelineConfig(**{**cfg.__dict__, "devices": 1, "threaded": False, "uneven_split": False,
                            "layer_split": None})
    return run_pipeline(cfg)
