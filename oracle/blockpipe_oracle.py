"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's block-wise
denoising path (numpy fp64), used as the checker in tests/ and never by the
product. Pinned against tests/golden/goldens.json, which tests/golden/
make_goldens.py generates from the UNMODIFIED reference library (oracle/_ref).

Each function cites the reference (P = /root/reference/proj) it restates.
matmul uses numpy's reduction order, so results match the reference to
~1e-15 relative, not bitwise; integer / schedule outputs are exact.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from collections import deque
from typing import Dict, List, Optional

import numpy as np

PHI = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1
_RNG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libbp_oracle_rng.so")


# ---- rng.cpp ----------------------------------------------------------------------
def mix(z: int) -> int:  # rng.cpp:12-18
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class RandomSource:
    """RandomSource (rng.hpp:28-47): splitmix64 + Box-Muller (rng.cpp:12-49)."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def next_u64(self) -> int:
        self.state = (self.state + PHI) & M64
        return mix(self.state)

    def next_normal(self) -> float:  # rng.cpp:24-31 (libm log/cos/sqrt, as glibc)
        a, b = self.next_u64(), self.next_u64()
        u1 = float((a >> 11) + 1) * (1.0 / 9007199254740992.0)
        u2 = float(b >> 11) * (1.0 / 9007199254740992.0)
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def normal_tensor(self, shape, sigma: float = 1.0) -> np.ndarray:  # rng.cpp:35-39
        n = int(np.prod(shape))
        if os.path.exists(_RNG):
            lib = C.CDLL(_RNG)
            lib.bpo_normals.restype = C.c_uint64
            lib.bpo_normals.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.POINTER(C.c_double)]
            out = np.empty(n)
            self.state = lib.bpo_normals(self.state, n, sigma, out.ctypes.data_as(C.POINTER(C.c_double)))
            return out.reshape(shape)
        return np.array([self.next_normal() * sigma for _ in range(n)]).reshape(shape)

    def next_below(self, n: int) -> int:  # rng.cpp:33
        return self.next_u64() % n

    def permutation(self, n: int) -> List[int]:  # rng.cpp:41-49, Fisher-Yates
        p = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.next_below(i + 1)
            p[i], p[j] = p[j], p[i]
        return p


def derive_seed(base: int, tags) -> int:  # rng.cpp:51-60
    s = base & M64
    for t in tags:
        s = mix(((s ^ (((t + 1) * PHI) & M64)) + PHI) & M64)
    return s


# ---- model.cpp --------------------------------------------------------------------------
ROLES = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "cq": 4, "ck": 5, "cv": 6, "co": 7, "w1": 8, "w2": 9,
         "ln1_g": 10, "ln1_b": 11, "ln2_g": 12, "ln2_b": 13, "ln3_g": 14, "ln3_b": 15}


def draw(seed, layer, role, shape, fan_in):  # model.cpp:26-30
    return RandomSource(derive_seed(seed, [layer, role])).normal_tensor(shape, 1.0 / math.sqrt(fan_in))


def build_layer(cfg, seed, layer):  # model.cpp:87-107
    h, F = cfg["hidden"], cfg.get("ffn") or 4 * cfg["hidden"]
    w = {}
    for name, role in ROLES.items():
        if name == "w1":
            w[name] = draw(seed, layer, role, (h, F), h)
        elif name == "w2":
            w[name] = draw(seed, layer, role, (F, h), F)
        elif name.startswith("ln"):
            w[name] = draw(seed, layer, role, (1, h), h)
        else:
            w[name] = draw(seed, layer, role, (h, h), h)
    return w


def build_chunk(cfg, seed, begin, end):  # model.cpp:109-128
    ch = {"cfg": cfg, "begin": begin, "end": end, "layers": [build_layer(cfg, seed, l) for l in range(begin, end)]}
    if begin == 0:
        ch["w_in"] = draw(seed, cfg["layers"], 100, (cfg["channels"], cfg["hidden"]), cfg["channels"])
    if end == cfg["layers"]:
        ch["w_out"] = draw(seed, cfg["layers"], 101, (cfg["hidden"], cfg["channels"]), cfg["hidden"])
    return ch


def build_context(cfg, seed):  # model.cpp:150-153
    return RandomSource(seed).normal_tensor((cfg["context_len"], cfg["hidden"]))


def layer_norm(x, eps=1e-5):  # tensor.cpp:128-146
    mean = x.sum(axis=1, keepdims=True) / x.shape[1]
    var = ((x - mean) ** 2).sum(axis=1, keepdims=True) / x.shape[1]
    return (x - mean) * (1.0 / np.sqrt(var + eps))


def ln_affine(x, g, b):  # model.cpp:32-41
    return layer_norm(x) * g + b


def gelu(x):  # model.cpp:43
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def attention(q, k, v, heads):  # model.cpp:47-72
    m, h = q.shape
    dh = h // heads
    out = np.zeros((m, h))
    for hd in range(heads):
        sl = slice(hd * dh, (hd + 1) * dh)
        s = (q[:, sl] @ k[:, sl].T) * (1.0 / math.sqrt(dh))
        s = np.exp(s - s.max(axis=1, keepdims=True))
        out[:, sl] = (s / s.sum(axis=1, keepdims=True)) @ v[:, sl]
    return out


def sinusoid(pos, hidden):  # model.cpp:155-163
    e = np.zeros(hidden)
    for i in range((hidden + 1) // 2):
        f = math.pow(10000.0, -2.0 * i / hidden)
        e[2 * i] = math.sin(pos * f)
        if 2 * i + 1 < hidden:
            e[2 * i + 1] = math.cos(pos * f)
    return e


def forward_chunk(ch, payload, levels, frame_ids, context, mode="off", cache=None, recorded=None,
                  capture=(), record_inputs=False):
    """forward_chunk (model.cpp:227-336). Returns (payload, captured, recorded)."""
    cfg = ch["cfg"]
    tpf = cfg["height"] * cfg["width"]
    h = cfg["hidden"]
    rows = [f * tpf + t for f in capture for t in range(tpf)]
    if ch["begin"] == 0:
        x = payload @ ch["w_in"]
        for f in range(len(levels)):
            te = sinusoid(levels[f] + 1000000, h)
            for t in range(tpf):
                x[f * tpf + t] += sinusoid(frame_ids[f] * tpf + t, h) + te
    else:
        x = payload.copy()
    captured = [] if (rows and mode == "on") else None
    rec = [] if (rows and (mode == "recompute" or record_inputs)) else None
    for li, w in enumerate(ch["layers"]):
        if rec is not None:
            rec.append(x[rows].copy())
        ln1 = ln_affine(x, w["ln1_g"], w["ln1_b"])
        q, k, v = ln1 @ w["wq"], ln1 @ w["wk"], ln1 @ w["wv"]
        if cache is not None:
            kp, vp = cache[li]
        elif recorded is not None:
            lp = ln_affine(recorded[li], w["ln1_g"], w["ln1_b"])
            kp, vp = lp @ w["wk"], lp @ w["wv"]
        else:
            kp = vp = None
        if captured is not None:
            captured.append((k[rows].copy(), v[rows].copy()))
        kk = k if kp is None else np.concatenate([kp, k])
        vv = v if vp is None else np.concatenate([vp, v])
        x = x + attention(q, kk, vv, cfg["heads"]) @ w["wo"]
        ln2 = ln_affine(x, w["ln2_g"], w["ln2_b"])
        x = x + attention(ln2 @ w["cq"], context @ w["ck"], context @ w["cv"], cfg["heads"]) @ w["co"]
        ln3 = ln_affine(x, w["ln3_g"], w["ln3_b"])
        x = x + gelu(ln3 @ w["w1"]) @ w["w2"]
    out = x @ ch["w_out"] if ch["end"] == cfg["layers"] else x
    return out, captured, rec


def sinusoid_rows(pos: np.ndarray, hidden: int) -> np.ndarray:
    """position_embedding (model.cpp:155-163) for many positions at once
    (numpy sin/cos: within an ulp or two of glibc's, enough for the
    fp32 / bf16 tolerances this restatement checks at Wan shapes)."""
    half = (hidden + 1) // 2
    f = np.array([math.pow(10000.0, -2.0 * i / hidden) for i in range(half)])
    ang = np.asarray(pos, dtype=np.float64)[:, None] * f[None, :]
    e = np.zeros((ang.shape[0], hidden))
    e[:, 0::2] = np.sin(ang)
    e[:, 1::2] = np.cos(ang)[:, :hidden // 2]
    return e


def forward_chunk_rows(ch, payload, levels, frame_ids, context, out_rows, prefix=None, capture=()):
    """forward_chunk (model.cpp:227-336) of a ONE-layer chunk, restated for
    the output rows `out_rows` only, so it runs at Wan shapes on a host.
    Every op except attention is per token, and attention needs the K/V of
    every row (prefix first, model.cpp:302-318) but the queries of the
    requested rows only. Returns (out[out_rows], (K, V) at the capture rows)."""
    cfg = ch["cfg"]
    assert len(ch["layers"]) == 1
    tpf, h = cfg["height"] * cfg["width"], cfg["hidden"]
    nf = len(levels)
    if ch["begin"] == 0:  # model.cpp:245-260
        x = payload @ ch["w_in"]
        t = np.arange(nf * tpf)
        f = t // tpf
        pos = np.asarray(frame_ids, dtype=np.int64)[f] * tpf + (t - f * tpf)
        te = sinusoid_rows(np.asarray(levels, dtype=np.int64) + 1000000, h)
        x += sinusoid_rows(pos, h) + te[f]
    else:
        x = payload.copy()
    w = ch["layers"][0]
    ln1 = ln_affine(x, w["ln1_g"], w["ln1_b"])
    k, v = ln1 @ w["wk"], ln1 @ w["wv"]
    cap_rows = [fr * tpf + tt for fr in capture for tt in range(tpf)]
    captured = (k[cap_rows].copy(), v[cap_rows].copy()) if cap_rows else None
    if prefix is not None:
        k, v = np.concatenate([prefix[0], k]), np.concatenate([prefix[1], v])
    R = np.asarray(out_rows)
    xr = x[R] + attention(ln1[R] @ w["wq"], k, v, cfg["heads"]) @ w["wo"]
    ln2 = ln_affine(xr, w["ln2_g"], w["ln2_b"])
    xr = xr + attention(ln2 @ w["cq"], context @ w["ck"], context @ w["cv"], cfg["heads"]) @ w["co"]
    ln3 = ln_affine(xr, w["ln3_g"], w["ln3_b"])
    xr = xr + gelu(ln3 @ w["w1"]) @ w["w2"]
    out = xr @ ch["w_out"] if ch["end"] == cfg["layers"] else xr
    return out, captured


# ---- block_queue.cpp / noise.cpp / engine.cpp (serial, round-atomic) ----------------------------
def run_pipeline(cfg: Dict, record_trace=False) -> Dict:
    """serial_oracle (engine.cpp:499-503): the run_pipeline round loop
    (engine.cpp:343-457) on one worker, cache per DeviceWorker semantics."""
    T, B, nb, nc = cfg["steps"], cfg["blocks"], cfg["num_b"], cfg["num_c"]
    ctx = nc // 2
    reverse = cfg.get("order", "reverse") == "reverse"
    mode = cfg.get("cache", "on")
    retain = cfg.get("retain_clean_context", True)
    H, W, Cc = cfg["height"], cfg["width"], cfg["channels"]
    tpf = H * W
    ch = build_chunk(cfg, cfg.get("seed_model", 1), 0, cfg["layers"])
    context = build_context(cfg, cfg.get("seed_context", 3))
    M = nb + ctx
    pool = RandomSource(derive_seed(cfg.get("seed_noise", 2), [0])).normal_tensor((M, H, W, Cc))  # noise.cpp:26-48
    rng = RandomSource(derive_seed(cfg.get("seed_noise", 2), [1]))
    q: deque = deque()
    retained = None
    emitted = []
    next_frame = 0
    cache = recorded = None
    trace = []
    for r in range(1, T + B):
        new = None
        if r <= B:  # make_block (engine.cpp:301-324), coordinated strategy (noise.cpp:70-101)
            if r == 1:
                ids = rng.permutation(M)
            else:
                window = q[-1]["noise_ids"][-ctx:] if ctx else []
                rem = [i for i in range(M) if i not in set(window)]
                ids = [rem[p] for p in rng.permutation(len(rem))]
            new = {"id": r, "frames": pool[ids].copy(), "prev": None, "level": T, "updates": 0, "noise_ids": ids,
                   "frame_ids": list(range(next_frame, next_frame + len(ids)))}
            next_frame += len(ids)
        if q and q[0]["level"] == 0:  # emit_if_clean + advance (block_queue.cpp:44-78)
            head = q.popleft()
            emitted.append(head)
            if retain and ctx:
                retained = (head["id"], head["frames"][-ctx:].copy(), head["frame_ids"][-ctx:])
        if new is not None:
            q.append(new)
        order = [b["id"] for b in q]
        if reverse:
            order.reverse()
        find = {b["id"]: b for b in q}
        results = []
        for bid in order:
            blk = find[bid]
            fr, lv, fi = [], [], []
            e = find.get(bid - 1)
            if ctx and e is not None:  # assemble_extended (block_queue.cpp:88-138)
                src = e["frames"] if e["updates"] == blk["updates"] else e["prev"]
                fr.append(src[-ctx:])
                lv += [blk["level"]] * ctx
                fi += e["frame_ids"][-ctx:]
            elif ctx and retained is not None and retained[0] == bid - 1:
                fr.append(retained[1])
                lv += [0] * ctx
                fi += list(retained[2])
            fr.append(blk["frames"])
            lv += [blk["level"]] * len(blk["frame_ids"])
            fi += blk["frame_ids"]
            payload = np.concatenate(fr).reshape(-1, Cc)
            use_cache = mode != "off" and reverse and ctx and (bid + 1) in find
            capture = list(range(len(lv) - len(blk["frame_ids"]), len(lv) - len(blk["frame_ids"]) + ctx)) \
                if (mode != "off" and reverse and ctx and (bid - 1) in find) else []
            out, cap, rec = forward_chunk(ch, payload, lv, fi, context, mode,
                                          cache=cache if (use_cache and mode == "on") else None,
                                          recorded=recorded if (use_cache and mode == "recompute") else None,
                                          capture=capture)
            cache, recorded = cap, rec
            results.append((bid, out))
        for bid, out in results:  # collect + scheduler_step + apply_update (engine.cpp:418-447)
            blk = find[bid]
            if record_trace:
                trace.append({"round": r, "block_id": bid, "eps": out})
            f = blk["frames"].shape[0]
            eps = out[-f * tpf:].reshape(blk["frames"].shape)
            blk["prev"], blk["frames"] = blk["frames"], blk["frames"] - eps * (1.0 / T)
            blk["level"] -= 1
            blk["updates"] += 1
    if q and q[0]["level"] == 0:
        emitted.append(q.popleft())
    return {"blocks": [{"block_id": b["id"], "frames": b["frames"], "noise_ids": b["noise_ids"],
                        "frame_ids": b["frame_ids"]} for b in emitted], "trace": trace}
