"""TEST INFRASTRUCTURE ONLY — numpy fp64 statement of the optional Wan2.1-style
block ("block": "wan"), the checker for the GPU's Wan mode in tests/. Never
imported by the product.

This mode is NOT part of the reference: the reference block is LayerNorm +
ln_affine with additive sinusoidal position / timestep embeddings
(P/src/model.cpp:32-43, 155-169, 227-336; P = /root/reference/proj).
BASELINE.json's north_star names adaLN modulation, 3D-RoPE and a timestep
embedding, the Wan2.1 DiT block (WanAttentionBlock / WanModel of the public
Wan2.1 release, Apache-2.0; no copy of it is in /root/reference or in this
image, so its published structure is restated here):

* time embedding per frame f, t = the frame's noise level (the integer the
  reference feeds timestep_embedding, model.cpp:165-169):
  s = [cos(t w_k), sin(t w_k)], w_k = 10000^(-k/128), k < 128;
  e_f = SiLU(s W_t1 + b_t1) W_t2 + b_t2;  e0_f = SiLU(e_f) W_tp + b_tp  (6h)
* per layer, (sh1, sc1, g1, sh2, sc2, g2) = mod_l + e0_f:
  y  = LN(x) (1 + sc1) + sh1                          (LN without affine, eps 1e-6)
  q  = RMS(y Wq) gq,  k = RMS(y Wk) gk,  v = y Wv      (RMSNorm over all h, eps 1e-6)
  q, k = RoPE3D(q), RoPE3D(k)                          (positions: frame id, row, column)
  x += g1 * (attention(q, [k_prefix ++ k], [v_prefix ++ v]) Wo)
  c  = LN(x) ln2_g + ln2_b                             (cross-attention norm, affine)
  x += attention(RMS(c Cq) gcq, RMS(ctx Ck) gck, ctx Cv) Co
  y2 = LN(x) (1 + sc2) + sh2
  x += g2 * (gelu_tanh(y2 W1) W2)
* head: (sh, sc) = head_mod + e_f;  eps = (LN(x) (1 + sc) + sh) W_out
* first stage: x = latents W_in (positions enter through RoPE, time through
  the modulation; no additive embeddings).
RoPE3D per head (dh = h / heads, c = dh / 2 complex pairs (x[2i], x[2i+1])):
pairs [0, nt) rotate by frame_id * 10000^(-2j / (2 nt)), the next nh by
row * 10000^(-2j / (2 nh)), the last nh by column * (same), with
nh = dh // 6 and nt = c - 2 nh (Wan: d - 4 (d // 6) and 2 (d // 6) rotary dims).

Weights: the reference's roles (model.cpp:17-24) keep their draws, so the
GEMM weights are the reference-mode ones; the Wan roles below are drawn the
same way (draw(seed, layer, role, shape, fan_in), model.cpp:26-30). RMSNorm
gains are 1 + draw(.., fan_in h).
"""
from __future__ import annotations

import math

import numpy as np

from oracle.blockpipe_oracle import attention, build_context, build_layer, draw, layer_norm

# Wan roles (per layer unless noted; "global" ones are keyed by layer = L like
# the reference's patchify / head draws)
R_MOD, R_QN, R_KN, R_CQN, R_CKN = 200, 201, 202, 203, 204
R_T1, R_TB1, R_T2, R_TB2, R_TP, R_TPB, R_HMOD = 210, 211, 212, 213, 214, 215, 216
FREQ_DIM = 256
EPS = 1e-6


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def rms(x, g):
    return x / np.sqrt((x * x).mean(axis=1, keepdims=True) + EPS) * g


def rope_split(dh):
    nh = dh // 6
    nt = dh // 2 - 2 * nh
    return nt, nh


def rope(x, heads, pos_t, pos_y, pos_x):
    """x [rows, h]; pos_* [rows] integer positions."""
    rows, h = x.shape
    dh = h // heads
    nt, nh = rope_split(dh)
    ang = np.zeros((rows, dh // 2))
    ang[:, :nt] = np.outer(pos_t, 10000.0 ** (-2.0 * np.arange(nt) / (2 * nt)))
    ang[:, nt:nt + nh] = np.outer(pos_y, 10000.0 ** (-2.0 * np.arange(nh) / (2 * nh)))
    ang[:, nt + nh:] = np.outer(pos_x, 10000.0 ** (-2.0 * np.arange(nh) / (2 * nh)))
    c, s = np.cos(ang), np.sin(ang)
    out = np.empty_like(x)
    for hd in range(heads):
        a = x[:, hd * dh:(hd + 1) * dh:2]
        b = x[:, hd * dh + 1:(hd + 1) * dh:2]
        out[:, hd * dh:(hd + 1) * dh:2] = a * c - b * s
        out[:, hd * dh + 1:(hd + 1) * dh:2] = a * s + b * c
    return out


def build_wan_chunk(cfg, seed, begin, end):
    """The reference chunk's draws plus the Wan roles."""
    h, L = cfg["hidden"], cfg["layers"]
    ch = {"cfg": cfg, "begin": begin, "end": end, "layers": []}
    for l in range(begin, end):
        w = build_layer(cfg, seed, l)
        w["mod"] = draw(seed, l, R_MOD, (6, h), h)
        for name, role in (("gq", R_QN), ("gk", R_KN), ("gcq", R_CQN), ("gck", R_CKN)):
            w[name] = 1.0 + draw(seed, l, role, (1, h), h)
        ch["layers"].append(w)
    ch["t1"] = draw(seed, L, R_T1, (FREQ_DIM, h), FREQ_DIM)
    ch["tb1"] = draw(seed, L, R_TB1, (1, h), FREQ_DIM)
    ch["t2"] = draw(seed, L, R_T2, (h, h), h)
    ch["tb2"] = draw(seed, L, R_TB2, (1, h), h)
    ch["tp"] = draw(seed, L, R_TP, (h, 6 * h), h)
    ch["tpb"] = draw(seed, L, R_TPB, (1, 6 * h), h)
    if begin == 0:
        ch["w_in"] = draw(seed, L, 100, (cfg["channels"], h), cfg["channels"])
    if end == L:
        ch["w_out"] = draw(seed, L, 101, (h, cfg["channels"]), h)
        ch["hmod"] = draw(seed, L, R_HMOD, (2, h), h)
    return ch


def time_embedding(ch, levels):
    """(e [frames, h], e0 [frames, 6h])"""
    half = FREQ_DIM // 2
    w = 10000.0 ** (-np.arange(half) / half)
    t = np.asarray(levels, dtype=np.float64)
    s = np.concatenate([np.cos(np.outer(t, w)), np.sin(np.outer(t, w))], axis=1)
    e = silu(s @ ch["t1"] + ch["tb1"]) @ ch["t2"] + ch["tb2"]
    e0 = silu(e) @ ch["tp"] + ch["tpb"]
    return e, e0


def forward_chunk_wan(ch, payload, levels, frame_ids, context, prefix=None, capture=()):
    """One Wan-mode pass. prefix: per layer (K, V) of the resident cache
    (post-RoPE), or None. Returns (out, captured [(K, V)] per layer or None)."""
    cfg = ch["cfg"]
    H, W = cfg["height"], cfg["width"]
    tpf = H * W
    heads = cfg["heads"]
    h = cfg["hidden"]
    nf = len(levels)
    S = nf * tpf
    frame_of = np.repeat(np.arange(nf), tpf)
    pos_t = np.repeat(np.asarray(frame_ids, dtype=np.float64), tpf)
    tok = np.tile(np.arange(tpf), nf)
    pos_y, pos_x = (tok // W).astype(np.float64), (tok % W).astype(np.float64)
    e, e0 = time_embedding(ch, levels)
    rows = [f * tpf + t for f in capture for t in range(tpf)]
    x = payload @ ch["w_in"] if ch["begin"] == 0 else payload.copy()
    captured = [] if rows else None
    for li, w in enumerate(ch["layers"]):
        m = (w["mod"][None, :, :] + e0.reshape(nf, 6, h))[frame_of]  # [S, 6, h]
        y = layer_norm(x, EPS) * (1.0 + m[:, 1]) + m[:, 0]
        q = rope(rms(y @ w["wq"], w["gq"]), heads, pos_t, pos_y, pos_x)
        k = rope(rms(y @ w["wk"], w["gk"]), heads, pos_t, pos_y, pos_x)
        v = y @ w["wv"]
        if captured is not None:
            captured.append((k[rows].copy(), v[rows].copy()))
        if prefix is not None:
            kk, vv = np.concatenate([prefix[li][0], k]), np.concatenate([prefix[li][1], v])
        else:
            kk, vv = k, v
        x = x + (attention(q, kk, vv, heads) @ w["wo"]) * m[:, 2]
        c = layer_norm(x, EPS) * w["ln2_g"] + w["ln2_b"]
        qc = rms(c @ w["cq"], w["gcq"])
        kc = rms(context @ w["ck"], w["gck"])
        x = x + attention(qc, kc, context @ w["cv"], heads) @ w["co"]
        y2 = layer_norm(x, EPS) * (1.0 + m[:, 4]) + m[:, 3]
        x = x + (gelu_tanh(y2 @ w["w1"]) @ w["w2"]) * m[:, 5]
    if ch["end"] == cfg["layers"]:
        hm = ch["hmod"][None, :, :] + e[:, None, :]  # [frames, 2, h]
        hm = hm[frame_of]
        x = (layer_norm(x, EPS) * (1.0 + hm[:, 1]) + hm[:, 0]) @ ch["w_out"]
    return x, captured


__all__ = ["build_wan_chunk", "build_context", "forward_chunk_wan", "time_embedding", "rope", "rope_split"]
