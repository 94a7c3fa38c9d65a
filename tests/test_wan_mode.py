"""The optional Wan2.1-style block ("block": "wan"; NOT a reference path, see
DESIGN.md section 10): adaLN modulation from the per-frame timestep MLP, gated
residuals, RMS-normalised Q/K with 3D RoPE, tanh-GELU. Checked against the
numpy fp64 statement in oracle/wan_oracle.py: fp64 <= 1e-10, fp32 <= 1e-4,
bf16 tensor-core path <= 2e-2 (rel-L2), the same tolerances as the reference
block's parity tests."""
import numpy as np
import pytest

from oracle import wan_oracle as wo


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


TINY = dict(layers=2, hidden=256, heads=2, channels=16, height=4, width=6, context_len=16, ffn=0)


# ---- CPU: the oracle's own invariants and the config surface ------------------------------


def test_rope_is_a_rotation_and_identity_at_origin():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 256))
    z = np.zeros(5)
    assert np.array_equal(wo.rope(x, 2, z, z, z), x)
    y = wo.rope(x, 2, np.arange(5.0), np.arange(5.0) + 1, np.arange(5.0) + 2)
    pair = lambda v: v[:, 0::2] ** 2 + v[:, 1::2] ** 2  # noqa: E731
    assert np.allclose(pair(y), pair(x), rtol=1e-12, atol=1e-12)
    # relative positions: <rope(q, p), rope(k, p')> depends on p - p' only
    q, k = x[:1], x[1:2]
    a = (wo.rope(q, 2, [3.0], [1.0], [2.0]) * wo.rope(k, 2, [1.0], [0.0], [5.0])).sum()
    b = (wo.rope(q, 2, [7.0], [4.0], [0.0]) * wo.rope(k, 2, [5.0], [3.0], [3.0])).sum()
    assert abs(a - b) < 1e-10


def test_rope_split_matches_wan_rotary_dims():
    # Wan: d - 4 (d // 6) temporal and 2 (d // 6) height / width rotary dims
    for dh in (64, 128, 256):
        nt, nh = wo.rope_split(dh)
        assert 2 * nt == dh - 4 * (dh // 6) and 2 * nh == 2 * (dh // 6) and nt + 2 * nh == dh // 2


def test_zero_modulation_reduces_to_layernorm():
    """mod = e0 = 0 gives y = LN(x), gates 0: the layer leaves x unchanged
    except for the ungated cross-attention."""
    cfg = dict(TINY, layers=1)
    ch = wo.build_wan_chunk(cfg, 5, 0, 1)
    ch["begin"], ch["end"] = 1, 2  # a middle chunk: no entry projection, no head
    w = ch["layers"][0]
    w["mod"][:] = 0.0
    w["co"][:] = 0.0
    for k in ("tp", "tpb"):
        ch[k][:] = 0.0
    x = np.random.default_rng(1).standard_normal((24, 256))
    out, _ = wo.forward_chunk_wan(ch, x, [3], [0], wo.build_context(cfg, 6))
    assert np.array_equal(out, x)


def test_wan_config_surface(bp):
    cfg = bp.PipelineConfig.from_dict({"block": "wan", "layers": 2, "hidden": 256, "heads": 2})
    assert cfg.model_desc().block == 1
    assert bp.PipelineConfig.from_dict({}).model_desc().block == 0
    with pytest.raises(bp.ConfigError):
        bp.PipelineConfig.from_dict({"block": "dit"})
    # the recompute route and its audit are not built for the Wan block
    for extra in ({"cache": "recompute"}, {"check_cache": True}):
        with pytest.raises(bp.ConfigError):
            bp.Schedule(bp.PipelineConfig.from_dict({"block": "wan", **extra}))
    bp.Schedule(bp.PipelineConfig.from_dict({"block": "wan", "cache": "on"}))


# ---- GPU: stages and the pipeline vs the oracle ------------------------------------------


def _oracle_two_passes(cfg, seed, begin, end, ctx_seed, x0, x1):
    ch = wo.build_wan_chunk(cfg, seed, begin, end)
    ctx = wo.build_context(cfg, ctx_seed)
    a, cap = wo.forward_chunk_wan(ch, x0, [7, 7], [0, 1], ctx, capture=[1])
    b, _ = wo.forward_chunk_wan(ch, x1, [6, 6], [1, 2], ctx, prefix=cap)
    return a, b, cap


def _stage_two_passes(st, x0, x1):
    a = st.forward_chunk(x0, [7, 7], [0, 1], capture_frames=[1], mode="on")["payload"]
    cap = [(st.cache_rows(l, 0), st.cache_rows(l, 1)) for l in range(st.end - st.begin)]
    b = st.forward_chunk(x1, [6, 6], [1, 2], mode="on", use_prev=1)["payload"]
    return a, b, cap


@pytest.mark.gpu
@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("f32", 1e-4), ("bf16", 2e-2)])
def test_wan_stage_vs_oracle(bp, prec, tol):
    """A whole 2-layer chunk (entry projection, layers, modulated head): a
    capture pass, then a pass over [cached post-RoPE K/V ++ current]; the
    captured K / V themselves too."""
    cfg = bp.PipelineConfig(block="wan", **TINY)
    rng = np.random.default_rng(3)
    x0, x1 = rng.standard_normal((48, 16)), rng.standard_normal((48, 16))
    wa, wb, wcap = _oracle_two_passes(TINY, 5, 0, 2, 6, x0, x1)
    st = bp.Stage(cfg, 5, 0, 2, 6, precision=prec)
    try:
        ga, gb, gcap = _stage_two_passes(st, x0, x1)
    finally:
        st.close()
    assert rel(ga, wa) <= tol, rel(ga, wa)
    assert rel(gb, wb) <= tol, rel(gb, wb)
    for (gk, gv), (k, v) in zip(gcap, wcap):
        assert rel(gk, k) <= tol and rel(gv, v) <= tol


@pytest.mark.gpu
def test_wan_stage_dh128_bf16_vs_oracle(bp):
    """Head dim 128 (Wan's; 22 / 21 / 21 rotary pairs), 4 heads, two chunks
    of a 2-layer model chained through the hidden state: the tcgen05 GEMMs
    with the gated-residual and tanh-GELU epilogues, the pair attention over
    the RoPE'd prefix, the bf16 RMSNorm+RoPE kernel."""
    m = dict(TINY, hidden=512, heads=4)
    cfg = bp.PipelineConfig(block="wan", **m)
    rng = np.random.default_rng(8)
    x0, x1 = rng.standard_normal((48, 16)), rng.standard_normal((48, 16))
    ch0, ch1 = wo.build_wan_chunk(m, 9, 0, 1), wo.build_wan_chunk(m, 9, 1, 2)
    ctx = wo.build_context(m, 10)
    h0, c0 = wo.forward_chunk_wan(ch0, x0, [7, 7], [0, 1], ctx, capture=[1])
    w0, c1 = wo.forward_chunk_wan(ch1, h0, [7, 7], [0, 1], ctx, capture=[1])
    h1, _ = wo.forward_chunk_wan(ch0, x1, [6, 6], [1, 2], ctx, prefix=c0)
    w1, _ = wo.forward_chunk_wan(ch1, h1, [6, 6], [1, 2], ctx, prefix=c1)
    s0, s1 = bp.Stage(cfg, 9, 0, 1, 10, precision="bf16"), bp.Stage(cfg, 9, 1, 2, 10, precision="bf16")
    try:
        g0 = s0.forward_chunk(x0, [7, 7], [0, 1], capture_frames=[1], mode="on")["payload"]
        ga = s1.forward_chunk(g0, [7, 7], [0, 1], capture_frames=[1], mode="on")["payload"]
        g1 = s0.forward_chunk(x1, [6, 6], [1, 2], mode="on", use_prev=1)["payload"]
        gb = s1.forward_chunk(g1, [6, 6], [1, 2], mode="on", use_prev=1)["payload"]
    finally:
        s0.close()
        s1.close()
    assert rel(g0, h0) <= 2e-2 and rel(ga, w0) <= 2e-2, (rel(g0, h0), rel(ga, w0))
    assert rel(gb, w1) <= 2e-2, rel(gb, w1)


@pytest.mark.gpu
def test_wan_recompute_rejected(bp):
    cfg = bp.PipelineConfig(block="wan", **TINY)
    st = bp.Stage(cfg, 5, 0, 2, 6, precision="f32")
    try:
        x = np.zeros((48, 16))
        with pytest.raises(bp.ConfigError):
            st.forward_chunk(x, [7, 7], [0, 1], capture_frames=[1], mode="recompute")
    finally:
        st.close()


@pytest.mark.gpu
def test_wan_pipeline_bf16_vs_f64_and_split(bp):
    """The block-wise denoising pipeline with the Wan block: bf16 latents
    within 2e-2 of the fp64 path; two loopback stages equal one in fp64."""
    base = dict(TINY, num_b=2, num_c=4, steps=3, blocks=2, mode="single", block="wan")

    def lat(out):
        return np.concatenate([b["frames"].ravel() for b in out["blocks"]])

    f64 = lat(bp.run_pipeline(bp.PipelineConfig.from_dict(dict(base, devices=1, precision="f64"))))
    two = lat(bp.run_pipeline(bp.PipelineConfig.from_dict(dict(base, devices=2, precision="f64"))))
    bf = lat(bp.run_pipeline(bp.PipelineConfig.from_dict(dict(base, devices=1, precision="bf16"))))
    assert np.isfinite(f64).all()
    assert rel(two, f64) <= 1e-12
    assert rel(bf, f64) <= 2e-2, rel(bf, f64)
    ref_block = lat(bp.run_pipeline(bp.PipelineConfig.from_dict(dict(base, block="reference", precision="f64"))))
    assert rel(ref_block, f64) > 1e-3  # the flag really switches the block


@pytest.mark.gpu
def test_gated_and_tanh_gemm_epilogues(bp):
    """kGemmResidualGatedF32 (x += gate[row / g] * A.W^T) and kGemmGeluTanhBf16
    on the tcgen05 pair GEMM vs fp64 numpy, ragged M / N."""
    from kernels import from_bf16_bits, load_testlib, to_bf16_bits
    lib = load_testlib()
    rng = np.random.default_rng(2)
    for M, N, K, grp in ((300, 256, 128, 7), (1000, 1536, 256, 130), (257, 4608, 64, 1000)):
        A = to_bf16_bits(rng.standard_normal((M, K)))
        W = to_bf16_bits(rng.standard_normal((N, K)) / np.sqrt(K))
        acc = from_bf16_bits(A).astype(np.float64) @ from_bf16_bits(W).astype(np.float64).T
        ng = (M + grp - 1) // grp
        gate = rng.standard_normal((ng, N)).astype(np.float32)
        x0 = rng.standard_normal((M, N)).astype(np.float32)
        x = x0.copy()
        st = lib.bp_selftest_gemm_gated(0, M, N, K, A.ctypes.data, K, W.ctypes.data, x.ctypes.data, N,
                                        gate.ctypes.data, grp, ng)
        assert st == 0, lib.bp_last_error()
        want = x0 + gate[np.arange(M) // grp] * acc
        assert rel(x, want) < 1e-5, rel(x, want)
        out = np.zeros((M, N), dtype=np.uint16)
        assert lib.bp_selftest_gemm(0, M, N, K, 5, A.ctypes.data, K, W.ctypes.data, out.ctypes.data, N) == 0
        g = 0.5 * acc * (1 + np.tanh(np.sqrt(2 / np.pi) * (acc + 0.044715 * acc ** 3)))
        assert rel(from_bf16_bits(out), g) < 1e-2, rel(from_bf16_bits(out), g)
