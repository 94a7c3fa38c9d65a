"""GPU parity through the C-ABI against the reference (goldens from the
unmodified reference library, and the library itself where it helps).
Tolerances are north_star's: fp64 parity mode <= 1e-12 rel-L2,
fp32 verification mode <= 1e-4, bf16 tensor-core path <= 2e-2; schedule,
noise ids and the noise pool are bit-exact."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "goldens.json")))


def golden(name):
    return np.load(os.path.join(ROOT, "tests", "golden", f"{name}_latents.npz"))["latents"]


def latents(out):
    return np.concatenate([b["frames"].ravel() for b in out["blocks"]])


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,prec,tol", [("cfg1", "f64", 1e-12), ("cfg1", "f32", 1e-4),
                                           ("cfg1_nocache", "f64", 1e-12), ("mid", "f64", 1e-12),
                                           ("mid", "f32", 1e-4), ("mid", "bf16", 2e-2)])
def test_pipeline_latents_vs_reference(bp, name, prec, tol):
    cfg = dict(G[name]["config"], precision=prec)
    out = bp.run_pipeline(cfg)
    r = rel(latents(out), golden(name))
    print(name, prec, r)
    assert r <= tol
    assert [b["noise_ids"] for b in out["blocks"]] == [b["noise_ids"] for b in G[name]["blocks"]]
    assert [b["frame_ids"] for b in out["blocks"]] == [b["frame_ids"] for b in G[name]["blocks"]]
    assert np.array_equal(out["events"], np.load(os.path.join(ROOT, "tests", "golden", f"{name}_latents.npz"))["events"])


@pytest.mark.parametrize("prec", ["f64", "bf16"])
@pytest.mark.parametrize("n", [2, 4])
def test_loopback_pipeline_equals_serial_bitwise(bp, prec, n):
    """test_engine.cpp:66-78 on the GPU: N stages == 1 stage, bitwise."""
    base = dict(G["mid"]["config"], precision=prec)
    a = bp.run_pipeline(dict(base, devices=n))
    b = bp.serial_oracle(base)
    assert all(np.array_equal(x["frames"], y["frames"]) for x, y in zip(a["blocks"], b["blocks"]))
    assert a["ledger"] != b["ledger"]  # different channel layout, same math


@pytest.mark.parametrize("prec", ["f64", "bf16"])
def test_cached_equals_recompute_bitwise(bp, prec):
    """test_engine.cpp:129-150: kCached == kRecompute on latents and on every pass's eps."""
    base = dict(G["mid"]["config"], precision=prec, devices=2, record_trace=True)
    c = bp.run_pipeline(dict(base, cache="on"))
    r = bp.run_pipeline(dict(base, cache="recompute"))
    assert all(np.array_equal(x["frames"], y["frames"]) for x, y in zip(c["blocks"], r["blocks"]))
    assert len(c["trace"]) == len(r["trace"]) == 18
    assert all(np.array_equal(x["eps"], y["eps"]) for x, y in zip(c["trace"], r["trace"]))


@pytest.mark.parametrize("prec", ["f64", "bf16"])
def test_fault_injection_caught(bp, prec):
    base = dict(G["mid"]["config"], precision=prec, devices=2, check_cache=True)
    with pytest.raises(bp.CacheError, match="cached V diverges at layer 0 flat index 0"):
        bp.run_pipeline(dict(base, fault_inject=True))
    quiet = bp.run_pipeline(base)  # the audit is quiet on an intact cache
    plain = bp.run_pipeline(dict(base, check_cache=False))
    assert all(np.array_equal(x["frames"], y["frames"]) for x, y in zip(quiet["blocks"], plain["blocks"]))


def test_trace_vs_reference_f64(bp, ref):
    """Per-pass eps (the sharper diagnostic) against the reference."""
    cfg = bp.PipelineConfig.from_dict(dict(G["cfg1"]["config"], record_trace=True, devices=2))
    got = bp.run_pipeline(cfg)["trace"]
    want = ref.run(cfg)["trace"]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g["round"], g["block_id"]) == (w["round"], w["block_id"])
        assert rel(g["eps"], w["eps"]) < 1e-12


@pytest.mark.parametrize("kw", [dict(strategy="complete-shuffle"), dict(strategy="subset"), dict(strategy="fresh"),
                                dict(strategy="repeat"), dict(retain_clean_context=False), dict(num_c=0),
                                dict(order="sequential"), dict(cache="off", order="sequential"),
                                dict(devices=4, steps=6, blocks=2)])
def test_engine_variants_vs_reference(bp, ref, kw):
    """test_engine.cpp:223-276 variants through the GPU engine vs the reference."""
    cfg = bp.PipelineConfig.from_dict(dict({"devices": 2, "layers": 4, "hidden": 16, "heads": 2, "steps": 4,
                                            "blocks": 4, "mode": "single"}, **kw))
    got, want = bp.run_pipeline(cfg), ref.run(cfg)
    assert [b["block_id"] for b in got["blocks"]] == [b["block_id"] for b in want["blocks"]]
    assert [b["noise_ids"] for b in got["blocks"]] == [b["noise_ids"] for b in want["blocks"]]
    assert rel(latents(got), latents(want)) < 1e-12
    assert np.array_equal(got["events"], want["events"])


def test_forward_chunk_cases_f64(bp, ref):
    """test_model.cpp:139-223 cases through bp_forward_chunk vs the reference."""
    cfg = bp.PipelineConfig(layers=2, hidden=8, heads=2, channels=2, height=1, width=1, context_len=3)
    st, rc = bp.Stage(cfg, 17, 0, 2, 19), ref.RefChunk(cfg, 17, 0, 2, 19)
    rng = np.random.default_rng(0)
    prev = rng.standard_normal((2, 2))
    a = st.forward_chunk(prev, [5, 5], [4, 5], capture_frames=[0], mode="on")
    b = rc.forward(prev, [5, 5], [4, 5], capture=[0], mode="on")
    assert rel(a["payload"], b) < 1e-12 and a["captured"] and a["captured_tokens"] == 1
    assert rel(st.cache_rows(0, 1), rc.cache(0, 1)) < 1e-12
    cur = rng.standard_normal((3, 2))
    a2 = st.forward_chunk(cur, [4, 4, 4], [1, 2, 3], mode="on", use_prev=1)
    b2 = rc.forward(cur, [4, 4, 4], [1, 2, 3], mode="on", use_prev=1)
    assert rel(a2["payload"], b2) < 1e-12
    # chunked == monolithic (test_model.cpp:155-176), bitwise on the GPU
    cfg4 = bp.PipelineConfig(layers=4, hidden=8, heads=2, channels=2, height=1, width=1, context_len=3)
    mono, p0, p1 = bp.Stage(cfg4, 9, 0, 4, 13), bp.Stage(cfg4, 9, 0, 2, 13), bp.Stage(cfg4, 9, 2, 4, 13)
    x = rng.standard_normal((3, 2))
    whole = mono.forward_chunk(x, [2, 2, 2], [5, 6, 7])["payload"]
    mid = p0.forward_chunk(x, [2, 2, 2], [5, 6, 7])["payload"]
    last = p1.forward_chunk(mid, [2, 2, 2], [5, 6, 7])["payload"]
    assert np.array_equal(whole, last)
    # cache supplied while caching is disabled (model.cpp:269-271)
    with pytest.raises(bp.CacheError):
        st.forward_chunk(cur, [4, 4, 4], [1, 2, 3], mode="off", use_prev=1)


def test_one_ulp_sensitivity(bp, ref):
    """test_model.cpp:178-223 with its exact inputs (RandomSource(23) draws):
    cached == recompute, and a 1-ulp bump of cached V[0][0] changes the output."""
    from oracle.blockpipe_oracle import RandomSource
    cfg = bp.PipelineConfig(layers=2, hidden=8, heads=2, channels=2, height=1, width=1, context_len=3)
    rs = RandomSource(23)
    prev, cur = rs.normal_tensor((2, 2)), rs.normal_tensor((3, 2))
    st = bp.Stage(cfg, 17, 0, 2, 19)
    st.forward_chunk(prev, [5, 5], [4, 5], capture_frames=[0], mode="on")
    clean = st.forward_chunk(cur, [4, 4, 4], [1, 2, 3], mode="on", use_prev=1)["payload"]
    rc = ref.RefChunk(cfg, 17, 0, 2, 19)
    rc.forward(prev, [5, 5], [4, 5], capture=[0], mode="on")
    assert rel(clean, rc.forward(cur, [4, 4, 4], [1, 2, 3], mode="on", use_prev=1)) < 1e-12
    st.forward_chunk(prev, [5, 5], [4, 5], capture_frames=[0], mode="recompute")
    via_rec = st.forward_chunk(cur, [4, 4, 4], [1, 2, 3], mode="recompute", use_prev=2)["payload"]
    assert np.array_equal(clean, via_rec)
    st.forward_chunk(prev, [5, 5], [4, 5], capture_frames=[0], mode="on")
    st.bump_ulp(0, 1, 0)
    bumped = st.forward_chunk(cur, [4, 4, 4], [1, 2, 3], mode="on", use_prev=1)["payload"]
    assert not np.array_equal(clean, bumped)


def test_scheduler_step_closed_form(bp):  # test_model.cpp:270-298
    rng = np.random.default_rng(71)
    x, eps = rng.standard_normal((2, 3)), rng.standard_normal((2, 3))
    assert np.array_equal(bp.scheduler_step(x, eps, 25, 50), x - 0.02 * eps)
    with pytest.raises(bp.SchedulerError):
        bp.scheduler_step(x, eps, 0, 8)
    with pytest.raises(bp.SchedulerError):
        bp.scheduler_step(x, eps, 9, 8)


def test_pool_720p_bit_exact(bp, ref):
    seed = bp.derive_seed(2, [0])
    assert np.array_equal(bp.build_pool(8, 8, (45, 80, 64), seed), ref.pool(8, 8, (45, 80, 64), seed))


def test_host_supplied_pool(bp):
    """bp_pipeline_set_pool: the reference's own pool handed in from pinned
    host memory gives bitwise the seeded run; a wrong size is a
    DimensionError and a pool with two equal entries fails build_pool's
    collision check (noise.cpp:38-46) with a ConfigError."""
    cfg = bp.PipelineConfig.from_dict(dict(G["mid"]["config"], precision="f64"))
    want = bp.run_pipeline(cfg)
    p = bp.Pipeline(cfg)
    m = cfg.num_b + cfg.num_c // 2
    pool = bp.pinned_empty((m, cfg.height, cfg.width, cfg.channels))
    pool[...] = bp.build_pool(cfg.num_b, cfg.num_c, (cfg.height, cfg.width, cfg.channels),
                              bp.derive_seed(cfg.seed_noise, [0]))
    p.set_pool(pool)
    got = p.run()
    assert all(np.array_equal(x["frames"], y["frames"]) for x, y in zip(got, want["blocks"]))
    st = p.stats()
    assert st["h2d_bytes"] == pool.nbytes
    assert st["d2h_bytes"] == sum(b["frames"].nbytes for b in got)
    with pytest.raises(bp.DimensionError):
        p.set_pool(np.zeros(7))
    dup = pool.copy()
    dup[1] = dup[0]
    p.set_pool(dup)
    with pytest.raises(bp.ConfigError):
        p.run()
    p.set_pool(None)
    again = p.run()
    assert all(np.array_equal(x["frames"], y["frames"]) for x, y in zip(again, want["blocks"]))


def _two_passes(stage_or_ref, is_ref, x0, x1):
    """A capture pass then a prefix pass (the cached-context route)."""
    if is_ref:
        a = stage_or_ref.forward(x0, [7, 7], [0, 1], capture=[1], mode="on")
        b = stage_or_ref.forward(x1, [6, 6], [1, 2], mode="on", use_prev=1)
        return a, b
    a = stage_or_ref.forward_chunk(x0, [7, 7], [0, 1], capture_frames=[1], mode="on")["payload"]
    b = stage_or_ref.forward_chunk(x1, [6, 6], [1, 2], mode="on", use_prev=1)["payload"]
    return a, b


def test_wan13_width_stage_vs_reference(bp, ref):
    """One Wan2.1-1.3B-width layer (h 1536, 12 heads, dh 128, C 64, 4h FFN)
    as a whole chunk (entry embedding + layer + head), a capture pass and a
    cached-prefix pass, through bp_forward_chunk vs the reference library:
    fp64 <= 1e-12, fp32 <= 1e-4, bf16 tensor-core path <= 2e-2."""
    cfg = bp.PipelineConfig(layers=1, hidden=1536, heads=12, channels=64, height=2, width=4, context_len=64)
    rng = np.random.default_rng(3)
    x0, x1 = rng.standard_normal((16, 64)), rng.standard_normal((16, 64))
    want = _two_passes(ref.RefChunk(cfg, 5, 0, 1, 6), True, x0, x1)
    for prec, tol in (("f64", 1e-12), ("f32", 1e-4), ("bf16", 2e-2)):
        got = _two_passes(bp.Stage(cfg, 5, 0, 1, 6, precision=prec), False, x0, x1)
        for g, w_ in zip(got, want):
            assert rel(g, w_) <= tol, (prec, rel(g, w_))


def test_wan14b_width_stage(bp):
    """Wan2.1-14B width (h 5120, 40 heads, FFN 13824) as two chunks of a
    2-layer model: bf16 and fp32 vs the fp64 GPU path (itself pinned to the
    reference at <= 1e-12), chunked == monolithic bitwise in bf16."""
    cfg = bp.PipelineConfig(layers=2, hidden=5120, heads=40, ffn=13824, channels=64, height=2, width=4,
                            context_len=64)
    rng = np.random.default_rng(4)
    x0, x1 = rng.standard_normal((16, 64)), rng.standard_normal((16, 64))
    base = _two_passes(bp.Stage(cfg, 5, 0, 2, 6, precision="f64"), False, x0, x1)
    for prec, tol in (("f32", 1e-4), ("bf16", 2e-2)):
        got = _two_passes(bp.Stage(cfg, 5, 0, 2, 6, precision=prec), False, x0, x1)
        for g, w_ in zip(got, base):
            assert rel(g, w_) <= tol, (prec, rel(g, w_))
    mono = bp.Stage(cfg, 5, 0, 2, 6, precision="bf16").forward_chunk(x0, [7, 7], [0, 1])["payload"]
    mid = bp.Stage(cfg, 5, 0, 1, 6, precision="bf16").forward_chunk(x0, [7, 7], [0, 1])["payload"]
    last = bp.Stage(cfg, 5, 1, 2, 6, precision="bf16").forward_chunk(mid, [7, 7], [0, 1])["payload"]
    assert np.array_equal(mono, last)


def test_wan_size_invariants(bp):
    """Size-independent properties at the production shape (Wan2.1-1.3B width,
    480p latent grid, S = 18720, cached prefix 6240; 2 blocks x 2 steps so
    both prefix and tail passes run): the 2-stage loopback pipeline equals the
    single stage bitwise, cached == recompute bitwise, every latent finite."""
    base = dict(layers=30, hidden=1536, heads=12, ffn=8960, channels=64, height=30, width=52,
                context_len=512, num_b=8, num_c=8, steps=2, blocks=2, precision="bf16")
    one = bp.run_pipeline(dict(base, devices=1))
    two = bp.run_pipeline(dict(base, devices=2))
    rec = bp.run_pipeline(dict(base, devices=1, cache="recompute"))
    a, b, c = latents(one), latents(two), latents(rec)
    assert a.size == (12 + 8) * 30 * 52 * 64
    assert np.isfinite(a).all()
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("strategy", ["coordinated", "complete-shuffle", "subset", "fresh", "repeat"])
def test_noise_draws_vs_reference(bp, ref, strategy):
    """draw_first_block + 6 x draw_next_block (noise.cpp:135-178) through
    bp_noise_draw against the reference's own draws: ids and the append
    stream bit-exact, frames bitwise (stacked pool entries, or fresh normals)."""
    num_b, num_c, shape, seed = 8, 8, (3, 4, 2), 5
    want = ref.noise_walk_frames(strategy, 6, num_b, num_c, shape, seed)
    pool = bp.build_pool(num_b, num_c, shape, seed)
    got = [bp.draw_first_block(strategy, pool, num_b, num_c, bp.derive_seed(seed, [1]))]
    for _ in range(6):
        ids = got[-1]["noise_ids"]
        window = ids[-(num_c // 2):] if len(ids) >= num_c // 2 else []
        got.append(bp.draw_next_block(strategy, pool, num_b, num_c, window, got[-1]["rng_state"]))
    for g, (ids, frames) in zip(got, want):
        assert g["noise_ids"] == ids
        assert np.array_equal(g["frames"], frames)


def test_gather_block_and_window_errors(bp):
    pool = bp.build_pool(4, 4, (2, 3, 2), 9)
    assert np.array_equal(bp.gather_block(pool, [5, 0, 5]), pool[[5, 0, 5]])
    with pytest.raises(bp.QueueError):
        bp.gather_block(pool, [6])
    for bad in ([1, 1], [1], [1, 99]):  # noise.cpp:79-90
        with pytest.raises(bp.QueueError):
            bp.draw_next_block("coordinated", pool, 4, 4, bad, 3)


@pytest.mark.parametrize("prec,tol", [("f64", 1e-12), ("bf16", 2e-2)])
def test_capture_size_change_uses_intact_cache(bp, ref, prec, tol):
    """A pass that consumes a resident 2-frame cache while capturing 4 frames
    (and the pass after it, on that 4-frame cache) over 3 layers: the new
    capture must not overwrite cached K/V of a later layer before that layer
    reads it (the reference keeps the two entries apart, model.cpp:302-324)."""
    cfg = bp.PipelineConfig(layers=3, hidden=128, heads=1, channels=4, height=2, width=4, context_len=8)
    rng = np.random.default_rng(8)
    xs = [rng.standard_normal((6 * 8, 4)) for _ in range(3)]
    lv, ids = [7] * 6, list(range(6))
    st = bp.Stage(cfg, 3, 0, 3, 4, precision=prec)
    rc = ref.RefChunk(cfg, 3, 0, 3, 4)
    st.forward_chunk(xs[0], lv, ids, capture_frames=[0, 1], mode="on")
    rc.forward(xs[0], lv, ids, capture=[0, 1], mode="on")
    a = st.forward_chunk(xs[1], lv, ids, capture_frames=[0, 1, 2, 3], mode="on", use_prev=1)["payload"]
    b = rc.forward(xs[1], lv, ids, capture=[0, 1, 2, 3], mode="on", use_prev=1)
    assert rel(a, b) <= tol
    a = st.forward_chunk(xs[2], lv, ids, mode="on", use_prev=1)["payload"]
    b = rc.forward(xs[2], lv, ids, mode="on", use_prev=1)
    assert rel(a, b) <= tol
