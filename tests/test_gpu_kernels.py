"""Kernel-level parity: tcgen05 GEMM / attention vs numpy and the SIMT check kernels."""
import numpy as np
import pytest

from kernels import DEFAULT_ATTN_IMPL, DEFAULT_GEMM_IMPL, attn, from_bf16_bits, gemm, ref_attn, load_testlib, to_bf16_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib(bp):
    L = load_testlib()
    yield L
    L.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 128), (1000, 1536, 1536), (257, 4608, 256),
                                   (64, 96, 64), (130, 8960, 128)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
@pytest.mark.parametrize("impl", [3])
def test_gemm_tcgen05(lib, M, N, K, epi, impl):
    """The cta_group::2 pair GEMM (one M = 256 MMA per k-step) vs fp64 numpy and the SIMT check kernel."""
    rng = np.random.default_rng(M * 7 + N + K + epi)
    A = to_bf16_bits(rng.standard_normal((M, K)))
    W = to_bf16_bits(rng.standard_normal((N, K)) / np.sqrt(K))
    want = from_bf16_bits(A).astype(np.float64) @ from_bf16_bits(W).astype(np.float64).T
    if epi in (0, 1):
        C0 = np.zeros((M, N), dtype=np.uint16)
    else:
        C0 = rng.standard_normal((M, N)).astype(np.float32)
    lib.bp_set_kernel_impl(impl, DEFAULT_ATTN_IMPL)
    got = gemm(lib, A, W, C0, epi)
    if epi == 1:
        from scipy.special import erf
        want = 0.5 * want * (1 + erf(want / np.sqrt(2)))
    if epi == 2:
        want = want + C0
    g = from_bf16_bits(got).astype(np.float64) if epi in (0, 1) else got.astype(np.float64)
    rel = np.linalg.norm(g - want) / np.linalg.norm(want)
    assert rel < (5e-3 if epi in (0, 1) else 1e-5), rel
    lib.bp_set_kernel_impl(0, DEFAULT_ATTN_IMPL)
    chk = gemm(lib, A, W, C0, epi)
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)
    c = from_bf16_bits(chk).astype(np.float64) if epi in (0, 1) else chk.astype(np.float64)
    assert np.linalg.norm(g - c) / np.linalg.norm(c) < (5e-3 if epi in (0, 1) else 1e-5)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 128), (1000, 1536, 1536), (64, 96, 64),
                                   (257, 1536, 8960)])
@pytest.mark.parametrize("impl", [3, 0])
def test_gemm_residual_out_equals_residual(lib, M, N, K, impl):
    """The fused-send epilogue (kGemmResidualOutF32: out = R + acc into a
    separate buffer, the next rank's receive slot) equals the in-place TMA
    reduce-add epilogue (x += acc) bitwise, so a fused send cannot change
    the latents."""
    rng = np.random.default_rng(M + N + K)
    A = to_bf16_bits(rng.standard_normal((M, K)))
    W = to_bf16_bits(rng.standard_normal((N, K)) / np.sqrt(K))
    C0 = rng.standard_normal((M, N)).astype(np.float32)
    lib.bp_set_kernel_impl(impl, DEFAULT_ATTN_IMPL)
    inplace = gemm(lib, A, W, C0, 2)
    out = gemm(lib, A, W, C0, 6)
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)
    assert np.array_equal(inplace, out)


@pytest.mark.parametrize("impl", [3])
def test_gemm_row_position_invariance(lib, impl):
    """A row's result does not depend on its M position (cached == recompute),
    nor on which GEMM implementation or cluster CTA computed it."""
    lib.bp_set_kernel_impl(impl, DEFAULT_ATTN_IMPL)
    rng = np.random.default_rng(5)
    A = to_bf16_bits(rng.standard_normal((700, 384)))
    W = to_bf16_bits(rng.standard_normal((768, 384)) / 20)
    full = gemm(lib, A, W, np.zeros((700, 768), dtype=np.uint16), 0)
    part = gemm(lib, np.ascontiguousarray(A[333:333 + 97]), W, np.zeros((97, 768), dtype=np.uint16), 0)
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)
    assert np.array_equal(full[333:333 + 97], part)


def test_gemm_bench(lib):
    ms = __import__("ctypes").c_double()
    for (M, N, K) in [(18720, 4608, 1536), (18720, 8960, 1536), (18720, 1536, 8960)]:
        assert lib.bp_bench_gemm(0, M, N, K, 0, 10, ms) == 0
        tf = 2 * M * N * K / (ms.value * 1e-3) / 1e12
        print(f"gemm {M}x{N}x{K}: {ms.value:.3f} ms  {tf:.0f} TFLOP/s")


@pytest.mark.parametrize("impl", [2, 4])
@pytest.mark.parametrize("rows,n0,n1,heads", [(128, 0, 128, 1), (300, 0, 300, 2), (300, 200, 300, 2),
                                              (511, 0, 512, 3), (513, 0, 512, 2), (1300, 0, 512, 5),
                                              (257, 256, 129, 2), (96, 0, 512, 3), (1000, 640, 1000, 1),
                                              (513, 65, 63, 2), (256, 0, 1, 1), (40, 7, 100, 2),
                                              (512, 0, 1024, 2), (256, 512, 1024, 1), (300, 0, 512, 1)])
def test_attention_tcgen05(lib, rows, n0, n1, heads, impl):
    """impl 2: the persistent single-CTA ping-pong over (query pair, head) items,
    64-key tiles (the cross-attention kernel, k_attn_ps); impl 4: the
    ping-pong on a cta_group::2 CTA pair, one query pair per CTA (the
    self-attention kernel, k_attn_pp2)."""
    dh = 128
    rng = np.random.default_rng(rows + n0 * 3 + n1 + heads)
    H = heads * dh
    q = to_bf16_bits(rng.standard_normal((rows, H)))
    k1 = to_bf16_bits(rng.standard_normal((n1, H)))
    v1 = to_bf16_bits(rng.standard_normal((n1, H)))
    k0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
    v0 = to_bf16_bits(rng.standard_normal((n0, H))) if n0 else None
    scale = 1 / np.sqrt(dh)
    kk = from_bf16_bits(np.concatenate([k0, k1]) if n0 else k1)
    vv = from_bf16_bits(np.concatenate([v0, v1]) if n0 else v1)
    want = ref_attn(from_bf16_bits(q), kk, vv, heads, dh, scale)
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, impl)
    try:
        got = from_bf16_bits(attn(lib, q, k0, v0, k1, v1, heads, dh, scale)).astype(np.float64)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 1e-2, rel
        lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, 0)
        chk = from_bf16_bits(attn(lib, q, k0, v0, k1, v1, heads, dh, scale)).astype(np.float64)
        assert np.linalg.norm(chk - want) / np.linalg.norm(want) < 1e-2
    finally:
        lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)


def test_attention_bench(lib):
    ms = __import__("ctypes").c_double()
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, DEFAULT_ATTN_IMPL)
    for (rows, n0, n1) in [(18720, 6240, 18720), (18720, 0, 512)]:
        assert lib.bp_bench_attn(0, rows, 12, 128, n0, n1, 5, ms) == 0, lib.bp_last_error()
        tf = 4 * rows * (n0 + n1) * 12 * 128 / (ms.value * 1e-3) / 1e12
        print(f"attn q={rows} kv={n0}+{n1}: {ms.value:.3f} ms  {tf:.0f} TFLOP/s")


def test_attention_boundary_sweep(lib):
    """Tile-boundary sweep of the default kernels: rows around the 128-row
    query tile and the 256-row CTA pair, both key segments around the 64-key
    tile (self-attention, k_attn_pp2), and the key count alone for the
    cross-attention launcher (k_attn_ps)."""
    from kernels import attn_cross
    dh, heads = 128, 1
    edges = (63, 64, 65, 127, 128, 129)
    worst = 0.0
    for rows in (127, 128, 129, 255, 256, 257):
        rng = np.random.default_rng(rows)
        q = to_bf16_bits(rng.standard_normal((rows, dh)))
        kk = to_bf16_bits(rng.standard_normal((260, dh)))
        vv = to_bf16_bits(rng.standard_normal((260, dh)))
        for n0 in edges:
            for n1 in edges:
                k0, v0 = np.ascontiguousarray(kk[:n0]), np.ascontiguousarray(vv[:n0])
                k1, v1 = np.ascontiguousarray(kk[130:130 + n1]), np.ascontiguousarray(vv[130:130 + n1])
                got = from_bf16_bits(attn(lib, q, k0, v0, k1, v1, heads, dh, 1 / np.sqrt(dh))).astype(np.float64)
                want = ref_attn(from_bf16_bits(q), from_bf16_bits(np.concatenate([k0, k1])),
                                from_bf16_bits(np.concatenate([v0, v1])), heads, dh, 1 / np.sqrt(dh))
                r = np.linalg.norm(got - want) / np.linalg.norm(want)
                worst = max(worst, r)
                assert r < 1e-2, (rows, n0, n1, r)
        for n1 in edges:
            k1, v1 = np.ascontiguousarray(kk[:n1]), np.ascontiguousarray(vv[:n1])
            got = from_bf16_bits(attn_cross(lib, q, k1, v1, heads, dh, 1 / np.sqrt(dh))).astype(np.float64)
            want = ref_attn(from_bf16_bits(q), from_bf16_bits(k1), from_bf16_bits(v1), heads, dh, 1 / np.sqrt(dh))
            r = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert r < 1e-2, (rows, n1, r)
    print("worst rel-L2", worst)
