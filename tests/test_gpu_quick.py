"""First GPU parity checks (bit-exact noise, fp64 forward, pipeline)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_normals_bit_exact(bp, ref):
    seed = bp.derive_seed(2, [0])
    got = bp.normals(seed, 200000, 0.7)
    want = ref.normals(seed, 200000, 0.7)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_pool_480p_bit_exact(bp, ref):
    """The 480p noise pool (num_b = num_c = 8) is bit-identical to the
    reference's build_pool; its byte-wise FNV-1a-64 is pinned in goldens.json."""
    seed = bp.derive_seed(2, [0])
    pool = bp.build_pool(8, 8, (30, 52, 64), seed)
    want = ref.pool(8, 8, (30, 52, 64), seed)
    assert np.array_equal(pool.view(np.uint64), want.view(np.uint64))
    assert ref.fnv1a64([pool]) == "507c6ce247b45327"


def test_tiny_pipeline_f64(bp, ref):
    cfg = bp.PipelineConfig.from_dict({"devices": 1, "layers": 2, "hidden": 128, "heads": 4,
                                       "steps": 10, "blocks": 4, "mode": "single"})
    got = bp.run_pipeline(cfg)
    want = ref.run(cfg)
    g = np.concatenate([b["frames"].ravel() for b in got["blocks"]])
    w = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    rel = np.linalg.norm(g - w) / np.linalg.norm(w)
    print("rel", rel)
    assert rel <= 1e-12
