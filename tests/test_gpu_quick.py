"""First GPU parity checks (bit-exact noise, fp64 forward, pipeline)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_normals_bit_exact(bp, ref):
    seed = bp.derive_seed(2, [0])
    got = bp.normals(seed, 200000, 0.7)
    want = ref.normals(seed, 200000, 0.7)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_pool_480p_fnv(bp, ref):
    pool = bp.build_pool(8, 8, (30, 52, 64), bp.derive_seed(2, [0]))
    assert ref.fnv1a64([pool]) == "d291ee90c83b2769"


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
