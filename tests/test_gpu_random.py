"""Randomised GPU sweep against the reference library: seeded random small
configurations over devices, layers, widths (hidden, heads, channels, latent
grid, context length), num_b / num_c, steps, blocks, order, cache mode,
noise strategy and seeds, run through the GPU engine (bp.run_pipeline, the
C-ABI) in the fp64 parity mode and the fp32 verification mode, compared with
the reference's run_pipeline (oracle/_ref): latents within north_star's
tolerance (fp64 <= 1e-12, fp32 <= 1e-4 rel-L2), events and noise / frame ids
exact. A bf16 subset at head dim 128 (the tensor-core path) is held to 2e-2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def latents(out):
    return np.concatenate([b["frames"].ravel() for b in out["blocks"]])


def random_configs(n, seed=7021, bf16=False):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        devices = int(rng.integers(1, 5))
        num_b = int(rng.integers(1, 4))
        heads = int(rng.choice([1, 2, 4]))
        dh = 128 if bf16 else int(rng.choice([4, 8, 16]))
        c = dict(devices=devices, layers=devices * int(rng.integers(1, 3)), hidden=heads * dh, heads=heads,
                 channels=int(rng.choice([1, 2, 4, 16])), height=int(rng.integers(1, 4)), width=int(rng.integers(1, 5)),
                 context_len=int(rng.integers(1, 9)), num_b=num_b, num_c=2 * int(rng.integers(0, num_b + 1)),
                 steps=int(rng.integers(1, 6)), blocks=int(rng.integers(1, 5)),
                 order=str(rng.choice(["reverse", "sequential"])), cache=str(rng.choice(["on", "off", "recompute"])),
                 strategy=str(rng.choice(["coordinated", "complete-shuffle", "subset", "fresh", "repeat"])),
                 retain_clean_context=bool(rng.integers(0, 2)), seed_model=int(rng.integers(0, 1 << 20)),
                 seed_noise=int(rng.integers(0, 1 << 20)), seed_context=int(rng.integers(0, 1 << 20)), mode="single")
        out.append(c)
    return out


def check(bp, ref, c, prec, tol):
    cfg = bp.PipelineConfig.from_dict(dict(c, precision=prec))
    want = ref.run(cfg)
    got = bp.run_pipeline(cfg)
    assert np.array_equal(got["events"], want["events"])
    assert [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in got["blocks"]] == \
        [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in want["blocks"]]
    w = latents(want)
    r = float(np.linalg.norm(latents(got) - w) / np.linalg.norm(w))
    assert r <= tol, (c, prec, r)


@pytest.mark.parametrize("i,c", list(enumerate(random_configs(24))))
def test_random_pipeline_f64_f32(bp, ref, i, c):
    check(bp, ref, c, "f64", 1e-12)
    check(bp, ref, c, "f32", 1e-4)


@pytest.mark.parametrize("i,c", list(enumerate(random_configs(6, seed=9113, bf16=True))))
def test_random_pipeline_bf16(bp, ref, i, c):
    check(bp, ref, c, "bf16", 2e-2)
