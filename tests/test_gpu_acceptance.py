"""The reference's release gates 4 and 5 (P/tests/acceptance.cpp:177-228,
SPEC.md:518-528) on the GPU engine.

Gate 4 runs over the same grid: layers {4, 8} x steps {4, 8} x blocks {4, 6}
x cache {on, off}, at math_cfg's shape (h 16, 2 heads, C 2, 2 x 2 latent
grid, Lc 4, num_b 2, num_c 4), for N in {1, 2, 4}. For every cell:
  * the GPU pipeline equals the GPU serial path bitwise, as the reference
    requires of itself, in the fp64 parity and fp32 verification modes (at
    h 16 the tcgen05 bf16 path does not apply; its N-invariance is tested at
    the mid shape in test_gpu_parity.py);
  * the fp64 (fp32) latents are within 1e-12 (1e-4) rel-L2 of the reference library's
    serial_oracle (oracle/_ref, the unmodified reference compiled from its
    sources);
  * the events (slot, device, block, level, phase, round) of every N, the
    noise ids and the frame ids match the reference's run_pipeline exactly.
Gate 5: the feature cache equals explicit recompute bitwise, on the latents
and on every pass's eps, and a 1-ulp cache fault is detected (CacheError)."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRID = list(itertools.product([4, 8], [4, 8], [4, 6], ["on", "off"]))


def math_cfg(devices, layers, steps, blocks, **kw):
    return dict(dict(devices=devices, layers=layers, hidden=16, heads=2, channels=2, height=2, width=2,
                     context_len=4, num_b=2, num_c=4, steps=steps, blocks=blocks, mode="single"), **kw)


def latents(out):
    return np.concatenate([b["frames"].ravel() for b in out["blocks"]])


@pytest.mark.parametrize("layers,steps,blocks,cache", GRID)
def test_gate4_pipeline_equals_serial_oracle(bp, ref, layers, steps, blocks, cache):
    base = math_cfg(1, layers, steps, blocks, cache=cache)
    want = ref.run(bp.PipelineConfig.from_dict(base), serial=True)
    w = latents(want)
    ref_events = {n: ref.run(bp.PipelineConfig.from_dict(dict(base, devices=n)))["events"] for n in (1, 2, 4)}
    for prec in ("f64", "f32"):
        serial = bp.serial_oracle(dict(base, precision=prec))
        s = latents(serial)
        for n in (1, 2, 4):
            got = bp.run_pipeline(dict(base, devices=n, precision=prec))
            g = latents(got)
            assert np.array_equal(g, s), f"{prec} N={n} L={layers} T={steps} B={blocks} cache={cache}"
            assert [b["noise_ids"] for b in got["blocks"]] == [b["noise_ids"] for b in want["blocks"]]
            assert [b["frame_ids"] for b in got["blocks"]] == [b["frame_ids"] for b in want["blocks"]]
            assert np.array_equal(got["events"], ref_events[n])
        tol = 1e-12 if prec == "f64" else 1e-4
        r = float(np.linalg.norm(s - w) / np.linalg.norm(w))
        assert r <= tol, f"{prec} serial vs reference serial_oracle: {r}"


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_gate5_cache_equals_recompute_and_fault_detected(bp, prec):
    base = math_cfg(2, 4, 6, 5, precision=prec, record_trace=True)
    c = bp.run_pipeline(dict(base, cache="on"))
    r = bp.run_pipeline(dict(base, cache="recompute"))
    assert np.array_equal(latents(c), latents(r))
    assert len(c["trace"]) == len(r["trace"]) > 0
    assert all(np.array_equal(a["eps"], b["eps"]) for a, b in zip(c["trace"], r["trace"]))
    with pytest.raises(bp.CacheError):
        bp.run_pipeline(dict(base, cache="on", fault_inject=True, check_cache=True))
