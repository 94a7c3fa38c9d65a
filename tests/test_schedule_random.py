"""Randomised sweep of the host schedule against the reference library
(oracle/_ref, no GPU): for seeded random configurations over every knob of
run_pipeline (engine.cpp:255-497) -- devices, layers, num_b / num_c,
steps, blocks, order, cache mode, noise strategy, retain_clean_context,
seeds -- the event log, ledger, queue snapshots, per-block noise / frame
ids, rounds and bubbles of bp.Schedule must equal the reference's run, and a
configuration the reference rejects must be rejected by the mirror with the
same error class (errors.hpp:11-41). Model widths are tiny: the schedule is
data-independent, so they only bound the reference's run time."""
import numpy as np
import pytest

N_CONFIGS = 150


def random_configs(n, seed=20505):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        devices = int(rng.integers(1, 9))
        num_b = int(rng.integers(1, 6))
        num_c = 2 * int(rng.integers(0, num_b + 1))
        layers = devices * int(rng.integers(1, 4))
        if rng.random() < 0.15:  # about one in seven is invalid somewhere: error parity
            which = int(rng.integers(0, 4))
            num_b = 0 if which == 0 else num_b
            num_c = num_c + 1 if which == 1 else (2 * num_b + 2 if which == 2 else num_c)
            layers = layers + 1 if which == 3 and devices > 1 else layers
        c = dict(devices=devices, layers=layers, hidden=8, heads=2, channels=1, height=1, width=1, context_len=2,
                 num_b=num_b, num_c=num_c, steps=int(rng.integers(1, 9)),
                 blocks=int(rng.integers(1, 8)), order=str(rng.choice(["reverse", "sequential"])),
                 cache=str(rng.choice(["on", "off", "recompute"])),
                 strategy=str(rng.choice(["coordinated", "complete-shuffle", "subset", "fresh", "repeat"])),
                 retain_clean_context=bool(rng.integers(0, 2)), seed_noise=int(rng.integers(0, 1 << 30)),
                 mode="single")
        out.append(c)
    return out


@pytest.mark.parametrize("i,c", list(enumerate(random_configs(N_CONFIGS))))
def test_random_schedule_equals_reference(bp, ref, i, c):
    try:
        r = ref.run(bp.PipelineConfig.from_dict(c)) if _valid_for_mirror(bp, c) else None
    except ref.RefError as e:
        with pytest.raises(getattr(bp.errors, e.kind, bp.errors.BlockpipeError)):
            bp.Schedule(bp.PipelineConfig.from_dict(c))
        return
    if r is None:  # the mirror's own config validation rejected it: the reference must too
        with pytest.raises(ref.RefError):
            ref.run(_raw_cfg(bp, c))
        return
    cfg = bp.PipelineConfig.from_dict(c)
    s = bp.Schedule(cfg)
    assert np.array_equal(r["events"], s.events)
    assert r["ledger"] == s.ledger
    assert r["queue_snapshots"] == s.snapshots
    assert [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in r["blocks"]] == \
        [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in s.blocks]
    assert r["bubbles"] == bp.measure_bubbles(s.events, cfg.devices)
    assert r["rounds"] == s.rounds


def _valid_for_mirror(bp, c):
    try:
        bp.PipelineConfig.from_dict(c)
        return True
    except bp.errors.BlockpipeError:
        return False


def _raw_cfg(bp, c):
    """The same fields without the mirror's validation (for the reference)."""
    cfg = bp.PipelineConfig()
    for k, v in c.items():
        if k != "mode":
            setattr(cfg, k, v)
    return cfg
