"""The reference's release gates (P/tests/acceptance.cpp)
that need no GPU, run against this repo's host side: the analytics, the
static schedule and the coordinated noise ids. Gates 4 and 5 (pipeline ==
serial oracle across the grid, cache == recompute, fault detection) run on
the GPU in test_gpu_acceptance.py; gate 9 (byte-identical artifacts, engines
agree) in test_gpu_operator.py."""
from fractions import Fraction

import pytest


@pytest.fixture(scope="module")
def op():
    from paper_2505_21070_b200 import operator
    return operator


def schedule_cfg(devices, steps, blocks):
    """acceptance.cpp:59-76."""
    return dict(devices=devices, layers=4, hidden=8, heads=2, channels=1, height=1, width=1, context_len=2,
                num_b=1, num_c=2, steps=steps, blocks=blocks, mode="single")


def test_gate1_bubble_formula_11_of_211(op):
    assert op.bubble_size(4, 50, 4) == 11
    assert abs(op.bubble_ratio(4, 50, 4) - 11 / 211) <= 5e-4


def test_gate2_regimes_exact_and_reverse_below_sequential(op):
    def exact(size, t, blocks):
        return size / (size + Fraction(t) * blocks)
    size = Fraction(3) * (4 - 50) + Fraction(4) * (50 - 2) + 1
    assert size == 55 and exact(size, 50, 3) == Fraction(55, 205)
    assert abs(op.bubble_ratio(4, 50, 3) - float(Fraction(55, 205))) <= 1e-15
    size = Fraction(4) * 4 - 1
    assert exact(size, 50, 4) == Fraction(15, 215)
    assert abs(op.bubble_ratio(4, 50, 4, "sequential") - float(Fraction(15, 215))) <= 1e-15
    points = 0
    for n in range(2, 9):
        for t in (4, 10, 50):
            for b in range(n, 3 * n + 1):
                assert op.bubble_ratio(n, t, b) < op.bubble_ratio(n, t, b, "sequential"), (n, t, b)
                points += 1
    assert points == sum(3 * (2 * n + 1) for n in range(2, 9))


def test_gate3_measured_schedules(bp, op):
    """Busy slots exact (T * blocks), zero steady idle, idle within N of the
    formula, over N {1, 2, 4} x T {4, 10, 50} x blocks {4, 9, 16}."""
    for n in (1, 2, 4):
        for t in (4, 10, 50):
            for blocks in (4, 9, 16):
                s = bp.Schedule(schedule_cfg(n, t, blocks))
                st = bp.measure_bubbles(s.events, n)
                tag = (n, t, blocks)
                assert st["busy_per_device"] == t * blocks, tag
                assert st["steady_idle"] == 0, tag
                assert abs(st["idle_per_device"] - op.bubble_size(n, t, blocks)) <= n, tag


def test_gate6_coordinated_noise_over_1000_appends(bp):
    """Every coordinated append is disjoint from the previous block's tail
    window and, with it, covers the whole pool (num_b = num_c = 8: M = 12)."""
    num_b, num_c = 8, 8
    ids = bp.coordinated_noise_ids(num_b, num_c, 1000, seed=42)
    assert len(ids) == 1001
    assert sorted(ids[0]) == list(range(num_b + num_c // 2))  # the first block is a full permutation
    for i in range(1, len(ids)):
        window = ids[i - 1][-(num_c // 2):]
        seen = set(window)
        for k in ids[i]:
            assert k not in seen, f"id overlap at append {i}"
            seen.add(k)
        assert len(seen) == num_b + num_c // 2, f"coverage hole at append {i}"


def test_gate6_repeat_strategy_always_overlaps(bp):
    num_b, num_c = 8, 8
    s = bp.Schedule(dict(num_b=num_b, num_c=num_c, steps=1, blocks=1001, devices=1, layers=1, hidden=2, heads=1,
                         channels=1, height=1, width=1, strategy="repeat", seed_noise=9))
    ids = [b["noise_ids"] for b in s.blocks]
    for i in range(1, len(ids)):
        window = ids[i - 1][-(num_c // 2):]
        assert any(k in window for k in ids[i]), f"repeat strategy shows no overlap at append {i}"


def test_gate7_cost_model_relationships(op):
    cp = dict(num_b=8, num_c=8, height=4, width=4, hidden=8, devices=4, model_mem=12.0)
    dual = op.method_cost("dualparal", **cp)
    assert dual["model_mem"] == cp["model_mem"] / cp["devices"]
    assert dual["comm_scalars"] == 2.0 * (8 + 4) * 4 * 4 * 8
    frames = 64
    for m in ("dualparal", "fifo"):  # constant in the video length
        assert (op.method_cost(m, **cp, frames=2 * frames)["kv_mem"] ==
                op.method_cost(m, **cp, frames=frames)["kv_mem"]), m
    for m in ("ring-attention", "ulysses", "video-infinity"):
        assert (op.method_cost(m, **cp, frames=2 * frames)["kv_mem"] >
                op.method_cost(m, **cp, frames=frames)["kv_mem"]), m
    assert (op.method_cost("ulysses", **dict(cp, devices=4))["comm_scalars"] ==
            op.method_cost("ulysses", **dict(cp, devices=2))["comm_scalars"] / 2.0)


def test_gate8_bubble_ratio_vanishes_for_long_generations(op):
    assert op.bubble_ratio(8, 50, 1000000) < 1e-4
