"""Host schedule (C-ABI, no GPU): event log, ledger, queue snapshots, noise
ids and bubbles must be bit-identical to the reference's run_pipeline, and
the reference's own schedule assertions (test_engine.cpp) must hold."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "goldens.json")))

CONFIGS = [dict(devices=1), dict(devices=2), dict(devices=4, steps=6, blocks=5), dict(devices=2, order="sequential"),
           dict(devices=2, cache="off"), dict(devices=2, cache="recompute"), dict(devices=2, strategy="fresh"),
           dict(devices=2, strategy="repeat"), dict(devices=2, strategy="subset"),
           dict(devices=2, strategy="complete-shuffle"), dict(devices=2, retain_clean_context=False),
           dict(devices=2, num_c=0), dict(devices=4, steps=6, blocks=2), dict(devices=1, steps=1, blocks=3),
           dict(devices=4, layers=8, steps=50, blocks=4), dict(devices=2, num_b=3, num_c=6, steps=5, blocks=7)]


def tiny(**kw):
    d = dict(layers=4, hidden=8, heads=2, channels=1, height=1, width=1, context_len=2, num_b=1, num_c=2, mode="single")
    d.update(kw)
    return d


@pytest.mark.parametrize("c", CONFIGS)
def test_schedule_equals_reference(bp, ref, c):
    cfg = bp.PipelineConfig.from_dict(dict(c, mode="single"))
    r = ref.run(cfg)
    s = bp.Schedule(cfg)
    assert np.array_equal(r["events"], s.events)
    assert r["ledger"] == s.ledger
    assert r["queue_snapshots"] == s.snapshots
    assert [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in r["blocks"]] == \
        [(b["block_id"], b["noise_ids"], b["frame_ids"]) for b in s.blocks]
    assert r["bubbles"] == bp.measure_bubbles(s.events, cfg.devices)
    assert r["rounds"] == s.rounds


@pytest.mark.parametrize("name", ["cfg1", "mid"])
def test_schedule_goldens(bp, name):
    s = bp.Schedule(G[name]["config"])
    assert np.array_equal(np.load(os.path.join(ROOT, "tests", "golden", f"{name}_latents.npz"))["events"], s.events)
    assert s.ledger == G[name]["ledger"]
    assert s.snapshots == G[name]["snapshots"]
    assert [b["noise_ids"] for b in s.blocks] == [b["noise_ids"] for b in G[name]["blocks"]]


def test_single_device_busy(bp):  # test_engine.cpp:53-64
    st = bp.measure_bubbles(bp.Schedule(dict(devices=1, layers=4, hidden=8, heads=2, steps=4, blocks=4)).events, 1)
    assert st["idle_per_device"] == 0 and st["ratio"] == 0.0 and st["busy_per_device"] == 16


def test_malformed_event_logs(bp):
    """measure_bubbles' validation (engine.cpp:508-530): a duplicated slot on
    one device, a device index out of range, unequal pass counts."""
    ev = bp.Schedule(tiny(devices=2, steps=4, blocks=3)).events.copy()
    firsts = [np.flatnonzero(ev[:, 1] == d)[0] for d in range(2)]
    dup = np.concatenate([ev, ev[firsts]])  # every device sees its first slot twice
    with pytest.raises(bp.SchedulingError, match="duplicate slot on one device"):
        bp.measure_bubbles(dup, 2)
    bad = ev.copy()
    bad[0, 1] = 5
    with pytest.raises(bp.SchedulingError, match="device out of range"):
        bp.measure_bubbles(bad, 2)
    with pytest.raises(bp.SchedulingError, match="different pass counts"):
        bp.measure_bubbles(ev[1:], 2)


def test_bubble_formula_proximity(bp):  # test_engine.cpp:152-173
    for n, steps, blocks in [(2, 8, 6), (4, 10, 8), (4, 50, 4)]:
        s = bp.Schedule(tiny(devices=n, steps=steps, blocks=blocks))
        st = bp.measure_bubbles(s.events, n)
        assert st["busy_per_device"] == steps * blocks
        assert st["steady_idle"] == 0
        assert st["warmup_idle"] + st["steady_idle"] + st["cooldown_idle"] == st["idle_per_device"] * n
        assert abs(st["idle_per_device"] - (n * n - n - 1)) <= n
    st = bp.measure_bubbles(bp.Schedule(tiny(devices=4, steps=50, blocks=4)).events, 4)
    assert abs(st["ratio"] - 11 / 211) <= 0.02


def test_precedence(bp):  # test_engine.cpp:175-188
    s = bp.Schedule(tiny(devices=4, steps=6, blocks=5))
    by = {}
    for slot, dev, blk, lvl, ph, rnd in s.events.tolist():
        by.setdefault((blk, rnd), {})[dev] = slot
    for d in by.values():
        assert [d[j] for j in range(4)] == sorted(d[j] for j in range(4))
        assert all(d[j] > d[j - 1] for j in range(1, 4))


def test_ledger_rows(bp):  # test_engine.cpp:190-210
    s = bp.Schedule(dict(devices=4, layers=4, hidden=8, heads=2, channels=2, height=2, width=2, num_b=2, num_c=4,
                         steps=6, blocks=6))
    rows = (2 + 2) * 4
    for e in s.ledger:
        if e["channel"] in ("host->dev0", "dev3->host"):
            assert e["scalars"] == e["passes"] * rows * 2
        if e["channel"] == "dev1->dev2":
            assert e["scalars"] == e["passes"] * rows * 8


def test_wan_schedule_shapes(bp):
    """cfg 2/3/4 pass counts and the N(N-1) idle law."""
    for blocks, passes, rounds in [(3, 150, 52), (9, 450, 58), (32, 1600, 81)]:
        s = bp.Schedule(tiny(devices=1, layers=30, steps=50, blocks=blocks, num_b=8, num_c=8))
        assert (s.npasses, s.rounds) == (passes, rounds)
    for n, makespan in [(2, 452), (4, 462), (8, 506)]:
        s = bp.Schedule(tiny(devices=n, layers=8, steps=50, blocks=9))
        assert s.events[:, 0].max() - s.events[:, 0].min() + 1 == makespan


def test_coordinated_windows_disjoint(bp):  # test_smoke.py:61-67, test_noise.cpp:108-121
    ids = bp.coordinated_noise_ids(8, 8, 50)
    assert sorted(ids[0]) == list(range(12))
    for prev, nxt in zip(ids, ids[1:]):
        window = set(prev[-4:])
        assert window.isdisjoint(nxt) and window | set(nxt) == set(range(12))


def test_uneven_split(bp):
    s = bp.Schedule(dict(tiny(devices=8, layers=30), uneven_split=True))
    assert s.partition == [(0, 4), (4, 8), (8, 12), (12, 16), (16, 20), (20, 24), (24, 27), (27, 30)]
    with pytest.raises(bp.ConfigError):
        bp.Schedule(tiny(devices=8, layers=30))


@pytest.mark.parametrize("bad,err", [(dict(devices=3), "ConfigError"), (dict(num_c=3), "ConfigError"),
                                     (dict(num_c=6, num_b=2), "ConfigError"), (dict(heads=3), "ConfigError"),
                                     (dict(steps=0), "ConfigError"), (dict(blocks=0), "ConfigError")])
def test_invalid_configs(bp, bad, err):  # test_engine.cpp:257-266
    base = dict(devices=2, layers=4, hidden=8, heads=2, num_b=2, num_c=4, steps=4, blocks=4)
    base.update(bad)
    with pytest.raises(getattr(bp, err)):
        bp.Schedule(base)


def test_unknown_key(bp):
    with pytest.raises(bp.ConfigError):
        bp.PipelineConfig.from_dict({"nope": 1})
