"""bench.py's FLOP accounting against SURVEY section 8(d)'s figures (the
roofline numerators of the bench line), from the static schedule on the
host: 1.347e14 per prefix pass at the 1.3B shape; 1.909e16 / 5.937e16 /
2.138e17 per 81- / 301- / 1025-frame video; 3.089e15 per 14B pass."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def bench():
    import bench as b
    return b


def schedule(bp, w):
    return bp.Schedule(bp.PipelineConfig(devices=1, layers=w["layers"], hidden=w["hidden"], heads=w["heads"],
                                         ffn=w["ffn"], channels=w["channels"], height=w["height"],
                                         width=w["width"], context_len=w["context_len"], num_b=w["num_b"],
                                         num_c=w["num_c"], steps=w["steps"], blocks=w["blocks"]))


def test_pass_flops_matches_survey(bench):
    w = bench.WORKLOADS["wan13-301"]
    tpf = w["height"] * w["width"]
    assert bench.pass_flops(w, 12 * tpf, 4 * tpf) == pytest.approx(1.347e14, rel=1e-3)
    w14 = bench.WAN14
    tpf14 = w14["height"] * w14["width"]
    assert bench.pass_flops(w14, 12 * tpf14, 4 * tpf14) == pytest.approx(3.089e15, rel=1e-3)


@pytest.mark.parametrize("name,want", [("wan13-81", 1.909e16), ("wan13-301", 5.937e16), ("wan13-1025", 2.138e17)])
def test_video_flops_matches_survey(bp, bench, name, want):
    w = bench.WORKLOADS[name]
    s = schedule(bp, w)
    flops, n_prefix = bench.video_flops(w, s)
    assert n_prefix == s.npasses - (w["steps"] + w["blocks"] - 1)
    assert flops == pytest.approx(want, rel=1e-3)
    # the self-attention numerator of roofline.achieved is the Skv part of it
    attn = bench.self_attn_flops(w, s)
    assert 0.6 < attn / flops < 0.7
