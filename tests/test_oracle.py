"""The oracle is pinned before it is trusted: the glibc log/cos port, the C
RNG restatement and the numpy restatement all against goldens generated from
the unmodified reference (tests/golden/make_goldens.py)."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import blockpipe_oracle as bo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "goldens.json")))


def test_glibc_port_bit_exact_on_host(tmp_path):
    """The device noise kernel's log/cos (paper_2505_21070_b200/csrc/glibc_port.h)
    compiled for the host equals this image's glibc on 2M Box-Muller draws."""
    exe = tmp_path / "chk"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2505_21070_b200", "csrc"),
                    os.path.join(ROOT, "tools", "check_glibc_port.c"), "-lm", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "2000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "bad_log=0 bad_cos=0 bad_boxmuller=0" in out.stdout


def test_rng_restatement_goldens():
    rs = bo.RandomSource(1)
    assert [rs.next_normal() for _ in range(3)] == G["rng"]["normals_seed1"]
    for k, v in G["rng"]["derive"].items():
        base, tags = k.split(",", 1)
        assert bo.derive_seed(int(base), json.loads(tags)) == v
    # SURVEY Appendix A known answers
    assert [hex(bo.RandomSource(1).next_u64())] == ["0x910a2dec89025cc1"]
    assert bo.derive_seed(2, [0]) == 0xBFC846100BFC1E42 and bo.derive_seed(2, [1]) == 0xD0D5127A96E8D90D


def test_pool_restatement_fnv():
    from oracle.ref import fnv1a64
    seed = bo.derive_seed(2, [0])
    for tag in ("tiny", "480p"):
        shape = G["pools"][tag]["shape"]
        pool = bo.RandomSource(seed).normal_tensor((12, *shape))
        assert fnv1a64([pool]) == G["pools"][tag]["fnv"]
    assert G["pools"]["480p"]["fnv"] == "507c6ce247b45327"


def test_coordinated_ids_goldens():
    assert G["coordinated_ids"][0] == [2, 9, 10, 4, 6, 5, 0, 11, 1, 3, 8, 7]
    assert G["coordinated_ids"][1] == [0, 4, 6, 10, 9, 2, 5, 11]


@pytest.mark.parametrize("name", ["cfg1", "cfg1_nocache", "mid"])
def test_numpy_restatement_matches_reference_latents(name):
    d = dict(G[name]["config"])
    cfg = {"layers": 4, "hidden": 16, "heads": 2, "channels": 2, "height": 2, "width": 2, "context_len": 4,
           "num_b": 2, "num_c": 4, "steps": 8, "blocks": 6}
    cfg.update({k: v for k, v in d.items() if k not in ("devices", "mode")})
    r = bo.run_pipeline(cfg)
    lat = np.concatenate([b["frames"].ravel() for b in r["blocks"]])
    want = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_latents.npz"))["latents"]
    assert np.linalg.norm(lat - want) / np.linalg.norm(want) < 1e-12
    assert [b["noise_ids"] for b in r["blocks"]] == [b["noise_ids"] for b in G[name]["blocks"]]
    if name == "cfg1":
        assert abs(G["cfg1"]["sumsq"] - 135.10119655928548) < 1e-12


def test_reference_library_matches_goldens(ref):
    import paper_2505_21070_b200 as bp
    cfg = bp.PipelineConfig.from_dict(G["cfg1"]["config"])
    r = ref.run(cfg)
    lat = np.concatenate([b["frames"].ravel() for b in r["blocks"]])
    assert ref.fnv1a64([lat]) == G["cfg1"]["fnv"]


def test_forward_chunk_rows_matches_full_restatement():
    """The sampled-rows restatement used at Wan shapes (one-layer chunk)
    equals the full restatement on the rows it returns, capture and prefix
    routes included."""
    from oracle import blockpipe_oracle as O
    cfg = {"layers": 1, "hidden": 16, "heads": 2, "channels": 4, "height": 2, "width": 3, "context_len": 5, "ffn": 24}
    ch = O.build_chunk(cfg, 7, 0, 1)
    ctx = O.build_context(cfg, 8)
    rng = np.random.default_rng(1)
    x0, x1 = rng.standard_normal((4 * 6, 4)), rng.standard_normal((4 * 6, 4))
    full0, cap0, _ = O.forward_chunk(ch, x0, [9, 9, 9, 9], [0, 1, 2, 3], ctx, mode="on", capture=[1, 2])
    rows = [0, 5, 7, 23]
    part0, pcap = O.forward_chunk_rows(ch, x0, [9, 9, 9, 9], [0, 1, 2, 3], ctx, rows, capture=[1, 2])
    assert np.allclose(part0, full0[rows], rtol=1e-12, atol=1e-12)
    assert np.array_equal(pcap[0], cap0[0][0]) and np.array_equal(pcap[1], cap0[0][1])
    full1, _, _ = O.forward_chunk(ch, x1, [8] * 4, [2, 3, 4, 5], ctx, mode="on", cache=cap0)
    part1, _ = O.forward_chunk_rows(ch, x1, [8] * 4, [2, 3, 4, 5], ctx, rows, prefix=pcap)
    assert np.allclose(part1, full1[rows], rtol=1e-12, atol=1e-12)
