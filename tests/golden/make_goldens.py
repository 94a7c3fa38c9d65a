"""Generates tests/golden/*.npz|json from the UNMODIFIED reference library
(oracle/_ref/libbp_ref.so, built from /root/reference by oracle/Makefile).
Run in the build container: python tests/golden/make_goldens.py"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2505_21070_b200 as bp  # noqa: E402  (config helper only)
from oracle import ref  # noqa: E402

CONFIGS = {
    # BASELINE configs[0]: tiny DiT, 2 layers, d=128, 4 heads, 4 blocks x 10 steps, defaults elsewhere
    "cfg1": {"devices": 1, "layers": 2, "hidden": 128, "heads": 4, "steps": 10, "blocks": 4, "mode": "single"},
    "cfg1_nocache": {"devices": 1, "layers": 2, "hidden": 128, "heads": 4, "steps": 10, "blocks": 4,
                     "cache": "off", "mode": "single"},
    # SURVEY Appendix A mid parity config (dh = 128, C = 64)
    "mid": {"devices": 1, "layers": 4, "hidden": 256, "heads": 2, "channels": 64, "height": 4, "width": 6,
            "context_len": 16, "num_b": 8, "num_c": 8, "steps": 6, "blocks": 3, "mode": "single"},
}


def main():
    out = {}
    for name, d in CONFIGS.items():
        cfg = bp.PipelineConfig.from_dict(d)
        r = ref.run(cfg, serial=True)
        lat = np.concatenate([b["frames"].ravel() for b in r["blocks"]])
        np.savez_compressed(os.path.join(HERE, f"{name}_latents.npz"), latents=lat, events=r["events"])
        out[name] = {"config": d, "fnv": ref.fnv1a64([lat]), "sumsq": float((lat ** 2).sum()),
                     "blocks": [{"block_id": b["block_id"], "noise_ids": b["noise_ids"], "frame_ids": b["frame_ids"]}
                                for b in r["blocks"]],
                     "ledger": r["ledger"], "snapshots": r["queue_snapshots"], "bubbles": r["bubbles"],
                     "rounds": r["rounds"]}
        print(name, out[name]["fnv"], out[name]["sumsq"], flush=True)
    seed = bp.derive_seed(2, [0])
    out["pools"] = {}
    for tag, shape in {"tiny": (2, 2, 2), "480p": (30, 52, 64), "720p": (45, 80, 64)}.items():
        p = ref.pool(8, 8, shape, seed)
        out["pools"][tag] = {"fnv": ref.fnv1a64([p]), "e0_0": float(p.ravel()[0]), "shape": shape}
    out["rng"] = {"u64_seed1": [], "normals_seed1": ref.normals(1, 3).tolist(),
                  "derive": {"2,[0]": bp.derive_seed(2, [0]), "2,[1]": bp.derive_seed(2, [1]),
                             "1,[0,0]": bp.derive_seed(1, [0, 0])}}
    out["coordinated_ids"] = bp.coordinated_noise_ids(8, 8, 3)
    with open(os.path.join(HERE, "goldens.json"), "w") as f:
        json.dump(out, f, indent=1)


ARTIFACT_CONFIGS = {
    "default": {},
    "n2_single": {"devices": 2, "mode": "single", "steps": 5, "blocks": 4},
    "n4_seq_trim": {"devices": 4, "order": "sequential", "cache": "off", "emit_first_surplus": False,
                    "steps": 4, "blocks": 3},
    "n2_fresh": {"devices": 2, "strategy": "fresh", "steps": 3, "blocks": 5, "retain_clean_context": False},
}


def make_artifacts():
    """Reference artifacts (artifacts.cpp:25-143) for byte-level comparison."""
    import shutil
    import subprocess
    import tempfile
    script = os.path.abspath(os.path.join(HERE, "..", "..", "oracle", "ref_artifacts.py"))
    for name, cfg in ARTIFACT_CONFIGS.items():
        dst = os.path.join(HERE, "artifacts", name)
        shutil.rmtree(dst, ignore_errors=True)
        with tempfile.TemporaryDirectory() as tmp:
            # relative out_dir "out": the reference prints out_dir into the
            # artifacts, tests reproduce it by writing from a temp cwd.
            subprocess.run([sys.executable, script, json.dumps(cfg), "out"], check=True, cwd=tmp)
            shutil.copytree(os.path.join(tmp, "out"), dst)
        with open(os.path.join(dst, "config.json"), "w") as f:
            json.dump(cfg, f)


if __name__ == "__main__":
    if not os.environ.get("ARTIFACTS_ONLY"):
        main()
    make_artifacts()
