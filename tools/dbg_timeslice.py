"""Determinism under time-slicing (tests/test_gpu_timeslice.py): the
production-shape pipeline run alone writes a reference; run while another
process shares the GPU it must match bitwise.
    python tools/dbg_timeslice.py ref OUT.npy | check REF.npy N"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2505_21070_b200 as bp
from paper_2505_21070_b200._lib import lib
if os.environ.get("BP_IMPL"):
    g, a = (int(v) for v in os.environ["BP_IMPL"].split(","))
    assert lib.bp_set_kernel_impl(g, a) == 0
base = dict(layers=int(os.environ.get("BP_DBG_LAYERS", "4")), hidden=1536, heads=12, ffn=8960, channels=64,
            height=30, width=52, context_len=512, num_b=8, num_c=8, steps=2, blocks=2, precision="bf16",
            mode="single", devices=1)
lat = lambda o: np.concatenate([b["frames"].ravel() for b in o["blocks"]])
if sys.argv[1] == "ref":
    np.save(sys.argv[2], lat(bp.run_pipeline(base)))
else:
    ref = np.load(sys.argv[2])
    pipe = bp.Pipeline(bp.PipelineConfig.from_dict(base))
    for k in range(int(sys.argv[3])):
        blocks = pipe.run()
        g = np.concatenate([b["frames"].ravel() for b in blocks])
        bad = np.flatnonzero(g != ref)
        print(os.environ.get("BP_IMPL", "default"), os.getpid(), k, "equal" if bad.size == 0 else
              f"DIFF n={bad.size} first={bad[0]} maxabs={np.abs(g-ref).max():.3e}", flush=True)
