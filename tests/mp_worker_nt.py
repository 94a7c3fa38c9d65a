"""One rank of a multi-process pipeline run WITHOUT PyTorch: the ranks
rendezvous through files (bp_bootstrap_nccl_ids / bp_bootstrap_ipc) in a
shared directory. Launched by tests/test_gpu_multiproc.py as plain
processes with RANK / WORLD_SIZE set:

    RANK=r WORLD_SIZE=n python tests/mp_worker_nt.py CONFIG_JSON OUT_PREFIX BOOTSTRAP_DIR [RUNS]

Rank 0 saves the emitted latents of each run; every rank saves its stats."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # several processes time-slice one GPU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np

    import paper_2505_21070_b200 as bp

    cfg = bp.PipelineConfig.from_dict(json.loads(sys.argv[1]))
    prefix, boot = sys.argv[2], sys.argv[3]
    runs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if cfg.transport == "nccl":  # all ranks share GPU 0: NCCL must treat them as separate hosts
        os.environ["NCCL_HOSTID"] = f"blockpipe-nt-rank-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
    pipe = bp.Pipeline(cfg, rank=rank, world=world, device=0, bootstrap_dir=boot)
    out = {}
    for r in range(runs):
        blocks = pipe.run()
        if rank == 0:
            out[f"run{r}"] = np.concatenate([b["frames"].ravel() for b in blocks])
    st = pipe.stats()
    if rank == 0:
        np.savez(prefix + ".npz", **out)
    with open(f"{prefix}.rank{rank}.json", "w") as f:
        json.dump({"boundary_copies": st["boundary_copies"], "registered_buffers": st["registered_buffers"],
                   "boundary_bytes": st["boundary_bytes"], "fused_sends": st["fused_sends"],
                   "passes": st["passes"], "torch_loaded": "torch" in sys.modules}, f)


if __name__ == "__main__":
    main()
