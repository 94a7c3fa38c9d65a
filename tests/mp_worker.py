"""One rank of a multi-process pipeline run (launched by torch.distributed.run
from tests/test_gpu_multiproc.py and usable by hand):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port 29611 tests/mp_worker.py CONFIG_JSON OUT_NPZ [RUNS]

Every rank builds the same pipeline (transport from the config: "ipc" for
several processes on one GPU, "nccl" for one process per GPU), exchanges its
IPC handle / NCCL ids over a gloo group, runs RUNS generations and rank 0
saves the emitted latents of each run."""
import json
import os
import sys

import numpy as np

# Processes time-slicing one GPU: a rank whose kernels are still lazily loaded
# can stall behind the other rank's polling wait kernel for seconds; load
# every module when the context is created instead.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist

    import paper_2505_21070_b200 as bp

    cfg = bp.PipelineConfig.from_dict(json.loads(sys.argv[1]))
    out = sys.argv[2]
    runs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist.init_process_group("gloo")
    one_gpu = cfg.transport == "ipc" or os.environ.get("BP_MP_ONE_GPU") == "1"
    device = 0 if one_gpu else local
    if cfg.transport == "nccl" and one_gpu:
        # NCCL refuses two ranks on one GPU of one host (duplicate bus id); a
        # distinct host id per rank makes it treat the ranks as separate hosts
        # and use its socket transport over loopback, which exercises the
        # NCCL executor path on a single device
        os.environ["NCCL_HOSTID"] = f"blockpipe-rank-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")

    def exchange(h):
        got = [None] * world
        dist.all_gather_object(got, h)
        return got

    ids = None
    if cfg.transport == "nccl":
        import ctypes
        from paper_2505_21070_b200._lib import lib
        obj = [None]
        if rank == 0:
            buf = bytearray()
            for _ in range(world):
                b = (ctypes.c_uint8 * 128)()
                assert lib.bp_nccl_unique_id(b) == 0
                buf += bytes(b)
            obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        ids = obj[0]
    pipe = bp.Pipeline(cfg, rank=rank, world=world, device=device, nccl_ids=ids, ipc_exchange=exchange)
    if os.environ.get("BP_IPC_WATCHDOG"):  # diagnostics: dump ring counters if a run hangs
        import ctypes
        import threading
        from paper_2505_21070_b200._lib import lib

        def watch():
            import time
            time.sleep(float(os.environ["BP_IPC_WATCHDOG"]))
            c = (ctypes.c_uint32 * 4)()
            lib.bp_ipc_counters(pipe._h, c)
            print(f"[rank {rank}] watchdog counters {list(c)}", file=sys.stderr, flush=True)
            os._exit(3)
        threading.Thread(target=watch, daemon=True).start()
    results = {}
    for r in range(runs):
        blocks = pipe.run()
        if rank == 0:
            results[f"run{r}"] = np.concatenate([b["frames"].ravel() for b in blocks])
            results[f"ids{r}"] = np.array([b["block_id"] for b in blocks])
    st = pipe.stats()
    dist.barrier()
    if rank == 0:
        np.savez(out, boundary_bytes=st["boundary_bytes"], **results)
    pipe.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
