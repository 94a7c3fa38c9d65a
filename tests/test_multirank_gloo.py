"""Row (e) on CPU: the one-process-per-GPU pipeline program, replayed across
world_size 2 and 3 gloo ranks.

Each rank runs exactly the op sequence the NCCL executor issues on that rank
(bp_schedule_rank_program: rank 0 merges its stage forwards and eps updates by
the logical slot clock), with the pass records of the host schedule
(bp_schedule_pass: state versions, context sources, capture frames, cache
ids), the numpy oracle as the stage compute (test infrastructure) and gloo
point-to-point transfers: non-blocking sends (the executor's send streams) and
receives at the point of use. The final latents must equal the serial,
round-atomic oracle bit for bit: any op order that read a stale state version
or a wrong cache would change them, and a deadlocking order would hang
(bounded by the timeout).
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE = {"layers": 4, "hidden": 16, "heads": 2, "channels": 2, "height": 2, "width": 2, "context_len": 3,
        "num_b": 2, "num_c": 4, "steps": 4, "blocks": 4, "mode": "single"}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, cfgd, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2505_21070_b200 as bp
    from oracle import blockpipe_oracle as bo

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = bp.PipelineConfig.from_dict(dict(cfgd, devices=world))
        s = bp.Schedule(cfg)
        begin, end = s.partition[rank]
        m = {k: cfgd[k] for k in ("layers", "hidden", "heads", "channels", "height", "width", "context_len")}
        ch = bo.build_chunk(m, cfg.seed_model, begin, end)
        context = bo.build_context(m, cfg.seed_context)
        tpf, C, h, T = cfg.height * cfg.width, cfg.channels, cfg.hidden, cfg.steps
        passes = [s.pass_record(i) for i in range(s.npasses)]
        cache = rec = None          # this stage's single-entry cache (DeviceWorker::cache_)
        cache_block = rec_block = -1
        sends = []
        if rank == 0:
            M = cfg.num_b + cfg.num_c // 2
            pool = bo.RandomSource(bo.derive_seed(cfg.seed_noise, [0])).normal_tensor((M, tpf * C))
            ids = {b["block_id"]: b["noise_ids"] for b in s.blocks}
            versions, emitted, appended = {}, [], 0
        for kind, i in s.rank_program(rank):
            p = passes[i]
            if kind == 0:
                if rank == 0:
                    while appended < cfg.blocks and s.block_meta(appended + 1)["append_round"] <= p["round"]:
                        appended += 1
                        versions[appended] = [pool[ids[appended]].reshape(-1, C).copy(), None, None]
                    parts = []
                    if p["ctx"]:
                        src = versions[p["ctx_block"]][p["ctx_version"] % 3]
                        r0 = p["ctx_first_frame"] * tpf
                        parts.append(src[r0:r0 + p["ctx_frames"] * tpf])
                    parts.append(versions[p["block"]][p["version"] % 3])
                    payload = np.concatenate(parts)
                else:
                    buf = torch.empty((p["tokens"], h), dtype=torch.float64)
                    dist.recv(buf, src=rank - 1)
                    payload = buf.numpy()
                use = p["cached_context_id"] >= 0 and cfg.cache != "off"
                if use:
                    have = cache_block if cfg.cache == "on" else rec_block
                    assert have == p["cached_context_id"], (rank, i, have, p["cached_context_id"])
                out, cap, rcd = bo.forward_chunk(
                    ch, payload, p["frame_levels"], p["frame_ids"], context, cfg.cache,
                    cache=cache if (use and cfg.cache == "on") else None,
                    recorded=rec if (use and cfg.cache == "recompute") else None,
                    capture=p["capture_frames"])
                cache, rec = cap, rcd
                cache_block = p["block"] if cap is not None else -1
                rec_block = p["block"] if rcd is not None else -1
                dst = rank + 1 if rank + 1 < world else 0
                sends.append(dist.isend(torch.from_numpy(np.ascontiguousarray(out)), dst))
            else:
                buf = torch.empty((p["tokens"], C), dtype=torch.float64)
                dist.recv(buf, src=world - 1)
                eps = buf.numpy()[-p["center_tokens"]:]
                x = versions[p["block"]][p["version"] % 3]
                versions[p["block"]][(p["version"] + 1) % 3] = x - eps * (1.0 / T)
                if p["finishes_block"]:
                    emitted.append((p["block"], versions[p["block"]][T % 3].copy()))
        for w in sends:
            w.wait()
        if rank == 0:
            q.put(emitted)
    finally:
        dist.destroy_process_group()


def _run(world, cfgd):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, cfgd, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    emitted = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return emitted


@pytest.mark.parametrize("world,extra", [(2, {}), (2, {"order": "sequential"}), (2, {"cache": "recompute"}),
                                         (3, {"uneven_split": True}), (2, {"blocks": 6, "steps": 3})])
def test_rank_programs_reproduce_serial_oracle(world, extra):
    from oracle import blockpipe_oracle as bo
    cfgd = dict(BASE, **extra)
    emitted = _run(world, cfgd)
    want = bo.run_pipeline({k: v for k, v in cfgd.items() if k not in ("mode", "uneven_split")})
    assert [b for b, _ in emitted] == [b["block_id"] for b in want["blocks"]]
    for (_, got), w in zip(emitted, want["blocks"]):
        assert np.array_equal(got.ravel(), w["frames"].ravel())


def test_rank0_program_respects_dependencies():
    """Every state a stage-0 forward reads was produced by an update placed
    earlier in rank 0's program (checked for the Wan-shaped 8-GPU schedule)."""
    import paper_2505_21070_b200 as bp
    s = bp.Schedule({"devices": 8, "layers": 30, "hidden": 8, "heads": 2, "channels": 1, "height": 1, "width": 1,
                     "num_b": 8, "num_c": 8, "steps": 50, "blocks": 9, "uneven_split": True})
    done = set()  # (block, version) available
    passes = [s.pass_record(i) for i in range(s.npasses)]
    for kind, i in s.rank_program(0):
        p = passes[i]
        if kind == 0:
            assert p["version"] == 0 or (p["block"], p["version"]) in done
            if p["ctx"] == 1 and p["ctx_version"] > 0:
                assert (p["ctx_block"], p["ctx_version"]) in done
            if p["ctx"] == 2:
                assert (p["ctx_block"], 50) in done
        else:
            done.add((p["block"], p["version"] + 1))
