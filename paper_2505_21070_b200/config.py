"""PipelineConfig / ModelConfig mirror (engine.hpp:24-38, model.hpp:21-32,
block_queue.hpp:36-43) and the reference's flat JSON keys (run_config.cpp:48-104),
plus the B200 extensions (ffn width, precision, transport, uneven split)."""
from __future__ import annotations

import dataclasses
import os
from typing import Any, Dict, Optional, Sequence

from . import errors
from ._lib import ModelDesc, PipelineDesc

ORDERS = {"reverse": 0, "sequential": 1}
CACHE = {"off": 0, "on": 1, "recompute": 2}
STRATEGIES = {"coordinated": 0, "complete-shuffle": 1, "subset": 2, "fresh": 3, "repeat": 4}
PRECISIONS = {"f64": 0, "f32": 1, "bf16": 2}
TRANSPORTS = {"loopback": 0, "nccl": 1, "ipc": 2}
BLOCKS = {"reference": 0, "wan": 1}  # bp_block


@dataclasses.dataclass
class PipelineConfig:
    devices: int = 2
    order: str = "reverse"
    cache: str = "on"
    threaded: bool = True          # accepted for compatibility; the GPU engine is stream-ordered
    num_b: int = 2
    num_c: int = 4
    steps: int = 8
    blocks: int = 6
    retain_clean_context: bool = True
    layers: int = 4
    hidden: int = 16
    heads: int = 2
    channels: int = 2
    height: int = 2
    width: int = 2
    context_len: int = 4
    strategy: str = "coordinated"
    seed_model: int = 1
    seed_noise: int = 2
    seed_context: int = 3
    fault_inject: bool = False
    record_trace: bool = False
    check_cache: bool = False
    # B200 extensions
    ffn: int = 0                   # 0 => 4*hidden (model.cpp:98-99)
    block: str = "reference"       # "wan": the optional non-parity Wan2.1-style block
    precision: str = "f64"
    transport: str = "loopback"
    uneven_split: bool = False
    layer_split: Optional[Sequence[int]] = None

    @classmethod
    def from_dict(cls, d: Optional[Dict[str, Any]] = None) -> "PipelineConfig":
        """run_config_from_json_text semantics: unknown keys are ConfigErrors;
        BLOCKPIPE_SEED supplies default seeds S, S+1, S+2."""
        cfg = cls()
        env = os.environ.get("BLOCKPIPE_SEED")
        if env is not None:
            base = int(env)
            cfg.seed_model, cfg.seed_noise, cfg.seed_context = base, base + 1, base + 2
        for k, v in (d or {}).items():
            if k == "mode":
                if v not in ("threaded", "single"):
                    raise errors.ConfigError("mode must be threaded or single")
                cfg.threaded = v == "threaded"
            elif k == "cache":
                if v not in CACHE:
                    raise errors.ConfigError(f"cache must be on, off or recompute, got {v}")
                cfg.cache = v
            elif k == "order":
                if v not in ORDERS:
                    raise errors.ConfigError(f"order must be reverse or sequential, got {v}")
                cfg.order = v
            elif k == "strategy":
                if v not in STRATEGIES:
                    raise errors.ConfigError(f"unknown noise strategy: {v}")
                cfg.strategy = v
            elif k == "fault_inject":
                cfg.fault_inject = bool(v)
            elif k == "block":
                if v not in BLOCKS:
                    raise errors.ConfigError(f"block must be reference or wan, got {v}")
                cfg.block = v
            elif k in ("out_dir", "emit_first_surplus", "format"):
                pass  # operator-surface keys (artifacts / CLI), not part of the hot path
            elif k in {f.name for f in dataclasses.fields(cls)}:
                setattr(cfg, k, v)
            else:
                raise errors.ConfigError(f"unknown config key: {k}")
        return cfg

    def model_desc(self) -> ModelDesc:
        if self.block not in BLOCKS:
            raise errors.ConfigError(f"block must be reference or wan, got {self.block}")
        return ModelDesc(self.layers, self.hidden, self.heads, self.channels, self.height,
                         self.width, self.context_len, self.ffn, BLOCKS[self.block])

    def to_desc(self) -> PipelineDesc:
        d = PipelineDesc()
        d.devices = self.devices
        d.order = ORDERS[self.order]
        d.cache_mode = CACHE[self.cache]
        d.num_b, d.num_c, d.steps, d.block_num = self.num_b, self.num_c, self.steps, self.blocks
        d.retain_clean_context = int(bool(self.retain_clean_context))
        d.strategy = STRATEGIES[self.strategy]
        d.model = self.model_desc()
        d.seed_model, d.seed_noise, d.seed_context = self.seed_model, self.seed_noise, self.seed_context
        d.fault_inject_ulp = int(bool(self.fault_inject))
        d.record_trace = int(bool(self.record_trace))
        d.check_cache = int(bool(self.check_cache))
        if self.precision not in PRECISIONS:
            raise errors.ConfigError(f"precision must be one of {sorted(PRECISIONS)}")
        d.precision = PRECISIONS[self.precision]
        d.transport = TRANSPORTS[self.transport]
        d.uneven_split = int(bool(self.uneven_split))
        if self.layer_split:
            for i, n in enumerate(self.layer_split):
                d.layer_split[i] = int(n)
        return d
