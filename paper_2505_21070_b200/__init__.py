"""blockpipe-b200: B200-native block-wise denoising (DualParal) behind the
reference blockpipe operator API. Every call goes through the C-ABI in
include/bp_cuda.h (lib/libbp_cuda.so, sm_100a); there is no CPU fallback."""
from .errors import (BlockpipeError, CacheError, ConfigError, CudaError, DimensionError, IoError,
                     NcclError, PartitionError, QueueError, SchedulerError, SchedulingError)
from .config import PipelineConfig
from .api import (Pipeline, Schedule, Stage, build_pool, coordinated_noise_ids, derive_seed, draw_first_block,
                  draw_next_block, gather_block,
                  measure_bubbles, nccl_unique_ids, normals, pinned_empty, run_pipeline, scheduler_step, serial_oracle)

__all__ = [
    "BlockpipeError", "CacheError", "ConfigError", "CudaError", "DimensionError", "IoError", "NcclError",
    "PartitionError", "QueueError", "SchedulerError", "SchedulingError", "PipelineConfig", "Pipeline",
    "Schedule", "Stage", "build_pool", "coordinated_noise_ids", "derive_seed", "draw_first_block",
    "draw_next_block", "gather_block", "measure_bubbles",
    "nccl_unique_ids", "normals", "pinned_empty", "run_pipeline", "scheduler_step", "serial_oracle",
]
