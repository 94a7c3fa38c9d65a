"""Exception taxonomy of the reference (errors.hpp:11-41), plus device errors.

bp_status codes from include/bp_cuda.h map 1:1 onto these classes.
"""


class BlockpipeError(RuntimeError):
    """Base of everything raised through the C-ABI."""


class ConfigError(BlockpipeError):
    pass


class DimensionError(BlockpipeError):
    pass


class PartitionError(ConfigError):
    pass


class CacheError(BlockpipeError):
    pass


class SchedulerError(BlockpipeError):
    pass


class QueueError(BlockpipeError):
    pass


class SchedulingError(BlockpipeError):
    pass


class IoError(BlockpipeError):
    pass


class CudaError(BlockpipeError):
    pass


class NcclError(BlockpipeError):
    pass


_BY_STATUS = {1: ConfigError, 2: DimensionError, 3: CacheError, 4: SchedulerError, 5: QueueError,
              6: SchedulingError, 7: PartitionError, 8: IoError, 9: CudaError, 10: NcclError}


def from_status(status: int, msg: str) -> BlockpipeError:
    return _BY_STATUS.get(status, BlockpipeError)(msg)
