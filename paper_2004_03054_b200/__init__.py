"""B200-native (sm_100a) LUDA compaction path — a drop-in for the reference's
offload-device plugin and its run_compaction entry point.

Public API (mirrors pkg/src/luda): make_device, DeviceConfig, StoreConfig,
run_compaction, KernelSpec, the error tree, SstMeta/CompactionJob/Version.
The CUDA library (libluda_b200.so) is loaded lazily on first device use; there
is no CPU fallback.
"""

from .config import DeviceConfig, StoreConfig  # noqa: F401
from .errors import (  # noqa: F401
    CapacityError,
    CorruptionError,
    DeviceError,
    FormatError,
    LudaError,
    OrderingError,
    SizeOverflowError,
    UnsupportedInputError,
)
from .version import CompactionJob, SstMeta, Version  # noqa: F401


def make_device(config=None):
    from .device import make_device as _mk

    return _mk(config or DeviceConfig())


def run_compaction(job, device, **kw):
    from .compaction import run_compaction as _rc

    return _rc(job, device, **kw)


def run_compactions(jobs, device, **kw):
    from .compaction import run_compactions as _rcs

    return _rcs(jobs, device, **kw)


__all__ = ["DeviceConfig", "StoreConfig", "make_device", "run_compaction", "run_compactions", "CompactionJob", "SstMeta", "Version",
           "LudaError", "FormatError", "CorruptionError", "OrderingError", "SizeOverflowError", "DeviceError",
           "CapacityError", "UnsupportedInputError"]
