"""Configuration mirrors of the reference's ``luda.config``.

Reference: ``pkg/src/luda/config.py:13-66``. ``DeviceConfig`` keeps every
field of the reference (so a reference-built config object can be passed
through unchanged) and adds the knobs of the ``"b200"`` backend:
``device_ordinal``, ``pinned_staging_bytes`` and ``subcompactions``.
``StoreConfig`` keeps the knobs that shape compaction output bytes
(block size, restart interval, bits per key, SST size target).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field


def default_device_workers() -> int:
    return max(1, (os.cpu_count() or 1) - 2)


@dataclass
class DeviceConfig:
    # "b200" selects this package's CUDA backend (the only backend here).
    backend: str = "b200"
    workers: int = 0
    bandwidth_bytes_per_sec: float = 8 * 2**30
    latency_sec: float = 20e-6
    # The reference caps the sum of live regions (config.py:19, 256 MiB).
    # The B200 backend keeps the check but defaults to a budget sized for HBM.
    region_capacity: int = 160 * 2**30
    pin_cores: bool = False
    unpack_expansion: int = 4
    # --- b200 backend knobs -------------------------------------------------
    device_ordinal: int = 0
    pinned_staging_bytes: int = 256 * 2**20
    # Fixed number of key-range subcompactions P (independent of GPU count).
    subcompactions: int = 1

    def effective_workers(self) -> int:
        return self.workers if self.workers > 0 else default_device_workers()


@dataclass
class StoreConfig:
    engine_mode: str = "offload"
    memtable_size: int = 4 * 2**20
    sst_size_target: int = 4 * 2**20
    block_size: int = 4096
    restart_interval: int = 16
    bits_per_key: int = 10
    block_cache_bytes: int = 32 * 2**20
    l0_compaction_trigger: int = 4
    l0_slowdown_files: int = 8
    l0_stall_files: int = 12
    level_base_bytes: int = 10 * 2**20
    level_size_multiplier: int = 10
    max_grandparent_overlap_files: int = 10
    background: bool = True
    stall_mode: str = "block"
    stall_timeout_sec: float = 120.0
    slowdown_sleep_sec: float = 0.001
    device: DeviceConfig = field(default_factory=DeviceConfig)
