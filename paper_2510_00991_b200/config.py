"""Configuration of the ICCL B200 path (RunConfig).

Defaults come from the C library (``iccl_config_init``): Table 5 values
 mapped onto the B200 path, each overridable through an
``ICCL_*`` environment variable, e.g. ``ICCL_IB_TIMEOUT`` /
``ICCL_IB_RETRY_CNT`` like the paper's knobs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

from ._lib import Config as _CConfig, lib
from .errors import raise_for

TRANSPORTS = {"auto": 0, "ce": 1, "sm": 2}
BACKUPS = {"sm": 0, "relay": 1}


@dataclass
class IcclConfig:
    chunk_bytes: int = 0
    streams_per_peer: int = 0
    sm_cap: int = 0
    window: int = 0
    monitor_window: int = 0
    monitor_enabled: bool = False
    backup_kind: str = "sm"
    transport: str = "auto"
    timeout_exponent: int = 0
    retry_count: int = 0
    delta_us: int = 0
    probe_period_us: int = 0
    sm_small_bytes: int = 0
    proxy_cpu: int = -1
    relay_slot_mib: int = 0
    direct_max_kib: int = 0

    @classmethod
    def defaults(cls, **overrides) -> "IcclConfig":
        c = _CConfig()
        raise_for(lib.iccl_config_init(C.byref(c)), "iccl_config_init")
        inv_t = {v: k for k, v in TRANSPORTS.items()}
        inv_b = {v: k for k, v in BACKUPS.items()}
        cfg = cls(chunk_bytes=c.chunk_bytes, streams_per_peer=c.streams_per_peer, sm_cap=c.sm_cap, window=c.window,
                  monitor_window=c.monitor_window, monitor_enabled=bool(c.monitor_enabled),
                  backup_kind=inv_b.get(c.backup_kind, "sm"), transport=inv_t.get(c.transport, "auto"),
                  timeout_exponent=c.timeout_exponent, retry_count=c.retry_count, delta_us=c.delta_us,
                  probe_period_us=c.probe_period_us, sm_small_bytes=c.sm_small_bytes, proxy_cpu=c.proxy_cpu,
                  relay_slot_mib=c.relay_slot_mib, direct_max_kib=c.direct_max_kib)
        names = {f.name for f in fields(cls)}
        for k, v in overrides.items():
            if k not in names:
                from .errors import ConfigError
                raise ConfigError(f"unknown config field {k!r}")
            setattr(cfg, k, v)
        return cfg

    def to_c(self) -> _CConfig:
        c = _CConfig()
        c.chunk_bytes = int(self.chunk_bytes)
        c.streams_per_peer = int(self.streams_per_peer)
        c.sm_cap = int(self.sm_cap)
        c.window = int(self.window)
        c.monitor_window = int(self.monitor_window)
        c.monitor_enabled = int(bool(self.monitor_enabled))
        c.backup_kind = BACKUPS[self.backup_kind]
        c.transport = TRANSPORTS[self.transport]
        c.timeout_exponent = int(self.timeout_exponent)
        c.retry_count = int(self.retry_count)
        c.delta_us = int(self.delta_us)
        c.probe_period_us = int(self.probe_period_us)
        c.sm_small_bytes = int(self.sm_small_bytes)
        c.proxy_cpu = int(self.proxy_cpu)
        c.relay_slot_mib = int(self.relay_slot_mib)
        c.direct_max_kib = int(self.direct_max_kib)
        return c

    def validate(self) -> "IcclConfig":
        if self.backup_kind not in BACKUPS or self.transport not in TRANSPORTS:
            from .errors import InvalidConfig
            raise InvalidConfig(f"backup_kind {self.backup_kind!r} / transport {self.transport!r}")
        c = self.to_c()
        raise_for(lib.iccl_config_validate(C.byref(c)), "iccl_config_validate")
        return self


def retry_timeout(timeout_exponent: int, retry_count: int) -> float:
    """retry_timeout in seconds: 4.096 µs × 2^exp × (retry + 1)."""
    return lib.iccl_retry_timeout_ns(int(timeout_exponent), int(retry_count)) * 1e-9
