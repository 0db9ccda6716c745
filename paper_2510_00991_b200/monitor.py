"""Window-based µs throughput monitor.

Records are the WR/WC pairs of the copy path: one per chunk, t1 at issue and
t2 at completion (``iccl_mon_rec_t``), drained from the communicator's ring.
The formulas run in the C library (``iccl_window_throughput`` …), the same
code the runtime uses; this module only marshals records.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

from ._lib import MonRec, lib
from .errors import raise_for


@dataclass
class MessageRecord:
    """WR/WC pair: ``size`` = ω(M), ``t1``/``t2`` in ns."""

    size: int
    t1: int
    t2: int
    peer: int = -1
    path: int = 0
    chunk: int = -1
    op_seq: int = 0
    dir: int = 0  # 0: a transfer this rank pushed to `peer`, 1: one it pulled from `peer`


@dataclass
class ThroughputSample:
    time: int
    value: float  # bytes/s
    window_size: int


def _to_c(records: Sequence[MessageRecord]):
    arr = (MonRec * max(1, len(records)))()
    for i, r in enumerate(records):
        arr[i].t1_ns = int(r.t1)
        arr[i].t2_ns = int(r.t2)
        arr[i].bytes = int(r.size)
        arr[i].peer = int(r.peer)
        arr[i].path = int(r.path)
        arr[i].chunk = int(r.chunk)
    return arr


def per_message_throughput(record: MessageRecord) -> float:
    """B = ω / (t2 − t1) in bytes/s; raises NonPositiveDuration."""
    arr = _to_c([record])
    out = C.c_double()
    raise_for(lib.iccl_per_message_throughput(arr, C.byref(out)), "per_message_throughput")
    return out.value


def window_throughput(records: Sequence[MessageRecord], window: Optional[int] = None) -> float:
    """B̄ = Σω / (t2_last − t1_first) over exactly W records in completion order
    (SPEC.md:331-339); raises WindowNotFull / NonPositiveDuration."""
    w = len(records) if window is None else int(window)
    arr = _to_c(records)
    out = C.c_double()
    raise_for(lib.iccl_window_throughput(arr, len(records), w, C.byref(out)), "window_throughput")
    return out.value


def sample_series(records: Sequence[MessageRecord], window: int = 8) -> List[ThroughputSample]:
    """One sample per completion once W records are in: N − W + 1 samples
    timestamped at the triggering t2."""
    recs = sorted(records, key=lambda r: r.t2)
    n = len(recs)
    m = max(0, n - window + 1)
    arr = _to_c(recs)
    vals = (C.c_double * max(1, m))()
    ts = (C.c_uint64 * max(1, m))()
    n_out = C.c_int()
    raise_for(lib.iccl_sample_series(arr, n, int(window), vals, ts, C.byref(n_out)), "sample_series")
    return [ThroughputSample(int(ts[i]), float(vals[i]), window) for i in range(n_out.value)]


def resample(samples: Sequence[ThroughputSample], period_ns: int = 10_000) -> List[ThroughputSample]:
    """Fixed-interval (10 µs) last-value resampling for figure parity."""
    out: List[ThroughputSample] = []
    if not samples:
        return out
    t, i = samples[0].time, 0
    while t <= samples[-1].time:
        while i + 1 < len(samples) and samples[i + 1].time <= t:
            i += 1
        out.append(ThroughputSample(t, samples[i].value, samples[i].window_size))
        t += period_ns
    return out


def detect_lagging_rank(op_counts: Dict[int, int], threshold: int = 1) -> Optional[int]:
    """opCount straggler: the unique strict
    minimum whose gap to the second smallest exceeds ``threshold``, else None."""
    ranks = sorted(op_counts)
    arr = (C.c_uint64 * len(ranks))(*[int(op_counts[r]) for r in ranks])
    out = C.c_int()
    raise_for(lib.iccl_detect_lagging_rank(arr, len(ranks), int(threshold), C.byref(out)), "detect_lagging_rank")
    return None if out.value < 0 else ranks[out.value]


class Monitor:
    """Per-communicator monitor: drains chunk records from the C ring and keeps
    them per peer; ``samples(peer)`` gives the window series (default W from
    the config, Table 5: 8)."""

    def __init__(self, comm, window: int = 8):
        self.comm = comm
        self.window = window
        self.records: List[MessageRecord] = []

    def enable(self, on: bool = True, window: Optional[int] = None) -> None:
        if window is not None:
            self.window = window
        raise_for(lib.iccl_monitor_config(self.comm._h, int(on), int(self.window)), "iccl_monitor_config")

    def drain(self) -> List[MessageRecord]:
        buf = (MonRec * 4096)()
        got: List[MessageRecord] = []
        while True:
            n = C.c_int()
            raise_for(lib.iccl_monitor_read(self.comm._h, buf, 4096, C.byref(n)), "iccl_monitor_read")
            for i in range(n.value):
                r = buf[i]
                got.append(MessageRecord(int(r.bytes), int(r.t1_ns), int(r.t2_ns), r.peer, r.path, r.chunk,
                                         int(r.op_seq), int(r.dir)))
            if n.value < 4096:
                break
        self.records.extend(got)
        return got

    def samples(self, peer: Optional[int] = None, window: Optional[int] = None) -> List[ThroughputSample]:
        self.drain()
        recs = [r for r in self.records if peer is None or r.peer == peer]
        return sample_series(recs, window or self.window)
