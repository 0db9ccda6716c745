"""Window throughput monitor of the oracle (test infrastructure only).

Restates SPEC.md:299-379 / PAPER.md:518-557 (no reference code exists):

* ``per_message_throughput`` B = ω / (t2 - t1), bytes/s.
* ``window_throughput`` B̄ = Σω / (t2_last - t1_first) over exactly W records
  ordered by completion; t1 of the window is the post time of the
  earliest-completing record.
* ``sample_series`` — one sample per WC once >= W records, timestamped at the
  triggering t2; N records give N - W + 1 samples.
* ``resample`` — fixed-interval (10 µs) resampling for figure parity
  (SPEC.md:378).
* ``detect_lagging_rank`` — the unique strict minimum opCount whose gap to the
  second smallest exceeds the threshold (strict), else None (SPEC.md:349-357,
  370).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence

from .des import SimulationError


class NonPositiveDuration(SimulationError):
    """t2 <= t1."""


class WindowNotFull(SimulationError):
    """window_throughput before W records."""


@dataclass
class Sample:
    time: int
    value: float
    window_size: int


def per_message_throughput(size: int, t1_ns: int, t2_ns: int) -> float:
    if t2_ns <= t1_ns:
        raise NonPositiveDuration(f"t2={t2_ns} <= t1={t1_ns}")
    return size / ((t2_ns - t1_ns) * 1e-9)


def window_throughput(records: Sequence, window: int) -> float:
    """``records``: objects with .size .t1 .t2 in completion order, len == W."""
    if window < 1:
        raise SimulationError("window size must be >= 1")
    if len(records) != window:
        raise WindowNotFull(f"{len(records)} of {window} records")
    t1_first = records[0].t1
    t2_last = records[-1].t2
    if t2_last <= t1_first:
        raise NonPositiveDuration(f"t2={t2_last} <= t1={t1_first}")
    return sum(r.size for r in records) / ((t2_last - t1_first) * 1e-9)


def sample_series(records: Iterable, window: int) -> List[Sample]:
    if window < 1:
        raise SimulationError("window size must be >= 1")
    recs = sorted(records, key=lambda r: r.t2)  # completion order
    out = []
    for i in range(window - 1, len(recs)):
        win = recs[i - window + 1:i + 1]
        out.append(Sample(win[-1].t2, window_throughput(win, window), window))
    return out


def resample(samples: Sequence[Sample], period_ns: int = 10_000) -> List[Sample]:
    """Last-value-held samples on a fixed grid starting at the first sample."""
    if not samples:
        return []
    out = []
    t = samples[0].time
    i = 0
    while t <= samples[-1].time:
        while i + 1 < len(samples) and samples[i + 1].time <= t:
            i += 1
        out.append(Sample(t, samples[i].value, samples[i].window_size))
        t += period_ns
    return out


def detect_lagging_rank(op_counts: Dict[int, int], threshold: int = 1) -> Optional[int]:
    if len(op_counts) < 2:
        raise SimulationError("need at least two ranks")
    ordered = sorted(op_counts.items(), key=lambda kv: kv[1])
    (rank, lo), (_, second) = ordered[0], ordered[1]
    if lo == second:
        return None
    return rank if second - lo > threshold else None
