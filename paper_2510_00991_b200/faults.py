"""Fault injection on the copy paths (FaultScript / apply_fault).

A fault names a directed path ``src -> dst`` (primary = copy engine, backup =
SM kernel) and a trigger: a time offset or the issue of a given chunk of the
sender's n-th send.  Down closes a gate (a stream wait on a host word) in
front of every copy the sender issues on that path from then on, so the path
genuinely stalls on the device; Up opens it ("RNIC port
down" -> injected gate on the primary copy-engine path).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

from .errors import InvalidArgument

PRIMARY, BACKUP = 0, 1


@dataclass
class FaultEntry:
    src: int
    dst: int
    up: bool = False
    path: int = PRIMARY
    t_us: int = 0
    chunk: int = -1     # >= 0: fire when the sender issues this chunk ...
    op_index: int = 0   # ... of its op_index-th send to dst (counted from install)

    @property
    def trigger_kind(self) -> int:
        return 1 if self.chunk >= 0 else 0


@dataclass
class FaultScript:
    """Time-ordered entries; Down/Up alternate per path."""

    entries: List[FaultEntry] = field(default_factory=list)

    def down(self, src: int, dst: int, *, t_us: int = 0, chunk: int = -1, op_index: int = 0,
             path: int = PRIMARY) -> "FaultScript":
        self.entries.append(FaultEntry(src, dst, False, path, t_us, chunk, op_index))
        return self

    def up(self, src: int, dst: int, *, t_us: int = 0, chunk: int = -1, op_index: int = 0,
           path: int = PRIMARY) -> "FaultScript":
        self.entries.append(FaultEntry(src, dst, True, path, t_us, chunk, op_index))
        return self

    def validate(self, nranks: int) -> None:
        state = {}
        last_t = -1
        for e in self.entries:
            if not (0 <= e.src < nranks and 0 <= e.dst < nranks):
                raise InvalidArgument(f"fault names unknown path {e.src}->{e.dst} (UnknownPort)")
            if e.trigger_kind == 0:
                if e.t_us < last_t:
                    raise InvalidArgument("time-triggered fault entries must be sorted by time")
                last_t = e.t_us
            key = (e.src, e.dst, e.path)
            # a script may open with Up: it restores a path a previous script left Down
            if key in state and state[key] == e.up:
                raise InvalidArgument(f"Down/Up must alternate on path {key}")
            state[key] = e.up
