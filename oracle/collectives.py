"""P2P collectives of the oracle (test infrastructure only).

Restates SPEC.md:381-466 for the hot-path members only — ``CommGroup``
(SPEC.md:386-389), ``send_recv`` and ``alltoall`` — plus
the builder-defined, torch-shaped ``alltoallv`` and batched P2P (SURVEY.md
F3: torch ``all_to_all_single`` / ``batch_isend_irecv`` semantics).  Every
ordered pair is a ``transport.Connection`` over the B200 box model
(``netsim.nvswitch_box``): primary path = copy-engine port, backup = SM port.

The delivered bytes are what the GPU path is compared against:
``recv_j[rdispl_j[i] : +count_ij] == send_i[sdispl_i[j] : +count_ij]``
(SURVEY.md §8c), computed here by really moving the bytes chunk by chunk
through the six-pointer protocol, and independently by ``expected_alltoallv``.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .des import SimulationError, Simulator
from .monitor import detect_lagging_rank  # noqa: F401  (re-export for callers)
from .netsim import FaultScript, nvswitch_box, path_port
from .transport import DEFAULT_CHUNK, Connection, MessageRecord
from .verbs import MemoryRegion, Verbs

PRIMARY, BACKUP = 0, 1


class GroupTooSmall(SimulationError):
    """alltoall with fewer than two ranks."""


class CommGroup:
    """Ordered ranks on one B200 box; ``qp_per_connection``
    is the "QP number" (Table 5: 2) mapped to copy streams per peer."""

    def __init__(self, n_ranks: int, chunk_size: int = DEFAULT_CHUNK, qp_per_connection: int = 1,
                 timeout_exponent: int = 0, retry_count: int = 0, delta_ns: Optional[int] = None,
                 window: int = 8, probe_period_ns: int = 500_000, nvlink_gbps: float = 900.0,
                 delay_ns: int = 1000, faults: Optional[FaultScript] = None, cts_timeout_ns: int = 0):
        if n_ranks < 1:
            raise SimulationError("group needs a rank")
        self.n = n_ranks
        self.sim = Simulator()
        self.net, self._path = nvswitch_box(self.sim, n_ranks, nvlink_gbps, delay_ns)
        self.verbs = Verbs(self.sim, self.net)
        self.kw = dict(chunk_size=chunk_size, qp_per_connection=qp_per_connection, timeout_exponent=timeout_exponent,
                       retry_count=retry_count, delta_ns=delta_ns, window=window, probe_period_ns=probe_period_ns,
                       cts_timeout_ns=cts_timeout_ns)
        self.conns: Dict[Tuple[int, int], Connection] = {}
        self.records: List[Tuple[int, int, MessageRecord]] = []
        self.op_count = {r: 0 for r in range(n_ranks)}
        if faults is not None:
            faults.install(self.net)
        self._rid = 0

    def conn(self, src: int, dst: int) -> Connection:
        key = (src, dst)
        if key not in self.conns:
            self.conns[key] = Connection(self.sim, self.verbs, self._path(src, dst, PRIMARY),
                                         self._path(src, dst, BACKUP), conn_id=f"{src}->{dst}",
                                         on_record=lambda r, s=src, d=dst: self.records.append((s, d, r)),
                                         **self.kw)
        return self.conns[key]

    def region(self, owner: int, data: np.ndarray) -> MemoryRegion:
        self._rid += 1
        return MemoryRegion(self._rid, owner, data.reshape(-1).view(np.uint8))

    def trace_sha256(self) -> str:
        return self.sim.trace.sha256()


def _as_bytes(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).reshape(-1).view(np.uint8)


def batch_p2p(group: CommGroup, ops: Sequence[Tuple[int, int, np.ndarray, int, np.ndarray, int, int]],
              ready_at: Optional[Dict[Tuple[int, int], int]] = None) -> None:
    """Run a batch of matched transfers concurrently, like one
    ``batch_isend_irecv`` group: each op is (src, dst, src_bytes, src_off,
    dst_bytes, dst_off, nbytes).  Transfers over the same ordered pair run in
    issue order (NCCL/torch P2P matching).  Self pairs are a local copy."""
    queues: Dict[Tuple[int, int], list] = {}
    for op in ops:
        src, dst, sb, so, db, do, n = op
        if n == 0:
            continue  # zero-count pairs complete at once (Appendix B9)
        if src == dst:
            db[do:do + n] = sb[so:so + n]
            continue
        queues.setdefault((src, dst), []).append(op)
    pending = {"n": sum(len(v) for v in queues.values())}

    def launch(key):
        q = queues[key]
        if not q:
            return
        src, dst, sb, so, db, do, n = q.pop(0)
        c = group.conn(src, dst)
        ra = (ready_at or {}).get(key, group.sim.now)

        def done(key=key):
            pending["n"] -= 1
            launch(key)

        c.send_message(group.region(src, sb), group.region(dst, db), n, so, do, ready_at=ra, on_complete=done)

    for key in queues:
        launch(key)
    group.sim.run()
    if pending["n"] != 0:
        raise SimulationError(f"{pending['n']} transfers did not complete")
    for r in range(group.n):
        group.op_count[r] += 1


def send_recv(group: CommGroup, src: int, dst: int, payload: np.ndarray, out: Optional[np.ndarray] = None,
              ready_at: int = 0) -> np.ndarray:
    """send_recv between two ranks; returns the receiver's
    buffer after delivery."""
    sb = _as_bytes(payload)
    db = np.zeros_like(sb) if out is None else _as_bytes(out)
    if sb.nbytes == 0:
        return db
    batch_p2p(group, [(src, dst, sb, 0, db, 0, sb.nbytes)], {(src, dst): ready_at} if ready_at else None)
    return db


def alltoall(group: CommGroup, send: Sequence[np.ndarray], nbytes_per_pair: int) -> List[np.ndarray]:
    """Uniform alltoall: rank i's block j goes to rank j's
    block i.  N < 2 raises GroupTooSmall; 0 bytes completes immediately."""
    if group.n < 2:
        raise GroupTooSmall(f"{group.n} ranks")
    counts = [[nbytes_per_pair] * group.n for _ in range(group.n)]
    return alltoallv(group, send, counts, counts_T(counts))


def counts_T(counts: Sequence[Sequence[int]]) -> List[List[int]]:
    n = len(counts)
    return [[counts[i][j] for i in range(n)] for j in range(n)]


def displs(splits: Sequence[int]) -> List[int]:
    out, acc = [], 0
    for s in splits:
        out.append(acc)
        acc += int(s)
    return out


def alltoallv(group: CommGroup, send: Sequence[np.ndarray], send_splits: Sequence[Sequence[int]],
              recv_splits: Sequence[Sequence[int]], elem_bytes: int = 1) -> List[np.ndarray]:
    """torch ``all_to_all_single`` semantics on bytes: ``send_splits[i][j]``
    elements go from rank i to rank j, landing at rank j's
    ``displs(recv_splits[j])[i]``.  Splits must agree pairwise."""
    n = group.n
    sb = [_as_bytes(s) for s in send]
    for i in range(n):
        for j in range(n):
            if send_splits[i][j] != recv_splits[j][i]:
                raise SimulationError(f"split mismatch {i}->{j}: {send_splits[i][j]} vs {recv_splits[j][i]}")
    out = [np.zeros(sum(recv_splits[j]) * elem_bytes, np.uint8) for j in range(n)]
    ops = []
    for s in range(1, n + 1):
        # rotated schedule j = (i + s) mod n; s == n is the self copy
        for i in range(n):
            j = (i + s) % n
            sd = displs(send_splits[i])[j] * elem_bytes
            rd = displs(recv_splits[j])[i] * elem_bytes
            ops.append((i, j, sb[i], sd, out[j], rd, send_splits[i][j] * elem_bytes))
    batch_p2p(group, ops)
    return out


def expected_alltoallv(send: Sequence[np.ndarray], send_splits: Sequence[Sequence[int]],
                       elem_bytes: int = 1) -> List[np.ndarray]:
    """Closed-form delivered bytes: recv_j = concat_i send_i[sdispl_i[j] : +c_ij]."""
    n = len(send)
    sb = [_as_bytes(s) for s in send]
    out = []
    for j in range(n):
        parts = []
        for i in range(n):
            d = displs(send_splits[i])[j] * elem_bytes
            parts.append(sb[i][d:d + send_splits[i][j] * elem_bytes])
        out.append(np.concatenate(parts) if parts else np.zeros(0, np.uint8))
    return out
