"""Verb layer of the oracle (test infrastructure only).

Restates SPEC.md:121-204 (the reference has no code for it):

* ``MemoryRegion`` — only registered regions transfer;
  here it also carries the real bytes (a numpy uint8 view), which the
  reference deliberately does not.
* ``WorkRequest`` / ``WorkCompletion`` — ω(M), t1 at post, t2 at completion,
  status Success | RetryExceeded | Flushed.
* ``QueuePair`` — Primary | Backup role, Init | Connected | Error state, FIFO
  send and recv queues, IB timeout exponent and retry count
  (SPEC.md:138-143).  A QP transmits its send queue one WR at a time (RC
  ordering); several QPs share links through max-min.
* ``CompletionQueue`` — FIFO, capacity 4096, overflow is fatal
  (SPEC.md:144-147, 195).
* ``post_send`` / ``post_recv`` / ``poll_cq`` / ``retry_timeout``
  (SPEC.md:150-185).  t2 - t1 = serialization + 2 x propagation delay, the
  ack modelled as one extra delay.  A WR that cannot
  progress because its path is Down yields a RetryExceeded WC after
  ``retry_timeout`` and moves the QP to Error, flushing the rest
  (SPEC.md:158, 167, 185).
* CTS is a zero-payload WR direction.
"""
from __future__ import annotations

import enum
import itertools
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Deque, List, Optional

import numpy as np

from .des import SimulationError, Simulator
from .netsim import Link, Network


class QpInErrorState(SimulationError):
    """Post on a QP in Error."""


class UnregisteredRegion(SimulationError):
    """Post referencing an unregistered region."""


class WcStatus(enum.Enum):
    SUCCESS = "Success"
    RETRY_EXCEEDED = "RetryExceeded"
    FLUSHED = "Flushed"


class QpState(enum.Enum):
    INIT = "Init"
    CONNECTED = "Connected"
    ERROR = "Error"


class Direction(enum.Enum):
    SEND = "Send"
    RECV = "Recv"
    CTS = "Cts"


@dataclass(eq=False)
class MemoryRegion:
    rid: int
    owner: int
    data: np.ndarray  # uint8
    kind: str = "ApplicationBuffer"  # | ChunkBuffer
    registered: bool = True

    @property
    def length(self) -> int:
        return int(self.data.nbytes)


@dataclass(eq=False)
class WorkRequest:
    wr_id: int
    direction: Direction
    region: Optional[MemoryRegion]
    offset: int
    length: int
    t1: int = -1
    tag: object = None  # chunk index, carried to the completion


@dataclass
class WorkCompletion:
    wr_id: int
    status: WcStatus
    t2: int
    bytes: int
    tag: object = None
    qp_id: int = -1


class CompletionQueue:
    def __init__(self, capacity: int = 4096):
        self.capacity = capacity
        self.entries: Deque[WorkCompletion] = deque()
        self.listeners: List[Callable[[], None]] = []

    def push(self, wc: WorkCompletion) -> None:
        if len(self.entries) >= self.capacity:
            raise SimulationError("completion queue overflow")
        self.entries.append(wc)
        for cb in list(self.listeners):
            cb()

    def poll(self, max_entries: int) -> List[WorkCompletion]:
        """poll_cq: up to ``max_entries`` WCs in FIFO order."""
        if max_entries < 1:
            raise SimulationError("poll_cq max must be >= 1")
        out = []
        while self.entries and len(out) < max_entries:
            out.append(self.entries.popleft())
        return out


def retry_timeout_ns(timeout_exponent: int, retry_count: int) -> int:
    """(4.096 µs x 2^exp) x (retry + 1) in ns."""
    return 4096 * (1 << timeout_exponent) * (retry_count + 1)


_qp_ids = itertools.count()


class QueuePair:
    """One end-to-end RC connection (sender side and receiver side share the
    object: the oracle drives both ends from one event loop)."""

    def __init__(self, verbs: "Verbs", path: List[Link], role: str, send_cq: CompletionQueue,
                 recv_cq: CompletionQueue, timeout_exponent: int, retry_count: int):
        self.verbs = verbs
        self.qp_id = next(_qp_ids)
        self.path = path
        self.role = role  # "Primary" | "Backup"
        self.state = QpState.CONNECTED
        self.send_cq = send_cq
        self.recv_cq = recv_cq
        self.timeout_exponent = timeout_exponent
        self.retry_count = retry_count
        self.send_queue: Deque[WorkRequest] = deque()
        self.recv_queue: Deque[WorkRequest] = deque()
        self._flow = None
        self._retry_timer = None
        self._stalled_since: Optional[int] = None

    # -- helpers ----------------------------------------------------------
    @property
    def path_up(self) -> bool:
        return all(l.up for l in self.path)

    def retry_timeout(self) -> int:
        return retry_timeout_ns(self.timeout_exponent, self.retry_count)

    def reset(self) -> None:
        """Error -> Connected (re-created QP; used before a switch back)."""
        self.state = QpState.CONNECTED
        self._stalled_since = None


class Verbs:
    """Owns QPs over one ``Network``; all calls happen on the event loop."""

    def __init__(self, sim: Simulator, net: Network):
        self.sim = sim
        self.net = net
        self._wr_ids = itertools.count(1)
        self.qps: List[QueuePair] = []
        net.link_listeners.append(self._on_link_change)

    def new_wr_id(self) -> int:
        return next(self._wr_ids)

    def create_qp(self, path: List[Link], role: str, send_cq: CompletionQueue, recv_cq: CompletionQueue,
                  timeout_exponent: int = 18, retry_count: int = 7) -> QueuePair:
        qp = QueuePair(self, path, role, send_cq, recv_cq, timeout_exponent, retry_count)
        self.qps.append(qp)
        return qp

    # -- posting ---------------------------------------------
    def post_send(self, qp: QueuePair, wr: WorkRequest) -> None:
        if qp.state == QpState.ERROR:
            raise QpInErrorState(f"qp {qp.qp_id}")
        if wr.direction != Direction.CTS and (wr.region is None or not wr.region.registered):
            raise UnregisteredRegion(str(wr.wr_id))
        if wr.region is not None and wr.offset + wr.length > wr.region.length:
            raise SimulationError("WR exceeds its region")
        wr.t1 = self.sim.now
        qp.send_queue.append(wr)
        if qp._flow is None:
            self._start_head(qp)

    def post_recv(self, qp: QueuePair, wr: WorkRequest) -> None:
        if qp.state == QpState.ERROR:
            raise QpInErrorState(f"qp {qp.qp_id}")
        if wr.region is None or not wr.region.registered:
            raise UnregisteredRegion(str(wr.wr_id))
        wr.t1 = self.sim.now
        qp.recv_queue.append(wr)

    # -- transmission --------------------------------------------------------------
    def _start_head(self, qp: QueuePair) -> None:
        if not qp.send_queue or qp.state != QpState.CONNECTED:
            return
        wr = qp.send_queue[0]
        qp._flow = self.net.start_flow(qp.path, wr.length, lambda t, qp=qp, wr=wr: self._delivered(qp, wr),
                                       on_sent=lambda t, qp=qp, wr=wr: self._sent(qp, wr))
        self._check_stall(qp)

    def _sent(self, qp: QueuePair, wr: WorkRequest) -> None:
        """Last byte left: the QP moves on to its next WR (RC in-order)."""
        if qp._flow is None or not qp.send_queue or qp.send_queue[0] is not wr:
            return
        qp.send_queue.popleft()
        qp._flow = None
        self._cancel_retry(qp)
        qp._in_propagation = getattr(qp, "_in_propagation", 0) + 1
        self._start_head(qp)

    def _delivered(self, qp: QueuePair, wr: WorkRequest) -> None:
        """Last byte + one delay has arrived at the receiver."""
        qp._in_propagation -= 1
        if qp.state == QpState.ERROR:
            return  # QP flushed while the bytes were in flight: dropped
        if wr.direction != Direction.CTS:
            # consume the matching recv WR in FIFO order and place the bytes
            if not qp.recv_queue:
                raise SimulationError(f"qp {qp.qp_id}: message arrived with no posted recv (RNR)")
            rwr = qp.recv_queue.popleft()
            if rwr.length < wr.length:
                raise SimulationError("recv WR shorter than message")
            src = wr.region.data[wr.offset:wr.offset + wr.length]
            rwr.region.data[rwr.offset:rwr.offset + wr.length] = src
            qp.recv_cq.push(WorkCompletion(rwr.wr_id, WcStatus.SUCCESS, self.sim.now, wr.length, rwr.tag, qp.qp_id))
        delay = sum(l.delay_ns for l in qp.path)
        # ack travels back one propagation delay
        self.sim.after(delay, lambda: qp.state != QpState.ERROR and qp.send_cq.push(
            WorkCompletion(wr.wr_id, WcStatus.SUCCESS, self.sim.now, wr.length, wr.tag, qp.qp_id)))

    # -- failure: retry budget, flush ------------------------------
    def _check_stall(self, qp: QueuePair) -> None:
        if qp._flow is not None and not qp.path_up:
            if qp._retry_timer is None:
                qp._stalled_since = self.sim.now
                qp._retry_timer = self.sim.after(qp.retry_timeout(), lambda: self._retry_exceeded(qp))
        else:
            self._cancel_retry(qp)

    def _cancel_retry(self, qp: QueuePair) -> None:
        if qp._retry_timer is not None:
            qp._retry_timer.cancel()
            qp._retry_timer = None
            qp._stalled_since = None

    def _on_link_change(self, link: Link) -> None:
        for qp in self.qps:
            if link in qp.path:
                self._check_stall(qp)

    def _retry_exceeded(self, qp: QueuePair) -> None:
        qp._retry_timer = None
        if qp._flow is None or not qp.send_queue:
            return
        head = qp.send_queue[0]
        qp.send_cq.push(WorkCompletion(head.wr_id, WcStatus.RETRY_EXCEEDED, self.sim.now, 0, head.tag, qp.qp_id))
        self.flush(qp, skip_head=True)

    def flush(self, qp: QueuePair, skip_head: bool = False) -> None:
        """Move to Error; every outstanding WR completes Flushed."""
        qp.state = QpState.ERROR
        if qp._flow is not None:
            self.net.cancel_flow(qp._flow)
            qp._flow = None
        self._cancel_retry(qp)
        first = True
        while qp.send_queue:
            wr = qp.send_queue.popleft()
            if first and skip_head:
                first = False
                continue
            first = False
            qp.send_cq.push(WorkCompletion(wr.wr_id, WcStatus.FLUSHED, self.sim.now, 0, wr.tag, qp.qp_id))
        while qp.recv_queue:
            wr = qp.recv_queue.popleft()
            qp.recv_cq.push(WorkCompletion(wr.wr_id, WcStatus.FLUSHED, self.sim.now, 0, wr.tag, qp.qp_id))

    # -- CTS probe ------------------------------------------------
    def probe(self, qp_path: List[Link], timeout_ns: int, on_result: Callable[[bool], None]) -> None:
        """Zero-payload round trip on a path: Success after 2 x delay if the path
        stays Up, failure after ``timeout_ns`` otherwise."""
        delay = sum(l.delay_ns for l in qp_path)
        if all(l.up for l in qp_path):
            self.sim.after(2 * delay, lambda: on_result(True))
        else:
            self.sim.after(timeout_ns, lambda: on_result(all(l.up for l in qp_path) and False))
