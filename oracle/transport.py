"""Transport layer of the oracle (test infrastructure only).

Restates SPEC.md:206-297 — chunked P2P with the six progress pointers of
PAPER.md Fig. 6 and primary-backup failover with breakpoint retransmission:

* ``PipelineMode`` — StagedCopy adds a BufferCopy stage per chunk, ZeroCopy
  sends the application buffer directly.
* ``SenderPointers`` / ``ReceiverPointers`` — posted >= transmitted >= acked
  and posted >= received >= done.
* ``Connection`` — primary + backup QP, active role, delta, last WR issue
  time.
* ``send_message`` chunks a message (default 4 MiB), advances
  posted on preparation, transmitted on post_send, acked on a Success WC
  (SPEC.md:228-236).  ``length == 0`` raises ``ZeroLengthMessage``.
* ``on_wc``, ``check_receiver_timeout`` with the CTS probe
  that tells an innocent stall from a dead link,
  ``switch_qp`` with the receiver-driven retreat and
  ``monitor_failed_link``.
* Both QPs dead -> ``ConnectionFailed``.

Beyond the SPEC, the oracle moves the real bytes so the B200 path's delivered
bytes can be compared to it, and it keeps the per-transfer event log
``time_ns, conn_id, role, event, chunk_index``.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from .des import SimulationError, Simulator
from .verbs import (CompletionQueue, Direction, MemoryRegion, QpState, QueuePair, Verbs, WcStatus,
                    WorkCompletion, WorkRequest, retry_timeout_ns)

MiB = 1 << 20
DEFAULT_CHUNK = 4 * MiB


class ZeroLengthMessage(SimulationError):
    """send_message with length 0."""


class ConnectionFailed(SimulationError):
    """Primary and backup both dead."""


class UnknownWr(SimulationError):
    """A WC for a chunk already acknowledged, or for no outstanding WR."""


class TargetQpDead(SimulationError):
    """switch_qp towards a QP that is not Connected."""


class Action(enum.Enum):
    NO_ACTION = "NoAction"
    TRIGGER_SWITCH = "TriggerSwitch"


class Mode(enum.Enum):
    STAGED_COPY = "StagedCopy"
    ZERO_COPY = "ZeroCopy"


@dataclass
class PipelineMode:
    """Stage costs per chunk in ns.  ZeroCopy has no
    BufferCopy stage by construction."""

    mode: Mode = Mode.ZERO_COPY
    prep_ns: int = 0
    buffer_copy_ns: int = 0

    def __post_init__(self):
        if self.prep_ns < 0 or self.buffer_copy_ns < 0:
            raise SimulationError("stage costs must be >= 0")
        if self.mode == Mode.ZERO_COPY:
            self.buffer_copy_ns = 0


@dataclass
class SenderPointers:
    posted: int = 0
    transmitted: int = 0
    acked: int = 0

    def check(self, total: int) -> None:
        assert 0 <= self.acked <= self.transmitted <= self.posted <= total, self


@dataclass
class ReceiverPointers:
    posted: int = 0
    received: int = 0
    done: int = 0

    def check(self, total: int) -> None:
        assert 0 <= self.done <= self.received <= self.posted <= total, self


def switch_pointers(receiver: ReceiverPointers, sender: SenderPointers):
    """The pointer part of switch_qp: the receiver retreats
    received to done and pushes done; the sender sets acked := done and
    posted := transmitted := acked.  Returns the chunk retransmission resumes
    at.  G14: receiver {10, 8, 6}, sender {10, 9, 5} -> 6 everywhere."""
    receiver.received = receiver.done
    sender.acked = receiver.done
    sender.posted = sender.acked
    sender.transmitted = sender.acked
    return sender.acked


def chunk_bounds(length: int, chunk: int, k: int):
    off = k * chunk
    return off, min(chunk, length - off)


def n_chunks(length: int, chunk: int) -> int:
    return (length + chunk - 1) // chunk


@dataclass
class MessageRecord:
    """Monitor tap: one per Success WC at the sender."""

    wr_id: int
    size: int
    t1: int
    t2: int
    chunk: int = -1
    path: str = "Primary"


class Connection:
    """A directed sender -> receiver connection with primary and backup QPs
    (SPEC.md:222-225).  One transfer at a time, like a NCCL P2P channel."""

    def __init__(self, sim: Simulator, verbs: Verbs, primary_path, backup_path, conn_id: str = "c0",
                 chunk_size: int = DEFAULT_CHUNK, timeout_exponent: int = 18, retry_count: int = 7,
                 delta_ns: Optional[int] = None, window: int = 8, probe_period_ns: int = 500_000_000,
                 mode: Optional[PipelineMode] = None, qp_per_connection: int = 1,
                 on_record: Optional[Callable[[MessageRecord], None]] = None, cts_timeout_ns: int = 0):
        self.sim = sim
        self.verbs = verbs
        self.conn_id = conn_id
        self.chunk_size = chunk_size
        self.window = window
        self.mode = mode or PipelineMode()
        self.send_cq = CompletionQueue()
        self.recv_cq = CompletionQueue()
        # qp_per_connection > 1 stripes chunks round-robin
        self.primary = [verbs.create_qp(primary_path, "Primary", self.send_cq, self.recv_cq, timeout_exponent,
                                        retry_count) for _ in range(qp_per_connection)]
        self.backup = [verbs.create_qp(backup_path, "Backup", self.send_cq, self.recv_cq, timeout_exponent,
                                       retry_count) for _ in range(qp_per_connection)]
        self.active = "Primary"
        max_delay = max(sum(l.delay_ns for l in primary_path), sum(l.delay_ns for l in backup_path))
        # delta default: retry_timeout + 2 x max propagation delay
        self.delta_ns = delta_ns if delta_ns is not None else (
            retry_timeout_ns(timeout_exponent, retry_count) + 2 * max_delay)
        self.probe_period_ns = probe_period_ns
        self.cts_timeout_ns = cts_timeout_ns  # CTS probe deadline; 0 = the QP retry timeout
        self.on_record = on_record
        self.records: List[MessageRecord] = []
        self.switches: List[tuple] = []  # (time, direction, resume_chunk)
        self.delivered_sequence: List[int] = []  # chunk indices in the order done advanced
        self.failed: Optional[str] = None
        self.send_cq.listeners.append(self._drain_send_cq)
        self.recv_cq.listeners.append(self._drain_recv_cq)
        self.xfer = None
        self._probe_timer = None
        self._rx_timer = None
        self._cts_out = False

    # -- helpers -------------------------------------------------------------------
    def qps(self, role: Optional[str] = None) -> List[QueuePair]:
        return self.primary if (role or self.active) == "Primary" else self.backup

    def log(self, role: str, event: str, chunk: int = -1) -> None:
        self.sim.emit("transport", self.conn_id, f"{role},{event},{chunk}")

    # -- send_message ---------------------------------------------
    def send_message(self, src: MemoryRegion, dst: MemoryRegion, length: int, src_off: int = 0, dst_off: int = 0,
                     ready_at: int = 0, on_complete: Optional[Callable[[], None]] = None) -> "Transfer":
        if length <= 0:
            raise ZeroLengthMessage(self.conn_id)
        if self.xfer is not None and not self.xfer.complete:
            raise SimulationError("connection busy")
        if all(q.state == QpState.ERROR for q in self.primary + self.backup):
            raise ConnectionFailed(self.conn_id)
        self.xfer = Transfer(self, src, dst, length, src_off, dst_off, ready_at, on_complete)
        self.xfer.start()
        return self.xfer

    # -- completions ---------------------------------------------------------------
    def _drain_send_cq(self) -> None:
        for wc in self.send_cq.poll(self.send_cq.capacity):
            if self.xfer is not None:
                act = self.on_wc(wc, "Sender")
                if act == Action.TRIGGER_SWITCH:
                    self.switch_qp("ToBackup" if self.active == "Primary" else "ToPrimary", trigger="sender-wc")

    def _drain_recv_cq(self) -> None:
        for wc in self.recv_cq.poll(self.recv_cq.capacity):
            if self.xfer is not None:
                self.on_wc(wc, "Receiver")

    def on_wc(self, wc: WorkCompletion, role: str) -> Action:
        """SPEC.md:237-245."""
        x = self.xfer
        active_ids = {q.qp_id for q in self.qps()}
        if wc.status == WcStatus.FLUSHED or wc.qp_id not in active_ids:
            return Action.NO_ACTION  # in-flight chunks of a dying QP
        if wc.status == WcStatus.RETRY_EXCEEDED:
            self.log(role, "retry_exceeded", wc.tag if wc.tag is not None else -1)
            return Action.TRIGGER_SWITCH
        k = wc.tag
        if role == "Sender":
            if k in x.acked_set or k is None:
                raise UnknownWr(f"duplicate Success for chunk {k}")
            x.acked_set.add(k)
            rec = MessageRecord(wc.wr_id, wc.bytes, x.wr_t1.get(wc.wr_id, wc.t2), wc.t2, k, self.active)
            self.records.append(rec)
            if self.on_record:
                self.on_record(rec)
            while x.s.acked in x.acked_set:
                x.s.acked += 1
            self.log("sender", "ack", k)
            x.pump()
            x.check_complete()
        else:
            x.last_progress = self.sim.now
            x.recv_set.add(k)
            while x.r.received in x.recv_set:
                x.r.received += 1
                # ZeroCopy: bytes already sit in the application buffer, so a
                # received chunk is done at once; StagedCopy would copy out here.
                x.r.done = x.r.received
                self.delivered_sequence.append(x.r.done - 1)
                self.log("receiver", "done", x.r.done - 1)
            x.post_recvs()
            x.check_complete()
        return Action.NO_ACTION

    # -- receiver watchdog ----------------------------------------
    def check_receiver_timeout(self, now: int, on_action: Optional[Callable[[Action], None]] = None) -> Action:
        """If nothing arrived for more than delta, probe the active QP with a
        CTS.  Returns NO_ACTION synchronously; the probe outcome is delivered
        through ``on_action`` (TriggerSwitch on a failed CTS)."""
        x = self.xfer
        if x is None or x.complete or now - x.last_progress <= self.delta_ns or self._cts_out:
            return Action.NO_ACTION
        qp = self.qps()[0]
        probed = self.active
        self._cts_out = True
        self.log("receiver", "cts_probe", x.r.done)

        def result(ok: bool):
            self._cts_out = False
            if x.complete or self.active != probed:
                return  # the connection moved on while the CTS was in flight
            if ok:
                self.log("receiver", "cts_ok", x.r.done)
                x.last_progress = self.sim.now
                if on_action:
                    on_action(Action.NO_ACTION)
            else:
                self.log("receiver", "cts_fail", x.r.done)
                if on_action:
                    on_action(Action.TRIGGER_SWITCH)
                self.switch_qp("ToBackup" if self.active == "Primary" else "ToPrimary", trigger="receiver-cts")

        self.verbs.probe(qp.path, self.cts_timeout_ns or qp.retry_timeout(), result)
        return Action.NO_ACTION

    def _arm_rx_watchdog(self) -> None:
        if self._rx_timer is not None:
            self._rx_timer.cancel()
        period = max(1, self.delta_ns // 2)

        def tick():
            self._rx_timer = None
            x = self.xfer
            if x is None or x.complete:
                return
            self.check_receiver_timeout(self.sim.now)
            self._arm_rx_watchdog()

        self._rx_timer = self.sim.after(period, tick)

    # -- switch_qp ------------------------------------------------
    def switch_qp(self, direction: str, trigger: str = "") -> None:
        target = "Backup" if direction == "ToBackup" else "Primary"
        if self.active == target:
            return
        x = self.xfer
        tq = self.qps(target)
        if direction == "ToBackup" and not all(l.up for l in tq[0].path):
            # backup unusable too: both dead
            self.failed = "both paths dead"
            self.log("receiver", "connection_failed", x.r.done if x else -1)
            raise ConnectionFailed(self.conn_id)
        for q in tq:
            if q.state == QpState.ERROR:
                q.reset()
        old = self.qps()
        self.active = target
        for q in old:
            if q.state != QpState.ERROR:
                self.verbs.flush(q)
        resume = switch_pointers(x.r, x.s) if x else 0
        if x:
            x.acked_set = set(range(resume))
            x.recv_set = set(range(resume))
            x.r.posted = resume
            x.last_progress = self.sim.now
        self.switches.append((self.sim.now, direction, resume, trigger))
        self.log("receiver", "switch_to_backup" if target == "Backup" else "switch_to_primary", resume)
        if x:
            # done == total: the retreat set acked := done, nothing to resend
            # — the acks still in flight on the old QP are flushed
            x.check_complete()
        if x and not x.complete:
            x.post_recvs()
            x.pump()
        if target == "Backup":
            self._arm_probe()

    def monitor_failed_link(self) -> None:
        """Probe the primary every period while on backup; on success switch
        back."""
        self._arm_probe()

    def _arm_probe(self) -> None:
        if self._probe_timer is not None:
            self._probe_timer.cancel()

        def probe():
            self._probe_timer = None
            if self.active != "Backup" or self.xfer is None or self.xfer.complete:
                return  # idle connections are probed again when the next transfer starts
            qp = self.primary[0]

            def result(ok: bool):
                if ok and self.active == "Backup":
                    if self.xfer is None or self.xfer.complete:
                        for q in self.primary:
                            q.reset()
                        self.active = "Primary"
                        self.switches.append((self.sim.now, "ToPrimary", -1, "probe"))
                        self.log("receiver", "switch_to_primary", -1)
                    else:
                        self.switch_qp("ToPrimary", trigger="probe")
                elif self.active == "Backup":
                    self._arm_probe()

            # a probe only answers if the path is up at send time and stays up
            # for the round trip; a Down path answers never (counted as fail)
            self.verbs.probe(qp.path, 1, result) if all(l.up for l in qp.path) else self._arm_probe()

        self._probe_timer = self.sim.after(self.probe_period_ns, probe)


class Transfer:
    """One message over a Connection: the sender's and the receiver's state
    machines driven by the WCs of the active QP set."""

    def __init__(self, conn: Connection, src: MemoryRegion, dst: MemoryRegion, length: int, src_off: int,
                 dst_off: int, ready_at: int, on_complete):
        self.conn = conn
        self.src, self.dst = src, dst
        self.length = length
        self.src_off, self.dst_off = src_off, dst_off
        self.total = n_chunks(length, conn.chunk_size)
        self.s = SenderPointers()
        self.r = ReceiverPointers()
        self.acked_set = set()
        self.recv_set = set()
        self.wr_t1 = {}
        self.ready_at = ready_at
        self.on_complete = on_complete
        self.complete = False
        self.last_progress = 0
        self._rr = 0
        self._prep_busy_until = 0

    def start(self) -> None:
        sim = self.conn.sim
        self.last_progress = sim.now
        self.post_recvs()
        self.conn._arm_rx_watchdog()
        if self.conn.active == "Backup":
            self.conn._arm_probe()
        sim.schedule(max(sim.now, self.ready_at), self.pump)

    def post_recvs(self) -> None:
        """Receiver keeps recv WRs posted for [received, total) on the active QPs."""
        c = self.conn
        qps = c.qps()
        while self.r.posted < self.total and self.r.posted < self.r.done + c.window:
            k = self.r.posted
            off, n = chunk_bounds(self.length, c.chunk_size, k)
            qp = qps[k % len(qps)]
            if qp.state == QpState.ERROR:
                return
            c.verbs.post_recv(qp, WorkRequest(c.verbs.new_wr_id(), Direction.RECV, self.dst, self.dst_off + off, n,
                                              tag=k))
            self.r.posted += 1

    def pump(self) -> None:
        """Sender: prepare and post chunks while the window allows."""
        c = self.conn
        sim = c.sim
        if self.complete or sim.now < self.ready_at:
            return
        qps = c.qps()
        # StagedCopy owns one chunk buffer: the next BufferCopy waits until the
        # previous chunk left it (acked), so copy and transmission serialise —
        # the regime in which the SPEC's 0.8x claim holds (B12).
        window = 1 if c.mode.mode == Mode.STAGED_COPY else c.window
        while self.s.posted < self.total and self.s.posted < self.s.acked + window:
            if any(q.state == QpState.ERROR for q in qps):
                return
            k = self.s.posted
            self.s.posted += 1
            c.log("sender", "post", k)
            stage = c.mode.prep_ns + c.mode.buffer_copy_ns
            if stage:
                # DataPreparation (+ BufferCopy in StagedCopy) is serial per chunk
                t = max(sim.now, self._prep_busy_until) + stage
                self._prep_busy_until = t
                epoch = c.active
                sim.schedule(t, lambda k=k, epoch=epoch: self._transmit(k, epoch))
            else:
                self._transmit(k, c.active)

    def _transmit(self, k: int, epoch: str) -> None:
        c = self.conn
        if c.active != epoch or k < self.s.acked or self.complete:
            return  # a switch happened while this chunk was being prepared
        qps = c.qps()
        qp = qps[k % len(qps)]
        if qp.state == QpState.ERROR:
            return
        off, n = chunk_bounds(self.length, c.chunk_size, k)
        wr = WorkRequest(c.verbs.new_wr_id(), Direction.SEND, self.src, self.src_off + off, n, tag=k)
        c.verbs.post_send(qp, wr)
        self.wr_t1[wr.wr_id] = wr.t1
        self.s.transmitted = max(self.s.transmitted, k + 1)
        c.log("sender", "transmit", k)

    def check_complete(self) -> None:
        if not self.complete and self.r.done == self.total and self.s.acked == self.total:
            self._finish()
        elif not self.complete and self.r.done == self.total:
            # wait for the last acks
            pass

    def _finish(self) -> None:
        self.complete = True
        self.conn.log("receiver", "complete", self.total)
        if self.on_complete:
            self.on_complete()

    def state(self):
        return dict(sender=dict(posted=self.s.posted, transmitted=self.s.transmitted, acked=self.s.acked),
                    receiver=dict(posted=self.r.posted, received=self.r.received, done=self.r.done),
                    total_chunks=self.total)
