"""Fluid network model of the oracle (test infrastructure only).

Restates the reference's link / path model and the SPEC's netsim operations:

* ``Link`` — directed, capacity in bits/s, integer-ns propagation delay, an
  up/down state and a delivered-bytes counter (topology.py:38-50,
  SPEC.md:49-52).
* ``closest_port`` / ``second_port`` — the primary / backup endpoint rule:
  minimal |port - gpu| with a lowest-index tie-break, and the next-closest
  distinct port for the backup; fewer than two ports raises
  (topology.py:140-151).  On B200 the "ports" are copy paths: port 0 is the
  copy-engine path, port 1 the SM-kernel path, port 2.. relay GPUs.
* ``allocate_bandwidth`` — max-min fair water-filling over the links flows
  share; every link's allocated sum stays within capacity.
* ``apply_fault`` / ``FaultScript`` — time-ordered Down/Up of a named port;
  flows over a Down link deliver 0 bytes and resume on Up (SPEC.md:53-56,
  90-98).  Link-layer detection latency is 0: the transport discovers a
  failure only through its own timeouts.
* ``nvswitch_box`` — the B200 box the product runs on: every GPU has its own
  900 GB/s egress and ingress port to the NVSwitch, uniform to every peer
  (SURVEY.md §8e, Appendix B4 explains why the reference's single shared
  intra-host link, topology.py:110-112 / 158-159, cannot express this).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .des import SimulationError, Simulator


class UnknownPort(SimulationError):
    """A fault or lookup names a port that does not exist (topology.py:20-21)."""


@dataclass(eq=False)
class Link:
    name: str
    capacity_bps: float
    delay_ns: int
    up: bool = True
    bytes_delivered: int = 0

    @property
    def bytes_per_ns(self) -> float:
        return self.capacity_bps / 8e9


def closest_port(n_ports: int, gpu: int) -> int:
    """Primary endpoint: argmin |p - gpu|, lowest index on ties (topology.py:140-143)."""
    return min(range(n_ports), key=lambda p: (abs(p - gpu), p))


def second_port(n_ports: int, gpu: int) -> int:
    """Backup endpoint: next-closest distinct port (topology.py:145-151)."""
    if n_ports < 2:
        raise SimulationError("backup NIC requires at least two ports per host")
    first = closest_port(n_ports, gpu)
    return min((p for p in range(n_ports) if p != first), key=lambda p: (abs(p - gpu), p))


def relay_gpu(n_gpus: int, src: int, dst: int, busy: Sequence[int] = ()) -> int:
    """Relay GPU for the two-hop backup path: the lowest-index GPU that is not an
    endpoint (the lowest-index tie-break of topology.py:143, 151), skipping
    relays already carrying a failed pair when another is free."""
    cands = [g for g in range(n_gpus) if g not in (src, dst)]
    if not cands:
        raise SimulationError("relay path needs a third GPU")
    free = [g for g in cands if g not in busy]
    return (free or cands)[0]


@dataclass(eq=False)
class Flow:
    """Bytes in flight over a path."""

    fid: int
    path: List[Link]
    remaining: float
    on_delivered: Callable[[int], None]
    start: int
    rate: float = 0.0  # bytes per ns
    last_update: int = 0
    done_event: object = None


def allocate_bandwidth(flows: Sequence[Flow]) -> Dict[int, float]:
    """Max-min fair rates in bytes/ns by progressive filling.

    Flows that cross a Down link get 0."""
    rates: Dict[int, float] = {}
    active = [f for f in flows if all(l.up for l in f.path)]
    for f in flows:
        if f not in active:
            rates[f.fid] = 0.0
    residual = {}
    users: Dict[int, List[Flow]] = {}
    for f in active:
        for l in f.path:
            residual[id(l)] = l.bytes_per_ns
            users.setdefault(id(l), []).append(f)
    unfrozen = set(f.fid for f in active)
    while unfrozen:
        # bottleneck: the link with the smallest fair share among unfrozen flows
        best = None
        for lid, fl in users.items():
            n = sum(1 for f in fl if f.fid in unfrozen)
            if n == 0:
                continue
            share = residual[lid] / n
            if best is None or share < best[0] - 1e-15:
                best = (share, lid)
        if best is None:
            break
        share, lid = best
        for f in users[lid]:
            if f.fid in unfrozen:
                rates[f.fid] = share
                unfrozen.discard(f.fid)
                for l in f.path:
                    residual[id(l)] -= share
    return rates


class Network:
    """Fluid flows over links on the DES clock; rates recomputed on every
    flow-set or link-state change."""

    def __init__(self, sim: Simulator):
        self.sim = sim
        self.flows: Dict[int, Flow] = {}
        self.ports: Dict[str, Link] = {}
        self._next = 0
        self.link_listeners: List[Callable[[Link], None]] = []

    def add_port(self, link: Link) -> Link:
        self.ports[link.name] = link
        return link

    def _advance(self) -> None:
        now = self.sim.now
        for f in self.flows.values():
            dt = now - f.last_update
            if dt > 0 and f.rate > 0:
                moved = min(f.remaining, f.rate * dt)
                f.remaining -= moved
            f.last_update = now

    def _reallocate(self) -> None:
        rates = allocate_bandwidth(list(self.flows.values()))
        for f in list(self.flows.values()):
            f.rate = rates.get(f.fid, 0.0)
            if f.done_event is not None:
                f.done_event.cancel()
                f.done_event = None
            if f.rate > 0:
                # serialization ends when the last byte leaves; delivery one
                # propagation delay later
                t_end = self.sim.now + max(0, math.ceil(f.remaining / f.rate - 1e-9))
                f.done_event = self.sim.schedule(t_end, lambda f=f: self._finish(f))

    def _finish(self, f: Flow) -> None:
        self._advance()
        f.remaining = 0.0
        del self.flows[f.fid]
        delay = sum(l.delay_ns for l in f.path)
        for l in f.path:
            l.bytes_delivered += f.total
        self._reallocate()
        if f.on_sent is not None:
            f.on_sent(self.sim.now)
        self.sim.after(delay, lambda: f.on_delivered(self.sim.now))

    def start_flow(self, path: List[Link], nbytes: int, on_delivered: Callable[[int], None],
                   on_sent: Optional[Callable[[int], None]] = None) -> Flow:
        """Start a flow; ``on_sent`` fires when the last byte leaves (the QP may
        start its next WR), ``on_delivered`` one propagation delay later."""
        self._advance()
        f = Flow(self._next, list(path), float(nbytes), on_delivered, self.sim.now, last_update=self.sim.now)
        f.total = int(nbytes)
        f.on_sent = on_sent
        self._next += 1
        self.flows[f.fid] = f
        self._reallocate()
        return f

    def cancel_flow(self, f: Flow) -> None:
        if f.fid in self.flows:
            self._advance()
            if f.done_event is not None:
                f.done_event.cancel()
            del self.flows[f.fid]
            self._reallocate()

    def set_link(self, link: Link, up: bool) -> None:
        """apply_fault at the current clock."""
        self._advance()
        link.up = up
        self._reallocate()
        for cb in list(self.link_listeners):
            cb(link)

    def apply_fault(self, port: str, up: bool, at: int) -> None:
        if port not in self.ports:
            raise UnknownPort(port)
        link = self.ports[port]
        self.sim.schedule(at, lambda: self.set_link(link, up))


@dataclass
class FaultScript:
    """Time-ordered (t_ns, port, up) entries; Down/Up alternate per port
    (SPEC.md:53-56)."""

    entries: List[Tuple[int, str, bool]] = field(default_factory=list)

    def validate(self) -> None:
        last_t = -1
        state: Dict[str, bool] = {}
        for t, port, up in self.entries:
            if t < last_t:
                raise SimulationError("fault script entries must be sorted by time")
            if state.get(port, True) == up:
                raise SimulationError(f"Down/Up must alternate for port {port}")
            state[port] = up
            last_t = t

    def install(self, net: Network) -> None:
        self.validate()
        for t, port, up in self.entries:
            net.apply_fault(port, up, t)


def nvswitch_box(sim: Simulator, n_gpus: int, nvlink_gbps: float = 900.0, delay_ns: int = 1000,
                 n_paths: int = 2):
    """B200 box: per-GPU egress/ingress ports at ``nvlink_gbps`` GB/s per
    direction, plus one zero-cost fault-domain link per (src, dst, path) so a
    single directed path can be brought Down ("RNIC port
    down" -> gate on the primary copy path)."""
    net = Network(sim)
    cap = nvlink_gbps * 8e9
    egress = [net.add_port(Link(f"gpu{g}.tx", cap, 0)) for g in range(n_gpus)]
    ingress = [net.add_port(Link(f"gpu{g}.rx", cap, 0)) for g in range(n_gpus)]
    gates: Dict[Tuple[int, int, int], Link] = {}
    for s in range(n_gpus):
        for d in range(n_gpus):
            for p in range(n_paths):
                gates[(s, d, p)] = net.add_port(Link(path_port(s, d, p), 1e30, delay_ns))

    def path(s: int, d: int, p: int) -> List[Link]:
        if s == d:
            return [gates[(s, d, p)]]
        return [egress[s], gates[(s, d, p)], ingress[d]]

    return net, path


def path_port(src: int, dst: int, path: int) -> str:
    return f"{src}->{dst}.p{path}"
