"""Pin the oracle's restated DES engine and endpoint rule against the
reference code's own behaviour (fixtures made by tests/golden/make_golden.py
from /root/reference/pkg/src/ccsim/netsim/{engine,topology}.py)."""
import json
import os

import pytest

from oracle.des import SchedulingInPast, SimulationError, Simulator
from oracle.netsim import closest_port, second_port

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_netsim.json")))


def test_fifo_same_time_order():  # engine.py:89-91, G34
    sim = Simulator()
    order = []
    for name, t in [("a", 5), ("b", 5), ("c", 7), ("d", 3), ("e", 5)]:
        sim.schedule(t, lambda n=name: order.append([n, sim.now]))
    sim.run_until(6)
    mid = sim.now
    sim.run()
    assert order == GOLD["fifo"]["order"]
    assert mid == GOLD["fifo"]["clock_after_run_until_6"]
    assert sim.now == GOLD["fifo"]["final"]


def test_scheduling_in_past():  # engine.py:87-88, 102-103, G33
    sim = Simulator()
    sim.schedule(6, lambda: None)
    sim.run()
    with pytest.raises(SchedulingInPast) as e:
        sim.schedule(2, lambda: None)
    assert str(e.value) == GOLD["past"]
    with pytest.raises(SchedulingInPast) as e:
        sim.run_until(1)
    assert str(e.value) == GOLD["past_run"]


def test_run_until_empty():  # engine.py:110, G35
    assert Simulator().run_until(100) == GOLD["empty_run_until"]


def test_cancel_and_pending():  # engine.py:32-33, 106-107, 127-128
    sim = Simulator()
    fired = []
    hs = [sim.schedule(10 * i, lambda i=i: fired.append(i)) for i in range(10)]
    for i in (1, 4, 7):
        hs[i].cancel()
    assert sim.pending() == GOLD["pending_after_cancel"]
    sim.run()
    assert fired == GOLD["fired_after_cancel"]


def test_event_budget_off_by_one():  # engine.py:113-125, SURVEY Appendix B6
    sim = Simulator()
    cnt = [0]

    def chain():
        cnt[0] += 1
        sim.after(1, chain)

    sim.schedule(0, chain)
    with pytest.raises(SimulationError) as e:
        sim.run(max_events=100)
    assert str(e.value) == GOLD["budget"]["msg"]
    assert cnt[0] == GOLD["budget"]["executed"]


def test_trace_hash_matches_reference():  # engine.py:36-69, G36
    sim = Simulator()
    for i, t in enumerate(GOLD["trace"]["times"]):
        sim.schedule(t, lambda i=i: sim.emit("ev", f"s{i % 7}", f"d{i}"))
    sim.run()
    assert sim.trace.lines()[:5] == GOLD["trace"]["first"]
    assert len(sim.trace.records) == GOLD["trace"]["n"]
    assert len(sim.trace.filter(subject="s3")) == GOLD["trace"]["filter_s3"]
    assert sim.trace.sha256() == GOLD["trace"]["sha256"]


def test_primary_backup_endpoint_rule():  # topology.py:140-151, G39
    assert [[closest_port(9, g), second_port(9, g)] for g in range(8)] == GOLD["nic_8x9"]
    assert [[closest_port(2, g), second_port(2, g)] for g in range(8)] == GOLD["nic_8x2"]
    with pytest.raises(SimulationError) as e:
        second_port(1, 0)
    assert str(e.value) == GOLD["nic_single"]


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted (GPU box)")
def test_live_reference_engine_randomised():
    """Where the reference is mounted, compare the two engines on random
    schedules including cancellations and run_until boundaries."""
    import random
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from ccsim.netsim import engine as ref
    for seed in range(20):
        rnd = random.Random(seed)
        a, b = ref.Simulator(), Simulator()
        for sim in (a, b):
            r2 = random.Random(seed)
            hs = []
            for i in range(200):
                hs.append(sim.schedule(r2.randrange(0, 1000), lambda i=i, sim=sim: sim.emit("e", str(i), "")))
            for i in range(0, 200, 7):
                hs[i].cancel()
            sim.run_until(r2.randrange(0, 1000))
            sim.run()
        assert a.trace.sha256() == b.trace.sha256()
        assert a.now == b.now
        del rnd
