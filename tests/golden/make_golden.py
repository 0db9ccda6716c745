"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
It imports the reference's discrete-event engine and topology
(/root/reference/pkg/src/ccsim/netsim/{engine,topology}.py), drives them
through deterministic scenarios and records their observable behaviour in
tests/golden/reference_netsim.json.  The oracle (oracle/des.py,
oracle/netsim.py) is checked against this file by tests/test_oracle_pinning.py,
which also works on the GPU box where /root/reference does not exist.
"""
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"


def main():
    sys.path.insert(0, REF)
    from ccsim.netsim import engine, topology  # noqa: E402

    out = {}

    # 1. same-time FIFO order + clock values (engine.py:85-111)
    sim = engine.Simulator()
    order = []
    for name, t in [("a", 5), ("b", 5), ("c", 7), ("d", 3), ("e", 5)]:
        sim.schedule(t, lambda n=name: order.append((n, sim.now)))
    sim.run_until(6)
    mid = sim.now
    sim.run()
    out["fifo"] = {"order": order, "clock_after_run_until_6": mid, "final": sim.now}

    # 2. SchedulingInPast message (engine.py:87-88)
    sim = engine.Simulator()
    sim.schedule(6, lambda: None)
    sim.run()
    try:
        sim.schedule(2, lambda: None)
        out["past"] = None
    except engine.SchedulingInPast as e:
        out["past"] = str(e)
    try:
        sim.run_until(1)
        out["past_run"] = None
    except engine.SchedulingInPast as e:
        out["past_run"] = str(e)

    # 3. run_until on empty queue (engine.py:110)
    sim = engine.Simulator()
    out["empty_run_until"] = sim.run_until(100)

    # 4. cancellation + pending (engine.py:32-33, 106-107, 127-128)
    sim = engine.Simulator()
    fired = []
    hs = [sim.schedule(10 * i, lambda i=i: fired.append(i)) for i in range(10)]
    for i in (1, 4, 7):
        hs[i].cancel()
    out["pending_after_cancel"] = sim.pending()
    sim.run()
    out["fired_after_cancel"] = fired

    # 5. event budget off-by-one (engine.py:113-125)
    sim = engine.Simulator()
    cnt = [0]

    def chain():
        cnt[0] += 1
        sim.after(1, chain)

    sim.schedule(0, chain)
    try:
        sim.run(max_events=100)
    except engine.SimulationError as e:
        out["budget"] = {"msg": str(e), "executed": cnt[0]}

    # 6. trace lines + sha256 of a seeded random workload (engine.py:36-69)
    rnd = random.Random(1234)
    sim = engine.Simulator()
    for i in range(500):
        t = rnd.randrange(0, 10_000)
        sim.schedule(t, lambda i=i: sim.emit("ev", f"s{i % 7}", f"d{i}"))
    sim.run()
    out["trace"] = {"sha256": sim.trace.sha256(), "first": list(sim.trace.lines())[:5], "n": len(sim.trace.records),
                    "filter_s3": len(sim.trace.filter(subject="s3"))}
    # the seeded schedule itself, so the oracle can replay it without `random` drift
    rnd = random.Random(1234)
    out["trace"]["times"] = [rnd.randrange(0, 10_000) for _ in range(500)]

    # 7. topology primary / backup endpoint choice (topology.py:140-151)
    topo = topology.Topology(topology.TopologyConfig(hosts=1, gpus_per_host=8, nics_per_host=9, leaf_switches=9))
    out["nic_8x9"] = [[topo.closest_nic(0, g), topo.second_nic(0, g)] for g in range(8)]
    topo = topology.Topology(topology.TopologyConfig(hosts=1, gpus_per_host=8, nics_per_host=2, leaf_switches=2))
    out["nic_8x2"] = [[topo.closest_nic(0, g), topo.second_nic(0, g)] for g in range(8)]
    topo = topology.Topology(topology.TopologyConfig(hosts=1, gpus_per_host=2, nics_per_host=1, leaf_switches=1))
    try:
        topo.second_nic(0, 0)
        out["nic_single"] = None
    except engine.SimulationError as e:
        out["nic_single"] = str(e)
    # intra-host path collapses onto one shared link
    topo = topology.Topology(topology.TopologyConfig(hosts=2, gpus_per_host=8, nics_per_host=2))
    out["intra_path"] = [l.id for l in topo.path_between((0, 0), (0, 5))]
    out["hops"] = [topo.hop_count((0, 1), (1, 0)), topo.hop_count((0, 1), (1, 1)), topo.hop_count((0, 1), (0, 3))]

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_netsim.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
