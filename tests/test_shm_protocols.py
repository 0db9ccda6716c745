"""The control block's two cross-process protocols, driven on CPU (no GPU).

libiccl_b200.so exports self-test hooks (include/iccl_b200.h) that run the
product's own shared-memory code on caller-owned memory.  Here several
processes share one anonymous mapping, exactly as ranks share the
communicator's POSIX shm segment:

- the rendezvous entry of an ordered pair (SPEC.md:194's RTS / CTS): for
  every op exactly one side arrives second, claims the transfer and sees the
  other side's half of the same op — also across the 1024-entry ring's reuse;
- small-op routing: while a third process arms and disarms the pair (fault
  scripts, switch_qp), the sender and the receiver route every small op the
  same way (LL or rendezvous), or the op would hang on the GPU.
"""
import ctypes as C
import mmap
import multiprocessing as mp
import random
import time

import numpy as np
import pytest

from paper_2510_00991_b200._lib import lib

# the forked children only run the hooks on shared memory (no CUDA, no torch threads)
pytestmark = pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")


def _addr(buf, off=0):
    return C.addressof(C.c_char.from_buffer(buf, off))


def _rzv_side(shared, out, kind, n, seed):
    rng = random.Random(seed)
    entry = _addr(shared)
    res = np.frombuffer(out, dtype=np.int64).reshape(2, n, 2)
    other = C.c_uint64()
    for k in range(n):
        if rng.random() < 0.3:
            for _ in range(rng.randint(1, 200)):
                pass
        if rng.random() < 0.02:
            time.sleep(0.0005)
        if kind == 0 and k == n // 2:
            time.sleep(0.2)  # the side that started first pauses: the other overtakes, both orders occur
        r = lib.iccl_selftest_rzv_post(entry + (k % 1024) * lib.iccl_selftest_rzv_bytes(), kind, k,
                                       1000 + 7 * k + (k % 3), C.byref(other))
        res[kind, k, 0] = r
        res[kind, k, 1] = other.value if r == 1 else -1


def test_rendezvous_exactly_one_issuer_per_op():
    n = 5000  # > 4 generations of the 1024-entry ring
    shared = mmap.mmap(-1, 1024 * lib.iccl_selftest_rzv_bytes())
    out = mmap.mmap(-1, 2 * n * 2 * 8)
    ctx = mp.get_context("fork")
    ps = [ctx.Process(target=_rzv_side, args=(shared, out, kind, n, 11 + kind)) for kind in (0, 1)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = np.frombuffer(out, dtype=np.int64).reshape(2, n, 2)
    second = res[:, :, 0]
    assert (second >= 0).all(), "a second arrival saw halves of different ops"
    assert (second.sum(axis=0) == 1).all(), "every op needs exactly one issuer"
    exp = 1000 + 7 * np.arange(n) + np.arange(n) % 3
    for kind in (0, 1):
        mine = second[kind] == 1
        assert (res[kind, mine, 1] == exp[mine]).all(), "the issuer must see the other half of the same op"
    assert 0 < second[0].sum() < n  # both sides issued some (the race is real)


def _route_side(shared, out, side, n, seed):
    rng = random.Random(seed)
    pair = _addr(shared)
    res = np.frombuffer(out, dtype=np.int8).reshape(2, n)
    for q in range(n):
        res[side, q] = lib.iccl_selftest_route_small(pair, side)
        if rng.random() < 0.05:
            for _ in range(rng.randint(1, 2000)):
                pass


def _route_toggler(shared, toggles, seed):
    rng = random.Random(seed)
    pair = _addr(shared)
    armed = False
    for _ in range(toggles):
        for _ in range(rng.randint(100, 5000)):
            pass
        if rng.random() < 0.5:
            lib.iccl_selftest_route_arm(pair, -1 if armed else 1, -1)  # a fault script installed / cleared
            armed = not armed
        else:
            lib.iccl_selftest_route_arm(pair, 0, rng.randint(0, 1))  # switch_qp to a path


def test_small_op_routing_agrees_under_concurrent_arming():
    n = 20000
    shared = mmap.mmap(-1, lib.iccl_selftest_pair_bytes())
    out = mmap.mmap(-1, 2 * n)
    ctx = mp.get_context("fork")
    ps = [ctx.Process(target=_route_side, args=(shared, out, side, n, 5 + side)) for side in (0, 1)]
    ps.append(ctx.Process(target=_route_toggler, args=(shared, 300, 9)))
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = np.frombuffer(out, dtype=np.int8).reshape(2, n)
    assert (res[0] == res[1]).all(), f"{int((res[0] != res[1]).sum())} small ops routed differently by the two sides"
    assert 0 < res[0].sum() < n, "both routes occur"


def test_route_segments_start_after_both_sides():
    """A change of route applies from the first op neither side has routed."""
    pair_mem = mmap.mmap(-1, lib.iccl_selftest_pair_bytes())
    pair = _addr(pair_mem)
    assert [lib.iccl_selftest_route_small(pair, 0) for _ in range(5)] == [0] * 5   # sender ahead: 5 LL
    assert [lib.iccl_selftest_route_small(pair, 1) for _ in range(2)] == [0, 0]    # receiver at 2
    lib.iccl_selftest_route_arm(pair, 1, -1)                                      # armed now
    assert [lib.iccl_selftest_route_small(pair, 1) for _ in range(4)] == [0, 0, 0, 1]  # ops 2..4 stay LL
    assert lib.iccl_selftest_route_small(pair, 0) == 1                             # op 5: rendezvous
    lib.iccl_selftest_route_arm(pair, -1, -1)                                     # disarmed at 6
    assert lib.iccl_selftest_route_small(pair, 0) == 0
    assert lib.iccl_selftest_route_small(pair, 1) == 0


# ---------------------------------------------------------------- failover protocol (armed transfers)
def _failover(scenario, nchunks=12, fault_chunk=5, delta_us=20_000):
    out = (C.c_int64 * 8)()
    rc = lib.iccl_selftest_failover(scenario, nchunks, fault_chunk, delta_us, out)
    keys = ("switches", "resume", "done", "total", "done_flags", "records", "probe", "async_err")
    return rc, dict(zip(keys, list(out)))


def test_failover_protocol_no_fault():
    rc, o = _failover(0)
    assert rc == 0 and o["switches"] == 0 and o["probe"] == 0 and o["async_err"] == 0
    assert o["done"] == o["total"] == 12 and o["done_flags"] == 1
    assert o["records"] == 12  # one record per chunk


def test_failover_protocol_slow_chunk_probe_lands_no_switch():
    """Fig. 7(b) innocent variant: no progress for > delta on a live path; the
    CTS probe crosses it, so the watchdog does not switch."""
    rc, o = _failover(1)
    assert rc == 0 and o["probe"] == 1 and o["switches"] == 0
    assert o["done"] == 12 and o["done_flags"] == 1


@pytest.mark.parametrize("fault_chunk", [0, 1, 5, 11])
def test_failover_protocol_dead_primary_switches_at_breakpoint(fault_chunk):
    """The primary Down from `fault_chunk`: the probe is lost, the watchdog
    switches with resume = the receiver's breakpoint, the
    backup attempt delivers chunks [resume, N), and the op completes exactly
    once: one record per chunk, both done flags written by the watchdog."""
    rc, o = _failover(2, fault_chunk=fault_chunk)
    assert rc == 0 and o["switches"] == 1 and o["async_err"] == 0
    assert o["resume"] == fault_chunk
    assert o["done"] == o["total"] == 12 and o["done_flags"] == 1
    assert o["records"] == 12


def test_failover_protocol_both_paths_dead_connection_failed():
    rc, o = _failover(3, fault_chunk=4)
    assert o["switches"] == 1 and o["async_err"] == 7  # ICCL_ERR_CONNECTION_FAILED


def test_failover_protocol_upstream_stall_never_probes():
    """A side's stream reaches the op late (ready flags set after 3 delta):
    an upstream stall, not a path failure — no probe, no switch."""
    rc, o = _failover(4)
    assert rc == 0 and o["probe"] == 0 and o["switches"] == 0 and o["done_flags"] == 1
