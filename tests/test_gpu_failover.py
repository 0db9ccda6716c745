"""GPU tests of the paper's side mechanisms on every size class.

- A fault script naming a pair arms it: ops of every size (those a healthy
  pair sends through K5 / K6) take the chunked path, stall behind the
  injected gate, switch at the receiver's breakpoint and land bit-exact
  (SPEC.md:90-98, 255-263, 275).
- A failed-over op releases the user streams only once the surviving attempt
  is done: buffers reused right after completion stay intact.
- Every op yields monitor records and a valid six-pointer
  state.
- switch_qp applies to every size class; LL routing stays in agreement while
  a pair toggles between paths.

Ranks share GPUs round-robin (gpu_helpers), so these run on one GPU too.
"""
import numpy as np
import pytest

from gpu_helpers import fault_delta_us, payload, run_ranks

pytestmark = pytest.mark.gpu

KiB, MiB = 1 << 10, 1 << 20


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _issuer(res):
    return 0 if len(res[0]["switch_to"]) else 1


@pytest.mark.parametrize("nbytes,chunk,fault_chunk", [
    (100 * KiB + 3, 64 * KiB, 1),     # LL size (K5 on a healthy pair): K1 primary, copy-engine backup
    (300 * KiB + 5, 64 * KiB, 2),     # K6 size
    (1 * MiB, 256 * KiB, 1),          # K6 size
    (16 * MiB, 1 * MiB, 7),           # K6 size (the largest direct op)
])
def test_fault_stops_every_size_class(torch_cuda, tmp_path, nbytes, chunk, fault_chunk):
    import gpu_scenarios as sc
    res = run_ranks(2, sc.fault_size_class, tmp_path, nbytes=nbytes, fault_chunk=fault_chunk,
                    config=dict(chunk_bytes=chunk, delta_us=fault_delta_us(2), window=4, monitor_enabled=True))
    assert np.array_equal(res[1]["recv"], payload(nbytes, seed=nbytes))
    i = _issuer(res)
    assert list(res[i]["switch_to"])[:1] == [1], "the injected Down must trigger a watchdog switch"
    assert res[i]["resume"][0] == fault_chunk
    nchunks = (nbytes + chunk - 1) // chunk
    recs = np.concatenate([res[0]["records"], res[1]["records"]])
    assert len(recs) == nchunks, "one monitor record per chunk (WR/WC pair)"
    assert recs.sum() == nbytes


@pytest.mark.parametrize("nbytes,chunk,fault_chunk", [(48 * MiB, 4 * MiB, 5), (3 * MiB + 7, 256 * KiB, 3)])
def test_failover_buffers_reused_after_completion(torch_cuda, tmp_path, nbytes, chunk, fault_chunk):
    import gpu_scenarios as sc
    res = run_ranks(2, sc.failover_reuse, tmp_path, nbytes=nbytes, fault_chunk=fault_chunk, reps=2,
                    config=dict(chunk_bytes=chunk, delta_us=fault_delta_us(2), window=4))
    for it in range(2):
        assert np.array_equal(res[1][f"recv{it}"], payload(nbytes, seed=500 + it)), it
        assert bool(res[1][f"marker_ok{it}"][0]), "a stale copy wrote into the receiver's buffer after completion"
    i = _issuer(res)
    assert list(res[i]["switch_to"])[:1] == [1]


def test_monitor_and_state_for_every_op(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    sizes = [1000, 64 * KiB + 3, 300 * KiB + 5, 3 * MiB, 20 * MiB]
    res = run_ranks(2, sc.monitor_every_op, tmp_path, sizes=sizes, config=dict(monitor_enabled=True))
    for r in range(2):
        peer = 1 - r
        for i, n in enumerate(sizes):
            assert np.array_equal(res[r][f"r{i}"], payload(n, seed=30_000 * peer + i))
            assert np.array_equal(res[r][f"s{i}"], payload(n, seed=40_000 + i))
        assert (res[r]["state_total"] == 1).all()
        assert (res[r]["state_done"] == res[r]["state_total"]).all()
    rec = sorted(np.concatenate([res[0]["rec_bytes"], res[1]["rec_bytes"]]).tolist())
    assert rec == sorted(sizes * 4), "exactly one record per transfer (LL, K6 and copy engine)"


def test_switch_qp_applies_to_every_size_class(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    sizes = [100 * KiB, 1 * MiB, 8 * MiB + 5, 40 * MiB]
    res = run_ranks(2, sc.api_switch_mid_size, tmp_path, sizes=sizes)
    for phase in range(2):
        for i, n in enumerate(sizes):
            assert np.array_equal(res[1][f"p{phase}_{i}"], payload(n, seed=60_000 + 100 * phase + i))
    assert int(res[0]["path_after_switch"][0]) == 1


def test_ll_routing_agrees_while_pair_toggles(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    res = run_ranks(2, sc.ll_route_toggle, tmp_path, n_msgs=40, size=4099)
    for i in range(40):
        assert np.array_equal(res[1]["recv"][i], payload(4099, seed=70_000 + i)), i


def test_register_deregister(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    res = run_ranks(2, sc.register_deregister, tmp_path, nbytes=5 * MiB + 1)
    for it in range(3):
        assert np.array_equal(res[1][f"recv{it}"], payload(5 * MiB + 1, seed=80_000 + it))
    assert int(res[0]["unregistered_rc"][0]) == 5  # ICCL_ERR_UNREGISTERED_REGION


def test_AC4_innocent_stall_never_switches(torch_cuda, tmp_path):
    """100/100 seeded trials: a stream held upstream (sender or receiver) for
    1.5-6 delta never triggers a switch."""
    import gpu_scenarios as sc
    d = fault_delta_us(2)
    res = run_ranks(2, sc.innocent_stall, tmp_path, trials=100, delta_us=d, timeout=280,
                    config=dict(chunk_bytes=1 * MiB, delta_us=d, window=4))
    assert len(res[1]["ok"]) == 100 and res[1]["ok"].all()
    assert int(res[0]["switches"][0]) == 0 and int(res[1]["switches"][0]) == 0


def _recs(res):
    r = res[0] if len(res[0]["t2"]) else res[1]
    return r["t1"], r["t2"], r["bytes"]


def _series(t1, t2, b, w):
    # window_throughput per completion, completion order
    return np.array([b[i - w + 1:i + 1].sum() / ((t2[i] - t1[i - w + 1]) * 1e-9) for i in range(w - 1, len(b))])


def test_AC5_monitor_accuracy_and_smoothing(torch_cuda, tmp_path):
    """AC5 on hardware.  Steady flow: every W=8 sample after
    warm-up within +-5% of the measured rate C.  Disturbance (the path gated
    mid-transfer, no switch): the W=8 series falls below C/2 within 8 samples
    of the disturbed record and recovers to within 10% of C 8 samples after
    it (the smoothing claim: test_AC5_competing_flow_smoothing)."""
    import gpu_scenarios as sc
    cfg = dict(chunk_bytes=64 * MiB, monitor_enabled=True, delta_us=200_000, window=1024)
    res = run_ranks(2, sc.monitor_accuracy, tmp_path, nchunks=40, chunk=64 * MiB, stall_chunk=-1, up_us=0,
                    config=cfg)
    t1, t2, b = _recs(res)
    assert len(b) == 40 and bool(res[1]["ok"][0])
    C_ = b.sum() / ((t2[-1] - t1[0]) * 1e-9)
    s8 = _series(t1, t2, b, 8)[8:]
    assert np.all(np.abs(s8 / C_ - 1) <= 0.05), (C_, s8.min(), s8.max())

    cfg["chunk_bytes"] = 16 * MiB
    cfg["delta_us"] = 5_000_000  # the disturbance must not switch
    (tmp_path / "d").mkdir()
    # the Up is timed from the install, the Down fires at the chunk's issue:
    # 200 ms leaves room for a slow issue (a stream creation, an IPC open)
    res = run_ranks(2, sc.monitor_accuracy, tmp_path / "d", nchunks=128, chunk=16 * MiB, stall_chunk=64,
                    up_us=200_000, config=cfg)
    t1, t2, b = _recs(res)
    assert len(b) == 128 and bool(res[1]["ok"][0])
    assert int(res[0]["switches"][0]) + int(res[1]["switches"][0]) == 0, (res[0]["switch_desc"], res[1]["switch_desc"])
    dur = t2 - t1
    k = int(np.argmax(dur))  # the disturbed record (waited behind the gate)
    assert dur[k] > 10 * np.median(dur), "the gate must show as one long record"
    # an armed pair's primary chunks are timed by the watchdog thread's host
    # observations (no CUDA call may sit on the failover path), so its
    # undisturbed rate is measured here, after the disturbance
    C_d = b[k + 1:].sum() / ((t2[-1] - t2[k]) * 1e-9)
    s8 = _series(t1, t2, b, 8)  # s8[i] ends at record i + 7
    first = k - 7  # first W=8 window that contains record k
    assert min(s8[max(0, first):first + 8]) < C_d / 2, "disturbance not seen within 8 samples"
    tail = s8[k + 8:k + 16]
    assert np.all(np.abs(tail / C_d - 1) <= 0.10), (C_d, tail)


def test_AC5_competing_flow_smoothing(torch_cuda, tmp_path):
    """AC5's smoothing claim on hardware: a second flow
    (SM stores through a second communicator) starts mid-transfer on the
    same link; the monitored flow's records slow down, and over the
    transition var(W=1) >= var(W=8) >= var(W=32).  Ranks sharing one GPU
    have no link to share (there the series' sample-to-sample variation is
    compared instead)."""
    import gpu_scenarios as sc
    cfg = dict(chunk_bytes=16 * MiB, monitor_enabled=True, window=1024)
    res = run_ranks(2, sc.monitor_competing, tmp_path, nchunks=384, chunk=16 * MiB, comp_bytes=2048 * MiB,
                    delay_us=2000, config=cfg)
    t1, t2, b = res[0]["t1"], res[0]["t2"], res[0]["bytes"]
    assert len(b) == 384 and bool(res[1]["ok"][0])
    n = len(b)
    # the three series indexed by completion (record i closes one sample of each)
    s1, s8, s32 = (np.concatenate([np.full(w - 1, np.nan), _series(t1, t2, b, w)]) for w in (1, 8, 32))
    if torch_cuda.cuda.device_count() == 1:
        # ranks sharing one GPU have no link to share: the "peer" copy is a
        # local copy the SM flow and the HBM traffic barely slow, so there
        # is no transition to find; the smoothing is checked on the whole
        # series' sample-to-sample variation (the variance of differences)
        k = -1
        v1, v8, v32 = (np.var(np.diff(x[31:])) for x in (s1, s8, s32))
    else:
        base = np.median(s1[:48])
        # the transition: the first completion from which the W=8 series
        # stays clearly below the steady rate for 16 samples; the variances
        # are compared over the same completions around it (+-32, the widest
        # window's span)
        slow = s8 < 0.85 * base
        ks = [i for i in range(48, n - 16) if slow[i:i + 16].all()]
        assert ks, "the competing flow must slow the monitored one"
        k = ks[0]
        lo, hi = k - 32, min(n, k + 32)
        v1, v8, v32 = np.var(s1[lo:hi]), np.var(s8[lo:hi]), np.var(s32[lo:hi])
    assert v1 >= v8 >= v32, (k, v1, v8, v32)


def test_AC3_fuzz_exactly_once_on_hardware(torch_cuda, tmp_path):
    """AC3 on the product: 240 randomised transfers of 1 KiB -
    64 MiB with random chunk sizes and fault scripts (Down at a random chunk,
    Down before the op, Down then restored, none).  Every transfer lands
    bit-exact, its monitor records name every chunk 0..N-1 exactly once (the
    delivered sequence is gapless and duplicate-free), and the sender's
    six-pointer state ends at done == total."""
    import gpu_scenarios as sc
    d = fault_delta_us(2)
    trials = 240
    res = run_ranks(2, sc.fuzz_failover, tmp_path, trials=trials, seed=31337, delta_us=d, timeout=900, _hang_s=880,
                    config=dict(delta_us=d, probe_period_us=max(200, d // 2), window=4, monitor_enabled=True))
    r0, r1 = res
    assert len(r1["ok"]) == trials and r1["ok"].all(), np.nonzero(~r1["ok"])
    for t in range(trials):
        got = np.concatenate([r["chunks"][r["chunks_off"][t]:r["chunks_off"][t + 1]] for r in res])
        n = int(r0["nchunks"][t])
        assert sorted(got.tolist()) == list(range(n)), (t, int(r0["n"][t]), int(r0["mode"][t]), got)
    assert (r0["state_done"] == r0["state_total"]).all()
    assert (r0["state_total"] == r0["nchunks"]).all()
    assert set(r0["mode"].tolist()) == {0, 1, 2, 3}
