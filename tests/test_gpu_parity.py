"""GPU parity: the B200 path's delivered bytes against the CPU oracle.

Every comparison is raw-byte (bit-exact).  Single-GPU tests drive the whole
product path through the C ABI with a world-size-1 communicator (self send /
recv through the proxy, copy engine, SM kernel, failover and monitor); the
multi-rank tests run one process per rank, mapped onto the visible GPUs
round-robin, so they never skip: on a one-GPU box 2-8 ranks share cuda:0
(CUDA IPC, stream memops, K5/K6/K7 and the copy engines all work between
processes on one device).
"""
import numpy as np
import pytest

from gpu_helpers import fault_delta_us, payload, run_ranks, to_dev
from oracle import collectives as oc

pytestmark = pytest.mark.gpu

MiB = 1 << 20


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _world(minimum: int) -> int:
    """Ranks for a multi-rank test: every GPU, and at least `minimum`."""
    import torch
    return max(minimum, torch.cuda.device_count())


def _comm1(**cfg):
    from paper_2510_00991_b200 import Communicator, IcclConfig
    return Communicator(0, 1, 0, IcclConfig.defaults(**cfg))


def _oracle_sendrecv(src: np.ndarray) -> np.ndarray:
    return oc.send_recv(oc.CommGroup(2, chunk_size=4 * MiB), 0, 1, src)


def _self_roundtrip(torch, comm, src_np, off_src=0, off_dst=0):
    from paper_2510_00991_b200 import P2POp
    n = src_np.nbytes - off_src
    s = to_dev(src_np, "cuda")
    d = torch.zeros(n + off_dst, dtype=torch.uint8, device="cuda")
    comm.batch_isend_irecv([P2POp("isend", s[off_src:], 0), P2POp("irecv", d[off_dst:], 0)])
    torch.cuda.synchronize()
    return d[off_dst:].cpu().numpy()


@pytest.mark.parametrize("transport", ["ce", "sm"])
@pytest.mark.parametrize("n", [1, 15, 4096, MiB + 3, 64 * MiB + 17])
def test_self_sendrecv_bytes(torch_cuda, transport, n):
    comm = _comm1(transport=transport, chunk_bytes=16 * MiB)
    try:
        src = payload(n, seed=n)
        got = _self_roundtrip(torch_cuda, comm, src)
        assert np.array_equal(got, _oracle_sendrecv(src))
        comm.check_async_error()
    finally:
        comm.destroy()


@pytest.mark.parametrize("offs", [(1, 0), (0, 3), (5, 9), (16, 32)])
def test_self_sendrecv_misaligned(torch_cuda, offs):
    comm = _comm1(transport="sm")
    try:
        src = payload(3 * MiB + 7, seed=11)
        got = _self_roundtrip(torch_cuda, comm, src, *offs)
        assert np.array_equal(got, src[offs[0]:])
    finally:
        comm.destroy()


def test_self_sendrecv_256mib_property(torch_cuda):
    """Full PP-activation size (bf16 [4,4096,8192]): checksum-of-chunks property
    instead of a byte-by-byte oracle run."""
    torch = torch_cuda
    comm = _comm1()
    try:
        g = torch.Generator(device="cuda").manual_seed(1)
        s = torch.randint(-32768, 32767, (4, 4096, 8192), dtype=torch.int16, device="cuda", generator=g).view(
            torch.bfloat16)
        d = torch.empty_like(s)
        from paper_2510_00991_b200 import P2POp
        comm.batch_isend_irecv([P2POp("isend", s, 0), P2POp("irecv", d, 0)])
        torch.cuda.synchronize()
        assert torch.equal(s.view(torch.int16), d.view(torch.int16))
    finally:
        comm.destroy()


def test_sm_copy_kernel_k1(torch_cuda):
    import ctypes as C
    from paper_2510_00991_b200._lib import lib
    torch = torch_cuda
    for n, so, do in [(1, 0, 0), (17, 1, 1), (33, 3, 7), (1 << 20, 0, 0), ((1 << 24) + 5, 2, 2), ((1 << 24) + 5, 0, 8)]:
        src = payload(n + so, seed=n)
        s = to_dev(src, "cuda")
        d = torch.zeros(n + do, dtype=torch.uint8, device="cuda")
        rc = lib.iccl_copy_sm(C.c_void_p(s.data_ptr() + so), C.c_void_p(d.data_ptr() + do), n, 16,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy()[do:], src[so:])


def test_k2_k3_gather_scatter(torch_cuda):
    torch = torch_cuda
    from paper_2510_00991_b200 import gather_rows, scatter_rows
    rng = np.random.default_rng(5)
    rows, H = 4096, 7168 * 2  # bf16 hidden 7168 -> 14336 B per row
    src = payload(rows * H, seed=3).reshape(rows, H)
    idx = rng.integers(0, rows, 3 * rows)
    s = to_dev(src, "cuda")
    i = torch.from_numpy(idx).cuda()
    g = gather_rows(s, i)
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), src[idx])
    from paper_2510_00991_b200 import expand_rows
    k = 3
    order = rng.permutation(rows * k)
    pos = np.empty_like(order)
    pos[order] = np.arange(rows * k)
    e = torch.zeros(rows * k, H, dtype=torch.uint8, device="cuda")
    expand_rows(s, torch.from_numpy(pos).cuda(), k, e)
    torch.cuda.synchronize()
    assert np.array_equal(e.cpu().numpy(), src[order // k])
    perm = rng.permutation(rows)
    out = torch.zeros_like(s)
    scatter_rows(s, torch.from_numpy(perm).cuda(), out)
    torch.cuda.synchronize()
    exp = np.zeros_like(src)
    exp[perm] = src
    assert np.array_equal(out.cpu().numpy(), exp)


def test_self_alltoallv_world1(torch_cuda):
    torch = torch_cuda
    comm = _comm1()
    try:
        src = to_dev(payload(1000 * 16, seed=2), "cuda").view(1000, 16)
        dst = torch.zeros_like(src)
        comm.alltoallv(dst, src, [1000], [1000])
        torch.cuda.synchronize()
        assert torch.equal(src, dst)
    finally:
        comm.destroy()


def test_self_failover_resumes_on_sm_path(torch_cuda):
    """Inject a Down on the primary (copy-engine) path at chunk 2 of the first
    send: the watchdog + probe must switch to the SM path and resume at the
    receiver's breakpoint, bit-exact."""
    torch = torch_cuda
    from paper_2510_00991_b200 import FaultScript
    comm = _comm1(chunk_bytes=MiB, delta_us=200, probe_period_us=100, window=4)
    try:
        comm.set_faults(FaultScript().down(0, 0, chunk=2, op_index=0))
        src = payload(16 * MiB, seed=77)
        got = _self_roundtrip(torch, comm, src)
        assert np.array_equal(got, _oracle_sendrecv(src))
        ev = comm.switch_events()
        assert ev and ev[0]["to"] == "backup" and ev[0]["trigger"] == "watchdog"
        assert ev[0]["resume_chunk"] == 2  # chunks 0,1 landed before the gate
        assert comm.active_path(0) == "backup"
        # next transfer goes straight over the backup path
        got = _self_roundtrip(torch, comm, src[::-1].copy())
        assert np.array_equal(got, src[::-1])
        comm.check_async_error()
    finally:
        comm.destroy()


def test_self_failover_switch_back(torch_cuda):
    torch = torch_cuda
    from paper_2510_00991_b200 import FaultScript
    comm = _comm1(chunk_bytes=MiB, delta_us=200, probe_period_us=100)
    try:
        comm.set_faults(FaultScript().down(0, 0, chunk=1, op_index=0).up(0, 0, t_us=50_000))
        src = payload(8 * MiB, seed=78)
        assert np.array_equal(_self_roundtrip(torch, comm, src), src)
        import time
        time.sleep(0.2)
        assert np.array_equal(_self_roundtrip(torch, comm, src), src)
        ev = comm.switch_events()
        assert [e["to"] for e in ev][:2] == ["backup", "primary"]
        assert comm.active_path(0) == "primary"
    finally:
        comm.destroy()


def test_api_switch_qp_mid_stream(torch_cuda):
    torch = torch_cuda
    comm = _comm1(chunk_bytes=MiB)
    try:
        src = payload(32 * MiB, seed=5)
        comm.switch_qp(0, "ToBackup")
        assert np.array_equal(_self_roundtrip(torch, comm, src), src)
        assert comm.active_path(0) == "backup"
        comm.switch_qp(0, "ToPrimary")
        assert np.array_equal(_self_roundtrip(torch, comm, src), src)
    finally:
        comm.destroy()


def test_monitor_records(torch_cuda):
    torch = torch_cuda
    from paper_2510_00991_b200 import sample_series
    comm = _comm1(chunk_bytes=MiB, monitor_enabled=True)
    try:
        src = payload(24 * MiB, seed=9)
        assert np.array_equal(_self_roundtrip(torch, comm, src), src)
        recs = comm.monitor.drain()
        assert len(recs) == 24
        assert sum(r.size for r in recs) == 24 * MiB
        assert all(r.t2 > r.t1 for r in recs)
        assert len(sample_series(recs, 8)) == 24 - 8 + 1
    finally:
        comm.destroy()


def test_errors(torch_cuda):
    torch = torch_cuda
    from paper_2510_00991_b200 import GroupTooSmall, InvalidArgument, ZeroLengthMessage
    comm = _comm1()
    try:
        with pytest.raises(ZeroLengthMessage):
            comm.send(torch.zeros(0, device="cuda"), 0)
        with pytest.raises(InvalidArgument):
            comm.send(torch.zeros(4, device="cuda"), 3)
        with pytest.raises(GroupTooSmall):
            comm.alltoall(torch.zeros(4, device="cuda"), torch.zeros(4, device="cuda"))
        assert comm.op_counts() == {0: 0}
    finally:
        comm.destroy()


# ---------------------------------------------------------------- multi-GPU
def test_pair_sendrecv_bytes(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    sizes = [8, 4096 + 1, 3 * MiB + 5, 64 * MiB]
    res = run_ranks(2, sc.sendrecv_pair, tmp_path, sizes=sizes, offsets=(0, 3))
    for i, n in enumerate(sizes):
        for off in (0, 3):
            src = payload(n + off, seed=1000 + i)[off:]
            assert np.array_equal(res[1][f"r_{n}_{off}"], _oracle_sendrecv(src.copy()))


@pytest.mark.parametrize("transport", ["ce", "sm"])
def test_pair_bidirectional(torch_cuda, tmp_path, transport):
    import gpu_scenarios as sc
    res = run_ranks(2, sc.bidirectional, tmp_path, nbytes=64 * MiB + 48, config=dict(transport=transport))
    for r in range(2):
        assert np.array_equal(res[r]["recv"], payload(64 * MiB + 48, seed=1 - r))


def test_ring_shift_all_gpus(torch_cuda, tmp_path):
    import torch
    import gpu_scenarios as sc
    w = _world(4)
    res = run_ranks(w, sc.ring_shift, tmp_path, nbytes=32 * MiB)
    for r in range(w):
        assert np.array_equal(res[r]["recv"], payload(32 * MiB, seed=50 + (r - 1) % w))


def test_alltoallv_uneven_vs_oracle(torch_cuda, tmp_path):
    import torch
    import gpu_scenarios as sc
    w = _world(4)
    rng = np.random.default_rng(0)
    splits = [[int(x) for x in rng.integers(0, 300, w)] for _ in range(w)]
    splits[0][w - 1] = 0  # a zero-count pair
    row = 7168 * 2
    res = run_ranks(w, sc.alltoallv_uneven, tmp_path, row_bytes=row, splits=splits)
    send = [payload(sum(splits[i]) * row, seed=7 + i) for i in range(w)]
    exp = oc.expected_alltoallv(send, splits, row)
    orc = oc.alltoallv(oc.CommGroup(w, chunk_size=4 * MiB), send, splits, oc.counts_T(splits), row)
    for r in range(w):
        assert np.array_equal(exp[r], orc[r])
        assert np.array_equal(res[r]["recv"], exp[r])


@pytest.mark.parametrize("ll_max", [32 * 1024, 256 * 1024])
def test_pair_ll_small_messages(torch_cuda, tmp_path, ll_max):
    """LL path (K5) mixed with copy-engine ops in one group, more LL messages
    per pair than slots; at 256 KiB ops span up to 16 CTAs each."""
    import gpu_scenarios as sc
    sizes = [1, 3, 4, 7, 64, 1000, 4096, 32 * 1024, 32 * 1024 + 1, 300 * 1024, 5, 6, 8, 9, 64 * 1024 + 5,
             200 * 1024 + 3, 256 * 1024]
    res = run_ranks(2, sc.ll_mixed, tmp_path, sizes=sizes, config=dict(sm_small_bytes=ll_max))
    for r in range(2):
        peer = 1 - r
        for rd in range(3):
            for i, n in enumerate(sizes):
                assert np.array_equal(res[r][f"r{rd}_{i}"], payload(n, seed=10_000 * peer + 100 * rd + i)), (r, rd, n)
        for i, n in enumerate(sizes):
            assert np.array_equal(res[r][f"single_{i}"], payload(n, seed=555 + i))


def test_pair_failover_mid_message(torch_cuda, tmp_path):
    import gpu_scenarios as sc
    n = 48 * MiB
    res = run_ranks(2, sc.failover_pair, tmp_path, nbytes=n, fault_chunk=5,
                    config=dict(chunk_bytes=4 * MiB, delta_us=fault_delta_us(2), window=4))
    assert np.array_equal(res[1]["recv"], _oracle_sendrecv(payload(n, seed=99)))
    issuer = 0 if len(res[0]["switch_to"]) else 1
    assert list(res[issuer]["switch_to"])[:1] == [1]
    assert res[issuer]["resume"][0] == 5


def test_relay_failover_mid_message(torch_cuda, tmp_path):
    """Backup = GPU relay (two copy-engine hops through the lowest-index
    non-endpoint GPU): primary 0->1 Down at chunk 3,
    resume through GPU 2 at the breakpoint, bit-exact."""
    import torch
    import gpu_scenarios as sc
    n = 48 * MiB + 80
    res = run_ranks(_world(3), sc.failover_pair, tmp_path, nbytes=n, fault_chunk=3,
                    config=dict(chunk_bytes=4 * MiB, delta_us=fault_delta_us(_world(3)), window=4, backup_kind="relay",
                                relay_slot_mib=3))
    assert np.array_equal(res[1]["recv"], _oracle_sendrecv(payload(n, seed=99)))
    issuer = 0 if len(res[0]["switch_to"]) else 1
    assert list(res[issuer]["switch_to"])[:1] == [1]
    assert res[issuer]["resume"][0] == 3


def test_relay_ring_api_switch(torch_cuda, tmp_path):
    import torch
    import gpu_scenarios as sc
    w = _world(3)
    n = 20 * MiB + 16
    res = run_ranks(w, sc.relay_ring, tmp_path, nbytes=n,
                    config=dict(chunk_bytes=8 * MiB, backup_kind="relay", relay_slot_mib=2))
    for r in range(w):
        frm = (r - 1) % w
        for it in range(2):
            assert np.array_equal(res[r][f"recv{it}"], payload(n, seed=70 + 10 * it + frm))
        assert np.array_equal(res[r]["recv_back"], payload(n, seed=90 + frm))
        assert int(res[r]["path"][0]) == 1


def test_pair_direct_mid_size(torch_cuda, tmp_path):
    """256 KiB < n <= 16 MiB: the side that arrives second runs K6 on its own
    stream (push or pull, zero-copy), bit-exact in groups and single ops."""
    import gpu_scenarios as sc
    MiB_ = 1 << 20
    sizes = [300 * 1024 + 5, MiB_, 3 * MiB_ + 7, 16 * MiB_, 1000, 40 * MiB_]
    res = run_ranks(2, sc.direct_mixed, tmp_path, sizes=sizes, config=dict(direct_max_kib=16 * 1024))
    for r in range(2):
        peer = 1 - r
        for rd in range(2):
            for i, n in enumerate(sizes):
                assert np.array_equal(res[r][f"r{rd}_{i}"], payload(n, seed=20_000 * peer + 100 * rd + i)), (r, rd, n)
        for i, n in enumerate(sizes):
            assert np.array_equal(res[r][f"single_{i}"], payload(n, seed=777 + i))
    assert int(res[0]["kernels"][0]) + int(res[1]["kernels"][0]) > 0  # K6 / LL ran


# ---------------------------------------------------------------- 8 ranks (configs 4 and 5)
def _moe_oracle_check(res, world, T, k=8, H=7168):
    row = 2 * H
    splits = [res[i]["send_counts"].tolist() for i in range(world)]
    send = [res[i]["packed"] for i in range(world)]
    exp = oc.expected_alltoallv(send, splits, row)
    orc = oc.alltoallv(oc.CommGroup(world, chunk_size=4 * MiB), send, splits, oc.counts_T(splits), row)
    for r in range(world):
        assert np.array_equal(exp[r], orc[r])
        assert np.array_equal(res[r]["recv"], orc[r]), f"rank {r} received bytes differ from the oracle"


def test_moe_alltoallv_8_ranks_vs_oracle(torch_cuda, tmp_path):
    """Config 4 at 8 ranks (oversubscribed on the visible GPUs): §8(d)
    routing, 64 experts, hidden 7168 bf16, T = 128 tokens per rank for the
    byte-for-byte oracle comparison; every one of the 56 ordered pairs moves."""
    import gpu_scenarios as sc
    world, T = 8, 128
    res = run_ranks(world, sc.moe_config4, tmp_path, T=T, timeout=300)
    for r in range(world):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    _moe_oracle_check(res, world, T)


def test_moe_alltoallv_8_ranks_full_size(torch_cuda, tmp_path):
    """Config 4 at full size (T = 4096 per rank, 448 MiB of packed rows per
    rank) on 8 ranks: received rows checked on the device against every
    source's regenerated routing and payload, and the combine round trip."""
    import gpu_scenarios as sc
    res = run_ranks(8, sc.moe_config4, tmp_path, T=4096, keep_bytes=False, timeout=300)
    for r in range(8):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r


def test_failover_3_to_5_under_alltoallv_8_ranks(torch_cuda, tmp_path):
    """Config 5 at 8 ranks: the primary path of pair 3 -> 5 goes Down in the
    middle of its first transfer of a config-4 alltoallv with the monitor on;
    the pair switches at the breakpoint and every rank's bytes equal the
    oracle's."""
    import gpu_scenarios as sc
    world, T = 8, 128
    res = run_ranks(world, sc.moe_config4, tmp_path, T=T, fault=(3, 5, 2), timeout=300,
                    config=dict(chunk_bytes=256 * 1024, delta_us=fault_delta_us(world), window=4, monitor_enabled=True))
    for r in range(world):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    _moe_oracle_check(res, world, T)
    sw = [(r, int(p), int(t)) for r in (3, 5) for p, t in zip(res[r]["switch_peers"], res[r]["switch_to"])]
    assert any(t == 1 and p == (5 if r == 3 else 3) for r, p, t in sw), sw
    assert sum(int(res[r]["records"][0]) for r in range(world)) > 0


@pytest.mark.parametrize("world", [1, 2, 4])
def test_fused_dispatch_vs_oracle(torch_cuda, tmp_path, world):
    """K8 (fused dispatch: K2's expand + the alltoallv push in one kernel, no
    staging buffer) delivers exactly the rows of K2 + alltoallv: checked on
    the device against every source's routing and payload, byte for byte
    against the oracle, and through the combine round trip; three
    back-to-back dispatches reuse the buffers."""
    import gpu_scenarios as sc
    T = 128
    res = run_ranks(world, sc.moe_config4, tmp_path, T=T, fused=True, reps=3, timeout=300)
    for r in range(world):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    if world > 1:
        _moe_oracle_check(res, world, T)


def test_fused_dispatch_8_ranks_full_size(torch_cuda, tmp_path):
    """K8 at config 4's full size on 8 ranks (T = 4096, 448 MiB of routed
    rows per rank): every received row and the combine round trip."""
    import gpu_scenarios as sc
    res = run_ranks(8, sc.moe_config4, tmp_path, T=4096, keep_bytes=False, fused=True, timeout=300)
    for r in range(8):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r


def test_fused_dispatch_armed_pair_falls_back(torch_cuda, tmp_path):
    """A fault script naming pair 1 -> 2 arms it: rank 1's dispatch takes the
    unfused form (K2 into staging + the alltoallv) where the gate, the
    watchdog and the switch apply; the other ranks stay fused; every rank
    receives exactly the oracle's bytes and pair 1 -> 2 switched."""
    import gpu_scenarios as sc
    world, T = 4, 128
    res = run_ranks(world, sc.moe_config4, tmp_path, T=T, fused=True, fault=(1, 2, 2), timeout=300,
                    config=dict(chunk_bytes=256 * 1024, delta_us=fault_delta_us(world), window=4))
    for r in range(world):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    _moe_oracle_check(res, world, T)
    sw = [(r, int(p), int(t)) for r in (1, 2) for p, t in zip(res[r]["switch_peers"], res[r]["switch_to"])]
    assert any(t == 1 for _, _, t in sw), sw


@pytest.mark.parametrize("world", [1, 2, 4])
def test_fused_combine_vs_oracle(torch_cuda, tmp_path, world):
    """K10 (fused combine: the reverse alltoallv as NVLink loads + K3's
    scatter in one kernel, no staging) returns every routed row to its
    (token, k) slot: the round trip after a fused dispatch equals the tokens,
    three back-to-back combines reuse the buffers, and the dispatched bytes
    equal the oracle's."""
    import gpu_scenarios as sc
    T = 128
    res = run_ranks(world, sc.moe_config4, tmp_path, T=T, fused=True, fused_combine=True, reps=3, timeout=300)
    for r in range(world):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    if world > 1:
        _moe_oracle_check(res, world, T)


def test_fused_combine_8_ranks_full_size_and_armed_fallback(torch_cuda, tmp_path):
    """Config 4 at full size on 8 ranks with K8 + K10, and a 4-rank run with
    pair 2 -> 1 armed (rank 1 combines through staging + the alltoallv + K3,
    where the failover applies): every round trip restores the tokens."""
    import gpu_scenarios as sc
    res = run_ranks(8, sc.moe_config4, tmp_path, T=4096, keep_bytes=False, fused=True, fused_combine=True,
                    timeout=300)
    for r in range(8):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r
    (tmp_path / "armed").mkdir()
    res = run_ranks(4, sc.moe_config4, tmp_path / "armed", T=128, fused=True, fused_combine=True,
                    fault=(2, 1, 1 << 20), timeout=300, config=dict(chunk_bytes=256 * 1024))
    for r in range(4):
        assert bool(res[r]["recv_ok"][0]) and bool(res[r]["roundtrip_ok"][0]), r


@pytest.mark.parametrize("world", [2, 4])
def test_pp_1f1b_schedule_bytes(torch_cuda, tmp_path, world):
    """SURVEY §8f row f2 on the product: Megatron's 1F1B schedule (batched
    send_forward_recv_backward / send_backward_recv_forward on a
    communication stream, GEMMs on the compute stream) over `world` stages,
    8 microbatches: no deadlock, and every received activation / gradient is
    byte-identical to what its stage sent."""
    import gpu_scenarios as sc
    res = run_ranks(world, sc.pp_1f1b, tmp_path, M=8, timeout=300)
    for r in range(world):
        n = int(res[r]["n"][0])
        exp = 0 if world == 1 else (8 if r in (0, world - 1) else 16)
        assert n == exp and int(res[r]["ok"][0]) == n, (r, n, int(res[r]["ok"][0]))
