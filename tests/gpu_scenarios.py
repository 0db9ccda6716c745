"""Rank programs for the multi-GPU parity tests (picklable top-level
functions run by gpu_helpers.run_ranks, one process per GPU)."""
import numpy as np
import torch

from gpu_helpers import dev_of, payload, to_dev


def sendrecv_pair(comm, rank, world, sizes, offsets=(0,)):
    """0 -> 1 for each size (and every offset into a larger buffer)."""
    out = {}
    dev = dev_of(rank)
    for i, n in enumerate(sizes):
        for off in offsets:
            src = payload(n + off, seed=1000 + i)
            if rank == 0:
                t = to_dev(src, dev)
                comm.send(t[off:], 1)
            elif rank == 1:
                r = torch.zeros(n + off, dtype=torch.uint8, device=dev)
                comm.recv(r[off:], 0)
                torch.cuda.synchronize()
                out[f"r_{n}_{off}"] = r[off:].cpu().numpy()
    torch.cuda.synchronize()
    return out


def bidirectional(comm, rank, world, nbytes, iters=3):
    dev = dev_of(rank)
    peer = 1 - rank
    src = to_dev(payload(nbytes, seed=rank), dev)
    dst = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    from paper_2510_00991_b200 import P2POp
    for _ in range(iters):
        comm.batch_isend_irecv([P2POp("isend", src, peer), P2POp("irecv", dst, peer)])
    torch.cuda.synchronize()
    return {"recv": dst.cpu().numpy()}


def ring_shift(comm, rank, world, nbytes):
    dev = dev_of(rank)
    from paper_2510_00991_b200 import P2POp
    src = to_dev(payload(nbytes, seed=50 + rank), dev)
    dst = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    comm.batch_isend_irecv([P2POp("isend", src, (rank + 1) % world), P2POp("irecv", dst, (rank - 1) % world)])
    torch.cuda.synchronize()
    return {"recv": dst.cpu().numpy()}


def alltoallv_uneven(comm, rank, world, row_bytes, splits, seed=7):
    dev = dev_of(rank)
    send_rows = splits[rank]
    recv_rows = [splits[i][rank] for i in range(world)]
    src = to_dev(payload(sum(send_rows) * row_bytes, seed=seed + rank), dev).view(-1, row_bytes)
    dst = torch.zeros(sum(recv_rows), row_bytes, dtype=torch.uint8, device=dev)
    comm.alltoallv(dst, src, recv_rows, send_rows)
    torch.cuda.synchronize()
    return {"recv": dst.cpu().numpy().reshape(-1)}


def ll_mixed(comm, rank, world, sizes, rounds=3):
    """Small (LL kernel) and large (copy engine) messages interleaved in one
    group per round, both directions, more LL messages per pair than LL slots."""
    from paper_2510_00991_b200 import P2POp
    dev = dev_of(rank)
    peer = 1 - rank
    out = {}
    for rd in range(rounds):
        ops, recvs = [], []
        for i, n in enumerate(sizes):
            s = to_dev(payload(n, seed=10_000 * rank + 100 * rd + i), dev)
            r = torch.zeros(n + 3, dtype=torch.uint8, device=dev)[3:]  # misaligned destination
            ops += [P2POp("isend", s, peer), P2POp("irecv", r, peer)]
            recvs.append(r)
        comm.batch_isend_irecv(ops)
        torch.cuda.synchronize()
        for i, r in enumerate(recvs):
            out[f"r{rd}_{i}"] = r.cpu().numpy()
    for i, n in enumerate(sizes):  # single (ungrouped) LL ops, ordered send/recv
        s = to_dev(payload(n, seed=555 + i), dev)
        r = torch.zeros(n, dtype=torch.uint8, device=dev)
        if rank == 0:
            comm.send(s, 1)
            comm.recv(r, 1)
        else:
            comm.recv(r, 0)
            comm.send(s, 0)
        torch.cuda.synchronize()
        out[f"single_{i}"] = r.cpu().numpy()
    return out


def failover_pair(comm, rank, world, nbytes, fault_chunk, restore_us=0):
    """0 -> 1 with the primary copy path 0->1 Down at `fault_chunk` of the
    first send; the transfer must resume on the SM path at the breakpoint."""
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    src = payload(nbytes, seed=99)
    fs = FaultScript().down(0, 1, chunk=fault_chunk, op_index=0)
    if restore_us:
        fs.up(0, 1, t_us=restore_us)
    comm.set_faults(fs)
    out = {}
    if rank == 0:
        comm.send(to_dev(src, dev), 1)
    elif rank == 1:
        r = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        comm.recv(r, 0)
        torch.cuda.synchronize()
        out["recv"] = r.cpu().numpy()
    # any other rank only takes part as a possible relay GPU
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    # either endpoint may have issued the transfer (push by 0 or pull by 1),
    # and the issuer's watchdog is the one that switches
    ev = [e for e in comm.switch_events() if e["peer"] == 1 - rank]
    out["switch_to"] = np.array([0 if e["to"] == "primary" else 1 for e in ev], np.int32)
    out["resume"] = np.array([e["resume_chunk"] for e in ev], np.int32)
    out["detect_ns"] = np.array([e["detect_ns"] for e in ev], np.int64)
    return out


def relay_ring(comm, rank, world, nbytes, iters=2):
    """Every pair of the ring shift forced onto the backup path (relay GPU)
    through the API switch (switch_qp ToBackup), then back to the primary."""
    from paper_2510_00991_b200 import P2POp
    dev = dev_of(rank)
    to, frm = (rank + 1) % world, (rank - 1) % world
    comm.switch_qp(to, "ToBackup")
    out = {}
    for it in range(iters):
        src = to_dev(payload(nbytes, seed=70 + 10 * it + rank), dev)
        dst = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        comm.batch_isend_irecv([P2POp("isend", src, to), P2POp("irecv", dst, frm)])
        torch.cuda.synchronize()
        out[f"recv{it}"] = dst.cpu().numpy()
    out["path"] = np.array([0 if comm.active_path(to) == "primary" else 1], np.int32)
    out["relay_copies"] = np.array([comm.stats()["copies_issued"]], np.int64)
    comm.switch_qp(to, "ToPrimary")
    src = to_dev(payload(nbytes, seed=90 + rank), dev)
    dst = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    comm.batch_isend_irecv([P2POp("isend", src, to), P2POp("irecv", dst, frm)])
    torch.cuda.synchronize()
    out["recv_back"] = dst.cpu().numpy()
    return out


def direct_mixed(comm, rank, world, sizes, rounds=2):
    """Mid-size messages (the direct K6 path) both ways in one group per round,
    mixed with an LL and a copy-engine message, then as single ordered ops."""
    from paper_2510_00991_b200 import P2POp
    dev = dev_of(rank)
    peer = 1 - rank
    out = {}
    for rd in range(rounds):
        ops, recvs = [], []
        for i, n in enumerate(sizes):
            s = to_dev(payload(n, seed=20_000 * rank + 100 * rd + i), dev)
            r = torch.zeros(n + 16, dtype=torch.uint8, device=dev)[16:]
            ops += [P2POp("irecv", r, peer), P2POp("isend", s, peer)] if rank else \
                   [P2POp("isend", s, peer), P2POp("irecv", r, peer)]
            recvs.append(r)
        comm.batch_isend_irecv(ops)
        torch.cuda.synchronize()
        for i, r in enumerate(recvs):
            out[f"r{rd}_{i}"] = r.cpu().numpy()
    for i, n in enumerate(sizes):
        s = to_dev(payload(n, seed=777 + i), dev)
        r = torch.zeros(n, dtype=torch.uint8, device=dev)
        if rank == 0:
            comm.send(s, 1)
            comm.recv(r, 1)
        else:
            comm.recv(r, 0)
            comm.send(s, 0)
        torch.cuda.synchronize()
        out[f"single_{i}"] = r.cpu().numpy()
    out["kernels"] = np.array([comm.stats()["kernels_launched"]], np.int64)
    return out


def _records(comm):
    return [(r.size, r.peer, r.dir, r.path, r.chunk) for r in comm.monitor.drain()]


def failover_reuse(comm, rank, world, nbytes, fault_chunk, reps=1):
    """0 -> 1 with the primary path Down at `fault_chunk` of the first send
    (ADVICE r1 high).  Right after each op completes on its stream, the sender
    overwrites its source and the receiver copies the received bytes out and
    then overwrites its buffer with a marker: a stale or re-issued copy still
    in flight after completion would corrupt the copy-out (sender side) or the
    marker (receiver side)."""
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    comm.set_faults(FaultScript().down(0, 1, chunk=fault_chunk, op_index=0))
    out = {}
    s = torch.cuda.current_stream()
    for it in range(reps):
        if rank == 0:
            src = to_dev(payload(nbytes, seed=500 + it), dev)
            comm.send(src, 1)
            # a synchronous pageable copy behind the failing op: while it
            # waits, every other CUDA call of this process blocks — the
            # failover must not need one
            int(src[:1].cpu()[0])
            src.fill_(0x5A)  # stream-ordered after the send completed
        elif rank == 1:
            r = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
            comm.recv(r, 0)
            int(r[:1].cpu()[0])
            got = r.clone()        # stream-ordered after the recv completed
            r.fill_(0xA5)
            torch.cuda.synchronize()
            import time
            time.sleep(0.3)        # time for any late stale write to land
            torch.cuda.synchronize()
            out[f"recv{it}"] = got.cpu().numpy()
            out[f"marker_ok{it}"] = np.array([bool((r == 0xA5).all().item())])
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    ev = [e for e in comm.switch_events() if e["peer"] == 1 - rank]
    out["switch_to"] = np.array([0 if e["to"] == "primary" else 1 for e in ev], np.int32)
    out["resume"] = np.array([e["resume_chunk"] for e in ev], np.int32)
    return out


def fault_size_class(comm, rank, world, nbytes, fault_chunk):
    """One 0 -> 1 op of a size that would take K5 (LL) or K6 (direct) on a
    healthy pair, with a fault script naming the pair: the op must take the
    chunked path, stall at `fault_chunk`, switch and complete bit-exact; the
    monitor yields one record per chunk."""
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    comm.set_faults(FaultScript().down(0, 1, chunk=fault_chunk, op_index=0))
    out = {}
    stats0 = comm.stats()
    if rank == 0:
        comm.send(to_dev(payload(nbytes, seed=nbytes), dev), 1)
    elif rank == 1:
        r = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        comm.recv(r, 0)
        torch.cuda.synchronize()
        out["recv"] = r.cpu().numpy()
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    ev = [e for e in comm.switch_events() if e["peer"] == 1 - rank]
    out["switch_to"] = np.array([0 if e["to"] == "primary" else 1 for e in ev], np.int32)
    out["resume"] = np.array([e["resume_chunk"] for e in ev], np.int32)
    out["records"] = np.array([r[0] for r in _records(comm)], np.int64)
    st = comm.stats()
    out["ll_or_direct_kernels"] = np.array([st["kernels_launched"] - stats0["kernels_launched"]], np.int64)
    return out


def monitor_every_op(comm, rank, world, sizes):
    """Healthy pair, monitor on: every op of every size class (K5 LL, K6
    direct, copy engine) yields exactly one record (default chunk), and
    iccl_req_state reports each finished op as done."""
    from paper_2510_00991_b200 import P2POp
    dev = dev_of(rank)
    peer = 1 - rank
    out = {}
    works = []
    for i, n in enumerate(sizes):
        s = to_dev(payload(n, seed=30_000 * rank + i), dev)
        r = torch.zeros(n, dtype=torch.uint8, device=dev)
        ops = [P2POp("isend", s, peer), P2POp("irecv", r, peer)] if rank == 0 else \
              [P2POp("irecv", r, peer), P2POp("isend", s, peer)]
        works += comm.batch_isend_irecv(ops)
        torch.cuda.synchronize()
        out[f"r{i}"] = r.cpu().numpy()
    for i, n in enumerate(sizes):  # single ops too
        s = to_dev(payload(n, seed=40_000 + i), dev)
        r = torch.zeros(n, dtype=torch.uint8, device=dev)
        if rank == 0:
            works.append(comm.isend(s, 1))
            works.append(comm.irecv(r, 1))
        else:
            works.append(comm.irecv(r, 0))
            works.append(comm.isend(s, 0))
        torch.cuda.synchronize()
        out[f"s{i}"] = r.cpu().numpy()
    torch.cuda.synchronize()
    import time
    time.sleep(0.1)
    recs = _records(comm)
    out["rec_bytes"] = np.array(sorted(r[0] for r in recs), np.int64)
    states = [w.state() for w in works]
    out["state_done"] = np.array([s["done"] for s in states], np.int64)
    out["state_total"] = np.array([s["total_chunks"] for s in states], np.int64)
    return out


def api_switch_mid_size(comm, rank, world, sizes):
    """switch_qp ToBackup applies to every size class (K5/K6 sizes take the
    chunked backup path), then ToPrimary restores the fast paths."""
    dev = dev_of(rank)
    out = {}
    if rank == 0:
        comm.switch_qp(1, "ToBackup")
    import time
    time.sleep(0.05)
    for phase in range(2):
        for i, n in enumerate(sizes):
            if rank == 0:
                comm.send(to_dev(payload(n, seed=60_000 + 100 * phase + i), dev), 1)
            else:
                r = torch.zeros(n, dtype=torch.uint8, device=dev)
                comm.recv(r, 0)
                torch.cuda.synchronize()
                out[f"p{phase}_{i}"] = r.cpu().numpy()
        torch.cuda.synchronize()
        if phase == 0 and rank == 0:
            out["path_after_switch"] = np.array([1 if comm.active_path(1) == "backup" else 0], np.int32)
            comm.switch_qp(1, "ToPrimary")
        time.sleep(0.05)
    return out


def ll_route_toggle(comm, rank, world, n_msgs, size):
    """Small messages 0 -> 1 while rank 0 toggles the pair between primary and
    backup (switch_qp) every few sends: both sides must route each small op
    the same way (LL or rendezvous) or the op would hang."""
    dev = dev_of(rank)
    out = {}
    if rank == 0:
        for i in range(n_msgs):
            if i % 5 == 2:
                comm.switch_qp(1, "ToBackup" if (i // 5) % 2 == 0 else "ToPrimary")
            comm.send(to_dev(payload(size, seed=70_000 + i), dev), 1)
        comm.switch_qp(1, "ToPrimary")
    else:
        bufs = []
        for i in range(n_msgs):
            r = torch.zeros(size, dtype=torch.uint8, device=dev)
            comm.recv(r, 0)
            bufs.append(r)
        torch.cuda.synchronize()
        out["recv"] = np.stack([b.cpu().numpy() for b in bufs])
    torch.cuda.synchronize()
    return out


def register_deregister(comm, rank, world, nbytes):
    """MemoryRegion: register, send, deregister (peer closes its mapping),
    then a fresh buffer; UnregisteredRegion for a range past its allocation."""
    import ctypes as C
    from paper_2510_00991_b200._lib import lib
    dev = dev_of(rank)
    out = {}
    for it in range(3):
        if rank == 0:
            t = to_dev(payload(nbytes, seed=80_000 + it), dev)
            h = comm.register(t)
            comm.send(t, 1)
            torch.cuda.synchronize()
            import time
            time.sleep(0.05)
            comm.deregister(h)
        else:
            r = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
            comm.recv(r, 0)
            torch.cuda.synchronize()
            out[f"recv{it}"] = r.cpu().numpy()
    t = torch.zeros(1024, dtype=torch.uint8, device=dev)
    h = C.c_uint64()
    rc = lib.iccl_register(comm._h, C.c_void_p(t.data_ptr()), 1 << 40, C.byref(h))
    out["unregistered_rc"] = np.array([rc], np.int32)
    return out


def innocent_stall(comm, rank, world, trials, delta_us):
    """AC4 on the product: the pair is armed (a fault that never
    fires keeps it on the watchdog-covered chunked path); in every trial one
    side's stream is held upstream for 1.5-6 x delta by a device-side sleep
    before its op — the sender's data (or the receiver's buffer) is simply not
    ready.  No trial may switch paths, and every trial lands bit-exact."""
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    comm.set_faults(FaultScript().down(0, 1, chunk=0, op_index=1 << 30))
    rng = np.random.default_rng(4242)
    ok = []
    cycles_per_us = 1900
    for t in range(trials):
        n = int(rng.integers(1, 8 << 20))
        stall_us = int(delta_us * rng.uniform(1.5, 6.0))
        who = int(rng.integers(0, 2))  # 0: the sender is held upstream, 1: the receiver
        if rank == who:
            torch.cuda._sleep(stall_us * cycles_per_us)
        if rank == 0:
            comm.send(to_dev(payload(n, seed=90_000 + t), dev), 1)
        else:
            r = torch.empty(n, dtype=torch.uint8, device=dev)
            comm.recv(r, 0)
            ok.append(bool(torch.equal(r, to_dev(payload(n, seed=90_000 + t), dev))))
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    return {"ok": np.array(ok, bool), "switches": np.array([len(comm.switch_events())], np.int64)}


def monitor_accuracy(comm, rank, world, nchunks, chunk, stall_chunk, up_us):
    """AC5 on the product: rank 0 pushes `nchunks` chunks in one
    op, the monitor on.  With stall_chunk < 0 the flow is steady; otherwise the
    pair's primary path is gated at that chunk and re-opened `up_us` after the
    script is installed (a disturbance; delta is large, so no switch).  Returns
    the sender-side records (t1, t2, bytes)."""
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    n = nchunks * chunk
    out = {}
    src = to_dev(payload(n, seed=5), dev) if rank == 0 else None
    dst = torch.empty(n, dtype=torch.uint8, device=dev) if rank == 1 else None
    # warm-up op on the same tensors: the first use of a peer allocation
    # opens its IPC mapping (135 ms for this 2 GiB buffer on a B200 box),
    # which would delay the issue — and the Down — past the timed Up
    if rank == 0:
        comm.send(src, 1)
    else:
        comm.recv(dst, 0)
    torch.cuda.synchronize()
    import time
    time.sleep(0.5)  # the peer's proxy premaps the other tensor in the background
    comm.monitor.drain()
    # the Up is timed from the install: both ranks install together, right
    # before the op, so the Down (at the chunk's issue) always precedes it
    _store_barrier(comm, "ac5")
    if stall_chunk >= 0:
        comm.set_faults(FaultScript().down(0, 1, chunk=stall_chunk, op_index=0).up(0, 1, t_us=up_us))
    if rank == 0:
        comm.send(src, 1)
    else:
        comm.recv(dst, 0)
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    recs = [r for r in comm.monitor.drain() if r.peer == 1 - rank]
    recs.sort(key=lambda r: r.t2)
    out["t1"] = np.array([r.t1 for r in recs], np.int64)
    out["t2"] = np.array([r.t2 for r in recs], np.int64)
    out["bytes"] = np.array([r.size for r in recs], np.int64)
    ev = comm.switch_events()
    out["switches"] = np.array([len(ev)], np.int64)
    out["switch_desc"] = np.array([f"{e['trigger']}->{e['to']}@{e['resume_chunk']} after {e['detect_ns']} ns"
                                   for e in ev] or [""])
    if rank == 1:
        out["ok"] = np.array([bool(torch.equal(dst, to_dev(payload(n, seed=5), dev)))])
    return out


def monitor_competing(comm, rank, world, nchunks, chunk, comp_bytes, delay_us):
    """AC5's smoothing claim ("competing flow halving
    bandwidth mid-stream ... var(W=1) >= var(W=8) >= var(W=32)") on the
    product: rank 0 pushes `nchunks` chunks to rank 1 (copy engine, monitor
    on); `delay_us` later a second communicator with the SM transport pushes
    `comp_bytes` over the same link with K1 — SM stores and copy-engine
    writes share the link, while a GPU's copy engine would only queue a
    second copy behind the first.  With both ranks on one GPU (local copies)
    the competitor adds an HBM-bound stream of device copies.  Rank 1 posts
    its receives first, so rank 0 pushes and holds the monitored records."""
    import time
    import torch.distributed as dist
    from paper_2510_00991_b200 import Communicator, IcclConfig
    dev = dev_of(rank)
    n = nchunks * chunk
    one_gpu = torch.cuda.device_count() == 1
    comm2 = Communicator(rank, world, dev.index, IcclConfig.defaults(transport="sm", sm_cap=32, chunk_bytes=n),
                         store=dist.PrefixStore("competitor", comm._test_store))
    src = to_dev(payload(n, seed=6), dev) if rank == 0 else None
    src2 = to_dev(payload(comp_bytes, seed=7), dev) if rank == 0 else None
    dst = torch.empty(n, dtype=torch.uint8, device=dev) if rank == 1 else None
    dst2 = torch.empty(comp_bytes, dtype=torch.uint8, device=dev) if rank == 1 else None
    sa, sb, sc = (torch.cuda.Stream(device=dev) for _ in range(3))
    hammer = [torch.empty(1 << 30, dtype=torch.uint8, device=dev) for _ in range(2)] if rank == 0 and one_gpu else None

    def round_(tag, delay):
        if rank == 1:
            wa = comm.irecv(dst, 0, stream=sa)
            wb = comm2.irecv(dst2, 0, stream=sb)
            _store_barrier(comm, tag)
            wa.synchronize()
            wb.synchronize()
        else:
            _store_barrier(comm, tag)
            comm.send(src, 1)
            time.sleep(delay * 1e-6)
            if delay and one_gpu:
                with torch.cuda.stream(sc):
                    for _ in range(12):
                        hammer[0].copy_(hammer[1])
            comm2.send(src2, 1, stream=sb)
        torch.cuda.synchronize()

    round_("mc0", 0)          # warm-up: IPC mappings opened
    time.sleep(0.5)
    comm.monitor.drain()
    round_("mc1", delay_us)
    time.sleep(0.05)
    out = {}
    recs = sorted([r for r in comm.monitor.drain() if r.peer == 1], key=lambda r: r.t2)
    out["t1"] = np.array([r.t1 for r in recs], np.int64)
    out["t2"] = np.array([r.t2 for r in recs], np.int64)
    out["bytes"] = np.array([r.size for r in recs], np.int64)
    if rank == 1:
        out["ok"] = np.array([bool(torch.equal(dst, to_dev(payload(n, seed=6), dev))) and
                              bool(torch.equal(dst2, to_dev(payload(comp_bytes, seed=7), dev)))])
    torch.cuda.synchronize()
    comm2.destroy()
    return out


def moe_config4(comm, rank, world, T, k=8, E=64, H=7168, fault=None, keep_bytes=True, fused=False, reps=1,
                fused_combine=False):
    """BASELINE config 4 at `world` ranks: K2 pack (expand), dispatch
    alltoallv, combine alltoallv, K3 unpack, with the §8(d) routing and
    payload.  Checks on the device, at any size: every rank's received rows
    equal the rows every source rank routed to it (regenerated from the
    sources' seeds), and the combine round trip restores (token, k) order.
    With keep_bytes the packed send rows and the received rows come back for
    the oracle comparison.  `fault` = (src, dst, chunk): a FaultScript Down on
    that pair's primary path at that chunk of its first transfer (config 5).
    fused: the dispatch is K8 (moe_dispatch_fused) instead of K2 + alltoallv;
    `packed` is then built afterwards, for the oracle comparison only.  reps:
    the dispatch runs that many times (buffers reused, the last one checked)."""
    from paper_2510_00991_b200 import FaultScript
    from paper_2510_00991_b200.moe import (config4_routing, config4_tokens, expand_rows, moe_combine_fused,
                                           moe_dispatch_fused, plan_dispatch, scatter_rows)
    dev = dev_of(rank)
    experts = config4_routing(rank, T, k, E, dev)

    def exchange(send_counts):
        if world == 1:
            return list(send_counts)
        s = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        comm.alltoall(r, s)  # the one exchange step, through the product's own alltoall
        torch.cuda.synchronize()
        return r.tolist()

    plan = plan_dispatch(experts, E, world, exchange)
    tokens = config4_tokens(rank, T, H, dev)
    if fault is not None:
        comm.set_faults(FaultScript().down(fault[0], fault[1], chunk=fault[2], op_index=0))
    torch.cuda.synchronize()
    packed = torch.empty(T * k, H, dtype=tokens.dtype, device=dev)
    recv = torch.empty(sum(plan.recv_counts), H, dtype=tokens.dtype, device=dev)
    back = torch.empty_like(packed)
    out = torch.empty_like(packed)
    for _ in range(reps):
        if fused:
            recv.fill_(0)
            moe_dispatch_fused(comm, tokens, plan, recv)
        else:
            expand_rows(tokens, plan.pos, k, packed)
            comm.alltoallv(recv, packed, plan.recv_counts, plan.send_counts)
    if fused:
        expand_rows(tokens, plan.pos, k, packed)
    if fused_combine:
        for _ in range(reps):
            out.fill_(0)
            moe_combine_fused(comm, recv, plan, T, k, out)
    else:
        comm.alltoallv(back, recv, plan.send_counts, plan.recv_counts)
        scatter_rows(back, plan.order, out)
    torch.cuda.synchronize()
    # device-side expected rows: what every source i routed to this rank
    per_rank = E // world
    exp = []
    for i in range(world):
        ex_i = config4_routing(i, T, k, E, dev).reshape(-1)
        order_i = torch.sort(ex_i, stable=True).indices
        mine = torch.div(ex_i[order_i], per_rank, rounding_mode="floor") == rank
        exp.append(config4_tokens(i, T, H, dev)[torch.div(order_i[mine], k, rounding_mode="floor")])
    exp = torch.cat(exp)
    res = {"recv_ok": np.array([bool(torch.equal(recv.view(torch.int16), exp.view(torch.int16)))]),
           "roundtrip_ok": np.array([bool(torch.equal(out.view(T, k, H).view(torch.int16),
                                                      tokens.view(torch.int16).unsqueeze(1).expand(T, k, H)))]),
           "send_counts": np.array(plan.send_counts, np.int64)}
    if keep_bytes:
        res["packed"] = packed.view(torch.uint8).cpu().numpy().reshape(-1)
        res["recv"] = recv.view(torch.uint8).cpu().numpy().reshape(-1)
    import time
    time.sleep(0.05)
    ev = comm.switch_events()
    res["switch_peers"] = np.array([e["peer"] for e in ev], np.int64)
    res["switch_to"] = np.array([0 if e["to"] == "primary" else 1 for e in ev], np.int64)
    res["records"] = np.array([len(comm.monitor.drain())], np.int64)
    res["kernels"] = np.array([comm.stats()["kernels_launched"]], np.int64)
    return res


def _store_barrier(comm, tag):
    import time
    st = comm._test_store
    st.add(tag, 1)
    while int(st.add(tag, 0)) < comm.world_size:
        time.sleep(0.0002)


def _wait_retired(comm, timeout_s=5.0):
    import time
    t0 = time.time()
    while comm.stats()["pending_xfers"] and time.time() - t0 < timeout_s:
        time.sleep(0.0005)


def fuzz_failover(comm, rank, world, trials, seed, delta_us):
    """AC3 on the product: `trials` randomised 0 -> 1 transfers,
    sizes log-uniform 1 KiB - 64 MiB, chunk sizes 16 KiB - 4 MiB, and a fault
    script per trial: the primary Down at a random chunk (or at a chunk past
    the end: armed, never fires), Down before the op (time-triggered), or Down
    at a chunk and restored (Up) at a random time around delta.  Before each
    trial the primary is restored and the pair is back on it.  Per trial the
    receiver checks the bytes on its GPU, and both sides return the chunk
    indices of their monitor records for the op (the delivered sequence: the
    test checks it is 0..N-1, gapless and duplicate-free) and the sender's
    six-pointer state.  Payloads are generated on the GPU from a seeded
    generator on both sides (the same Philox stream)."""
    import time
    from paper_2510_00991_b200 import FaultScript
    dev = dev_of(rank)
    peer = 1 - rank
    out = {"n": [], "nchunks": [], "mode": [], "ok": [], "state_done": [], "state_total": []}
    chunks_all, chunks_off = [], [0]
    for t in range(trials):
        rng = np.random.default_rng(seed + t)
        size = min(64 << 20, int(2.0 ** rng.uniform(10.0, 26.0)))
        chunk = 1 << int(rng.integers(14, 23))
        while (size + chunk - 1) // chunk > 256:
            chunk <<= 1
        nch = (size + chunk - 1) // chunk
        mode = int(rng.integers(0, 4))
        f = int(rng.integers(0, nch + 1))
        # restore the primary a previous trial left Down, and wait until the
        # pair is back on it (monitor_failed_link's probe)
        comm.set_faults(FaultScript().up(0, 1, t_us=0))
        time.sleep(0.002)
        if rank == 0:
            t0 = time.time()
            while comm.active_path(1) != "primary" and time.time() - t0 < 10:
                time.sleep(0.0005)
        _store_barrier(comm, f"fz{t}a")
        fs = FaultScript()
        if mode == 0:
            fs.down(0, 1, chunk=f, op_index=0)
        elif mode == 1:
            fs.down(0, 1, t_us=0)
        elif mode == 2:
            fs.down(0, 1, chunk=f, op_index=0).up(0, 1, t_us=int(delta_us * rng.uniform(0.2, 4.0)))
        comm.set_faults(fs)  # mode 3: an empty script (the pair is healthy)
        comm.set_chunk_bytes(chunk)
        if mode == 1:
            time.sleep(0.001)
        _store_barrier(comm, f"fz{t}b")
        comm.monitor.drain()
        g = torch.Generator(device=dev)
        g.manual_seed(seed * 7919 + t)
        ref = torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev, generator=g)
        if rank == 0:
            w = comm.isend(ref, 1)
        else:
            r = torch.full((size,), 0xEE, dtype=torch.uint8, device=dev)
            w = comm.irecv(r, 0)
        torch.cuda.synchronize()
        _wait_retired(comm)
        _store_barrier(comm, f"fz{t}c")
        _wait_retired(comm)
        st = w.state()
        recs = [x for x in comm.monitor.drain() if x.peer == peer]
        chunks_all.extend(x.chunk for x in recs)
        chunks_off.append(len(chunks_all))
        out["n"].append(size)
        # a healthy pair (mode 3) sends <= direct_max_kib through K5 / K6: one record, one chunk
        out["nchunks"].append(1 if mode == 3 and size <= comm.config.direct_max_kib * 1024 else nch)
        out["mode"].append(mode)
        out["ok"].append(rank == 0 or bool(torch.equal(r, ref)))
        out["state_done"].append(st["done"])
        out["state_total"].append(st["total_chunks"])
    comm.set_faults(FaultScript().up(0, 1, t_us=0))
    res = {k: np.array(v) for k, v in out.items()}
    res["chunks"] = np.array(chunks_all, np.int64)
    res["chunks_off"] = np.array(chunks_off, np.int64)
    return res


def pp_1f1b(comm, rank, world, M, T=64, H=256):
    """Megatron's non-interleaved 1F1B schedule (benchmarks/pp_1f1b.py: fused
    send_forward_recv_backward / send_backward_recv_forward as one batched
    isend/irecv on a communication stream, GEMMs on the compute stream) on
    small activations.  Every sent tensor's bytes are published through the
    store under (src, dst, direction, microbatch); every received tensor is
    compared with them.  Returns the number of matching / total receives."""
    import paper_2510_00991_b200 as iccl
    dev = dev_of(rank)
    st = comm._test_store
    S = world
    first, last = rank == 0, rank == S - 1
    g = torch.Generator(device=dev).manual_seed(10 + rank)
    W = torch.randn(H, H, dtype=torch.bfloat16, device=dev, generator=g) * 0.05
    x0 = torch.randn(T, H, dtype=torch.bfloat16, device=dev, generator=g)
    comp = torch.cuda.current_stream()
    cstream = torch.cuda.Stream(device=dev)
    sent = {"f": 0, "b": 0}
    got = {"f": 0, "b": 0}
    checks = []

    def exchange(sends, recvs):
        cstream.wait_stream(comp)
        outs = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in recvs]
        with torch.cuda.stream(cstream):
            ops = [iccl.P2POp("isend", t, p) for t, p, _ in sends] + \
                  [iccl.P2POp("irecv", o, p) for o, (p, _) in zip(outs, recvs)]
            comm.batch_isend_irecv(ops, stream=cstream)
        cstream.synchronize()
        for t, p, d in sends:
            st.set(f"pp/{rank}/{p}/{d}/{sent[d]}", t.view(torch.int16).cpu().numpy().tobytes())
            sent[d] += 1
        for o, (p, d) in zip(outs, recvs):
            want = st.get(f"pp/{p}/{rank}/{d}/{got[d]}")
            checks.append(o.view(torch.int16).cpu().numpy().tobytes() == want)
            got[d] += 1
        comp.wait_stream(cstream)
        return outs

    def forward(x):
        return (x0 if x is None else x) @ W

    def backward(dy):
        return dy @ W.t()

    warm = min(S - rank - 1, M)
    for _ in range(warm):
        x = None if first else exchange([], [(rank - 1, "f")])[0]
        exchange([(forward(x), rank + 1, "f")], [])
    steady = M - warm
    x = None if (first or steady == 0) else exchange([], [(rank - 1, "f")])[0]
    for i in range(steady):
        y = forward(x)
        dy = y if last else exchange([(y, rank + 1, "f")], [(rank + 1, "b")])[0]
        dx = backward(dy)
        if i == steady - 1:
            if not first:
                exchange([(dx, rank - 1, "b")], [])
        elif first:
            x = None
        else:
            x = exchange([(dx, rank - 1, "b")], [(rank - 1, "f")])[0]
    for _ in range(warm):
        dy = exchange([], [(rank + 1, "b")])[0]
        dx = backward(dy)
        if not first:
            exchange([(dx, rank - 1, "b")], [])
    torch.cuda.synchronize()
    return {"ok": np.array([sum(checks)]), "n": np.array([len(checks)])}
