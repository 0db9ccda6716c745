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
