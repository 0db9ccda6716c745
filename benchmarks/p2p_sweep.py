#!/usr/bin/env python
"""Config 2: send/recv bandwidth + latency sweep, 8 B .. 1 GiB, 2 ranks on
2 x B200: the ICCL copy-engine path, the ICCL SM path (K1 / LL kernel) and
same-box NCCL (torch.distributed, NCCL 2.28.9) — the comparison the paper
makes.

NCCL runs in the three modes the paper's comparison must cover:
``nccl`` (default, SM kernels), ``nccl-ce`` (NCCL_P2P_USE_CUDA_MEMCPY=1, its
own copy-engine P2P) and ``nccl-zero`` (NCCL_CTA_POLICY=2, the zero-CTA
policy of nccl.h:66).  ``--bidir`` times both directions at once (each rank
sends and receives in one batched group).

Two regimes per size, both nccl-tests style (device time, max over ranks):
* ``gpu``: the whole loop is enqueued behind a ~30 ms device sleep, so the
  GPU runs the ops back to back — per-op device time, host API cost hidden;
* ``api``: plain loop — includes the host cost of every call when the host
  cannot run ahead.
Bandwidth: K back-to-back 0->1 sends; latency: half the 0->1->0 ping-pong,
from the difference of two loop lengths (cancels the start skew).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        benchmarks/p2p_sweep.py --impl iccl-ce
"""
import argparse
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["iccl-ce", "iccl-sm", "iccl-auto", "nccl", "nccl-ce", "nccl-zero"],
                    required=True)
    ap.add_argument("--bidir", action="store_true", help="both directions at once (batched isend + irecv)")
    ap.add_argument("--min-pow", type=int, default=3)
    ap.add_argument("--max-pow", type=int, default=30)
    ap.add_argument("--step", type=int, default=1)
    ap.add_argument("--out", default="")
    ap.add_argument("--chunk-bytes", type=int, default=0)
    ap.add_argument("--ll-bytes", type=int, default=-1)
    ap.add_argument("--armed", action="store_true",
                    help="install a fault script on pair 0->1 that never fires: its ops take the failover-capable path")
    ap.add_argument("--records", action="store_true", help="window monitor on")
    ap.add_argument("--backup-path", action="store_true",
                    help="switch_qp both directions to the backup path first (the SM-kernel K1 path): its bandwidth "
                         "as a fraction of the primary's is the paper's backup retention")
    args = ap.parse_args()
    if args.impl == "nccl-ce":
        os.environ["NCCL_P2P_USE_CUDA_MEMCPY"] = "1"
    elif args.impl == "nccl-zero":
        os.environ["NCCL_CTA_POLICY"] = "2"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    peer = 1 - rank
    comm = None
    if args.impl.startswith("iccl"):
        import paper_2510_00991_b200 as iccl
        cfg = iccl.IcclConfig.defaults(transport=args.impl.split("-")[1])
        if args.chunk_bytes:
            cfg.chunk_bytes = args.chunk_bytes
        if args.ll_bytes >= 0:
            cfg.sm_small_bytes = args.ll_bytes
        cfg.monitor_enabled = bool(args.records)
        comm = iccl.init(rank, world, local, cfg)
        if args.armed:
            comm.set_faults(iccl.FaultScript().down(0, 1, chunk=1 << 30, op_index=1 << 30))
        if args.backup_path:
            comm.switch_qp(peer, "ToBackup")

    def send(t):
        comm.send(t, peer) if comm else dist.send(t, peer)

    def recv(t):
        comm.recv(t, peer) if comm else dist.recv(t, peer)

    maxb = 1 << args.max_pow
    g = torch.Generator(device=dev).manual_seed(7)
    buf = torch.randint(0, 255, (maxb,), dtype=torch.uint8, device=dev, generator=g)
    rbuf = torch.zeros(maxb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    cycles_per_ms = 1.9e6  # ~1.9 GHz

    def timed(fn, iters, pre_sleep):
        torch.cuda.synchronize()
        dist.barrier()
        if pre_sleep:
            torch.cuda._sleep(int(30 * cycles_per_ms))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3  # us

    def both(s, r):
        if comm:
            comm.batch_isend_irecv([iccl.P2POp("isend", s, peer), iccl.P2POp("irecv", r, peer)])
        else:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, s, peer), dist.P2POp(dist.irecv, r, peer)]):
                w.wait()

    def bw_loop(s, r):
        if args.bidir:
            return lambda: both(s, r)
        return lambda: send(s) if rank == 0 else recv(r)

    def pp_loop(s, r):
        def f():
            if rank == 0:
                send(s)
                recv(r)
            else:
                recv(r)
                send(s)
        return f

    out = []
    for p in range(args.min_pow, args.max_pow + 1, args.step):
        n = 1 << p
        s, r = buf[:n], rbuf[:n]
        iters = 100 if n <= (4 << 20) else (30 if n <= (64 << 20) else 10)
        for _ in range(3):
            pp_loop(s, r)()
        rec = {"impl": args.impl, "bytes": n, "bidir": bool(args.bidir), "armed": bool(args.armed),
               "monitor": bool(args.records), "chunk_bytes": args.chunk_bytes, "path": "backup" if args.backup_path
               else "primary"}
        if comm:
            comm.monitor.drain()
        for mode, pre in (("gpu", True), ("api", False)):
            t = torch.tensor([timed(bw_loop(s, r), iters, pre) / iters], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            per_op = float(t.item())
            k1, k2 = max(4, iters // 4), max(12, iters)
            t1 = timed(pp_loop(s, r), k1, pre)
            t2 = timed(pp_loop(s, r), k2, pre)
            lat = (t2 - t1) / (2 * (k2 - k1))
            rec[f"{mode}_us_per_op"] = round(per_op, 3)
            rec[f"{mode}_GBps"] = round(n / per_op / 1e3, 2)
            rec[f"{mode}_lat_us"] = round(lat, 3)
        torch.cuda.synchronize()
        if comm:
            # SMs used: CTAs the library launched per 0->1 transfer, both ranks summed
            st0 = comm.stats()
            for _ in range(4):
                bw_loop(s, r)()
            torch.cuda.synchronize()
            st1 = comm.stats()
            d = torch.tensor([st1["ctas_launched"] - st0["ctas_launched"],
                              st1["kernels_launched"] - st0["kernels_launched"]], device=dev, dtype=torch.float64)
            dist.all_reduce(d)
            rec["ctas_per_op"] = float(d[0].item()) / 4
            rec["kernels_per_op"] = float(d[1].item()) / 4
        if rank == 1 or args.bidir:
            ok = torch.equal(rbuf[:n], buf[:n])
            okt = torch.tensor([1 if ok else 0], device=dev)
        else:
            okt = torch.tensor([1], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        rec["bit_exact"] = bool(okt.item())
        out.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)
    if comm:
        st = comm.stats()
        if rank == 0:
            print(json.dumps({"impl": args.impl, "stats": st}), flush=True)
        comm.destroy()
    if rank == 0 and args.out:
        with open(args.out, "a") as fh:
            for rec in out:
                fh.write(json.dumps(rec) + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
