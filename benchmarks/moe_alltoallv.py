#!/usr/bin/env python
"""Config 4 comparison: MoE expert-parallel dispatch + combine alltoallv,
ICCL copy-engine path vs same-box NCCL (torch ``all_to_all_single``), the
comparison the paper makes for alltoall (NCCL holds 24.7% of
the SMs at 8x8).

T=4096 tokens per rank, top-8 of 64 experts (8 per rank at 8 ranks), hidden
7168 bf16 (14,336 B per row), skewed routing p_e ~ (e+1)^-0.8,
so the splits are uneven.  One step = dispatch alltoallv + combine alltoallv
(the reverse, same counts); the round trip must return every row bit for bit.

Bound: t* = 2 x max_i max(egress_i, ingress_i) / 770 GB/s (NVLink per
direction, measured peer-copy peak; the self segment is a local copy).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        benchmarks/moe_alltoallv.py --impl iccl
"""
import argparse
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["iccl", "nccl"], required=True)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dump-records", action="store_true", help="monitor on; print rank 0's chunk records of one step")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from bench import moe_routing
    T, k, E, H = 4096, 8, 64, 7168
    row = 2 * H
    experts = moe_routing(rank, world, T, k, E, dev)
    dest = torch.div(experts.reshape(-1), E // world, rounding_mode="floor")
    send = torch.bincount(dest, minlength=world)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    sc, rc = send.tolist(), recv.tolist()
    g = torch.Generator(device=dev).manual_seed(3000 + rank)
    packed = torch.randint(-32768, 32767, (sum(sc), H), dtype=torch.int16, device=dev, generator=g).view(
        torch.bfloat16)  # NCCL has no int16; bits compared as int16 below
    inbox = torch.empty(sum(rc), H, dtype=torch.bfloat16, device=dev)
    back = torch.empty_like(packed)
    comm = None
    if args.impl == "iccl":
        import paper_2510_00991_b200 as iccl
        comm = iccl.init(rank, world, local, iccl.IcclConfig.defaults(monitor_enabled=args.dump_records))

    def step():
        if comm:
            comm.alltoallv(inbox, packed, rc, sc)
            comm.alltoallv(back, inbox, sc, rc)
        else:
            dist.all_to_all_single(inbox, packed, rc, sc)
            dist.all_to_all_single(back, inbox, sc, rc)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ok = torch.equal(back.view(torch.int16), packed.view(torch.int16))
    s0 = comm.stats() if comm else None
    dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    eg = (sum(sc) - sc[rank]) * row
    ig = (sum(rc) - rc[rank]) * row
    lim = torch.tensor([max(eg, ig)], device=dev, dtype=torch.float64)
    tot = torch.tensor([2.0 * (eg + ig) / 2], device=dev, dtype=torch.float64)  # NVLink bytes per step
    okt = torch.tensor([1.0 if ok else 0.0], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(lim, op=dist.ReduceOp.MAX)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    ms = float(t.item())
    t_star = 2 * float(lim.item()) / 770e9
    res = {"bench": "moe_alltoallv", "impl": args.impl, "n_gpus": world, "ms_per_step": round(ms, 4),
           "nvlink_GBps_total": round(float(tot.item()) / (ms * 1e-3) / 1e9, 1),
           "t_star_ms": round(t_star * 1e3, 4), "frac_of_bound": round(t_star / (ms * 1e-3), 4),
           "max_rank_egress_or_ingress_MiB": round(float(lim.item()) / 2**20, 1),
           "bit_exact_roundtrip": bool(okt.item() > 0), "send_rows_rank0": sc,
           "step": "dispatch alltoallv + combine alltoallv (same counts, reversed)"}
    if comm and args.dump_records:
        comm.monitor.drain()
        torch.cuda.synchronize()
        dist.barrier()
        step()
        torch.cuda.synchronize()
        import time
        time.sleep(0.01)
        recs = comm.monitor.drain()
        t0 = min(r.t1 for r in recs) if recs else 0
        res[f"records_rank{rank}"] = [(r.peer, r.dir, r.op_seq, r.size >> 20, round((r.t1 - t0) / 1e3, 1),
                                       round((r.t2 - t0) / 1e3, 1)) for r in recs]
        for r_ in range(world):
            if r_ == rank and rank != 0:
                print(json.dumps({"rank": rank, "records": res[f"records_rank{rank}"]}), flush=True)
    if comm:
        s1 = comm.stats()
        res["kernels_launched"] = s1["kernels_launched"] - s0["kernels_launched"]
        res["rank0_pulls_issued"] = s1["pulls_issued"] - s0["pulls_issued"]
        res["rank0_cts_timeouts"] = s1["cts_timeouts"] - s0["cts_timeouts"]
        comm.destroy()
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
