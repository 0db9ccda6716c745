#!/usr/bin/env python
"""1F1B pipeline-parallel harness on real B200s.

The paper's training gain comes from overlapping PP send/recv with compute
without stealing SMs from it (SPEC.md:500-517
``enforce_order`` / ``run_1f1b``).  Every rank is one stage; each microbatch
carries a bf16 [4, 4096, 8192] activation (256 MiB, config 3's hop).  Stage
compute is a cuBLAS bf16 GEMM chain on the compute stream (forward: one
[16384, 8192] x [8192, 8192] GEMM, backward: two), P2P runs on a separate
communication stream and the compute stream waits only for the activation /
gradient it consumes — so communication overlaps the neighbouring
microbatches' compute.

Schedule (non-interleaved 1F1B): stage s runs min(S - s - 1, M) warm-up
forwards, then alternates one forward / one backward, then drains the
backwards.  Metric: iteration time for M microbatches (max over ranks,
device-timed) and achieved TFLOP/s per GPU; ``--impl nccl`` runs the same
schedule with torch.distributed isend/irecv on NCCL (its kernels take SMs
from the GEMMs), ``--impl iccl`` the copy-engine path (0 SMs).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        benchmarks/pp_1f1b.py --impl iccl
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["iccl", "nccl"], required=True)
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    S, M = world, args.microbatches
    T, H = 4 * 4096, 8192
    comm = None
    if args.impl == "iccl":
        import paper_2510_00991_b200 as iccl
        comm = iccl.init(rank, world, local, iccl.IcclConfig.defaults())
    g = torch.Generator(device=dev).manual_seed(10 + rank)
    W = torch.randn(H, H, dtype=torch.bfloat16, device=dev, generator=g) * 0.01
    comp = torch.cuda.current_stream()
    # one communication stream per (direction, peer): every stream carries one
    # ordered pair's ops in FIFO order, so no op waits behind another pair's
    streams = {}

    def stream_for(kind, peer):
        if (kind, peer) not in streams:
            streams[(kind, peer)] = torch.cuda.Stream(device=dev)
        return streams[(kind, peer)]
    # per-microbatch buffers: activation in / out, gradient in / out
    act_in = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    act_out = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    grad_in = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    grad_out = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    x0 = torch.randn(T, H, dtype=torch.bfloat16, device=dev, generator=g)
    tmp = torch.empty(T, H, dtype=torch.bfloat16, device=dev)

    def p2p(kind, t, peer):
        """Enqueue on the pair's comm stream after the compute that produced t; return an event."""
        cstream = stream_for(kind, peer)
        if kind == "send":
            cstream.wait_stream(comp)  # the data is produced by the compute stream; a recv posts early
        with torch.cuda.stream(cstream):
            if comm:
                (comm.isend if kind == "send" else comm.irecv)(t, peer, stream=cstream)
            else:
                op = dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer)
                for w in dist.batch_isend_irecv([op]):
                    w.wait()
            t.record_stream(cstream)
        ev = torch.cuda.Event()
        ev.record(cstream)
        return ev

    def forward(i):
        if rank > 0:
            comp.wait_event(p2p("recv", act_in[i], rank - 1))
            src = act_in[i]
        else:
            src = x0
        torch.matmul(src, W, out=act_out[i])
        if rank < S - 1:
            p2p("send", act_out[i], rank + 1)

    def backward(i):
        if rank < S - 1:
            comp.wait_event(p2p("recv", grad_in[i], rank + 1))
            gsrc = grad_in[i]
        else:
            gsrc = act_out[i]
        torch.matmul(gsrc, W.t(), out=grad_out[i])   # dX
        torch.matmul(gsrc, W, out=tmp)               # stands in for dW (same flops)
        if rank > 0:
            p2p("send", grad_out[i], rank - 1)

    def iteration():
        warm = min(S - rank - 1, M)
        f = b = 0
        for _ in range(warm):
            forward(f)
            f += 1
        while f < M:
            forward(f)
            f += 1
            backward(b)
            b += 1
        while b < M:
            backward(b)
            b += 1
        for cs in streams.values():
            comp.wait_stream(cs)

    for _ in range(args.warmup):
        iteration()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(args.iters):
        iteration()
    e1.record(comp)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops = M * 3 * 2.0 * T * H * H  # per GPU per iteration: 1 forward + 2 backward GEMMs per microbatch
    res = {"bench": "pp_1f1b", "impl": args.impl, "stages": S, "microbatches": M, "ms_per_iter": round(ms, 3),
           "tflops_per_gpu": round(flops / (ms * 1e-3) / 1e12, 1),
           "hop_bytes": T * H * 2, "gemm": f"[{T},{H}]x[{H},{H}] bf16 (1 fwd + 2 bwd per microbatch)"}
    if comm:
        res["iccl_stats"] = comm.stats()
        comm.destroy()
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
