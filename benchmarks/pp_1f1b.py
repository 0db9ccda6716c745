#!/usr/bin/env python
"""1F1B pipeline-parallel harness on real B200s.

The paper's training gain comes from overlapping PP send/recv with compute
without stealing SMs from it (SPEC.md:500-517
``enforce_order`` / ``run_1f1b``).  Every rank is one stage; each microbatch
carries a bf16 [4, 4096, 8192] activation (256 MiB, config 3's hop).  Stage
compute is a cuBLAS bf16 GEMM chain on the compute stream (forward: one
[16384, 8192] x [8192, 8192] GEMM, backward: two).

Schedule: Megatron's non-interleaved 1F1B with its fused exchanges —
``send_forward_recv_backward`` / ``send_backward_recv_forward`` are one
batched isend/irecv each (the pattern that keeps NCCL deadlock-free) — on a
communication stream; the compute stream waits only for the tensor it
consumes.  Metric: iteration time for M microbatches (max over ranks,
device-timed) and achieved TFLOP/s per GPU.  ``--impl nccl`` runs the
identical schedule with ``torch.distributed.batch_isend_irecv`` on NCCL (its
kernels take SMs from the GEMMs), ``--impl iccl`` the copy-engine path (0 SMs).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        benchmarks/pp_1f1b.py --impl iccl
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
    first, last = rank == 0, rank == S - 1
    comm = None
    iccl = None
    if args.impl == "iccl":
        import paper_2510_00991_b200 as iccl
        comm = iccl.init(rank, world, local, iccl.IcclConfig.defaults())
    g = torch.Generator(device=dev).manual_seed(10 + rank)
    W = torch.randn(H, H, dtype=torch.bfloat16, device=dev, generator=g) * 0.01
    comp = torch.cuda.current_stream()
    cstream = torch.cuda.Stream(device=dev)
    pool = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(8)]
    x0 = torch.randn(T, H, dtype=torch.bfloat16, device=dev, generator=g)
    tmp = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    nxt = [0]

    def buf():
        b = pool[nxt[0] % len(pool)]
        nxt[0] += 1
        return b

    def exchange(sends, recvs):
        """One batched isend/irecv on the comm stream after the compute that
        produced the sends; the compute stream then waits for the received
        tensors, which are returned."""
        cstream.wait_stream(comp)
        outs = [buf() for _ in recvs]
        with torch.cuda.stream(cstream):
            if comm:
                ops = [iccl.P2POp("isend", t, p) for t, p in sends] + \
                      [iccl.P2POp("irecv", o, p) for o, p in zip(outs, recvs)]
                comm.batch_isend_irecv(ops, stream=cstream)
            else:
                ops = [dist.P2POp(dist.isend, t, p) for t, p in sends] + \
                      [dist.P2POp(dist.irecv, o, p) for o, p in zip(outs, recvs)]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for t, _ in sends:
                t.record_stream(cstream)
        if recvs:
            comp.wait_stream(cstream)
        return outs

    def forward(x):
        y = buf()
        torch.matmul(x0 if x is None else x, W, out=y)
        return y

    def backward(dy):
        dx = buf()
        torch.matmul(dy, W.t(), out=dx)   # dX
        torch.matmul(dy, W, out=tmp)      # stands in for dW (same flops)
        return dx

    def iteration():
        warm = min(S - rank - 1, M)
        for _ in range(warm):
            x = None if first else exchange([], [rank - 1])[0]              # recv_forward
            y = forward(x)
            exchange([(y, rank + 1)], [])                                     # send_forward
        steady = M - warm
        x = None if (first or steady == 0) else exchange([], [rank - 1])[0]
        for i in range(steady):
            y = forward(x)
            dy = y if last else exchange([(y, rank + 1)], [rank + 1])[0]     # send_forward_recv_backward
            dx = backward(dy)
            if i == steady - 1:
                if not first:
                    exchange([(dx, rank - 1)], [])                            # send_backward
            elif first:
                x = None
            else:
                x = exchange([(dx, rank - 1)], [rank - 1])[0]                # send_backward_recv_forward
        for _ in range(warm):
            dy = exchange([], [rank + 1])[0]                                  # recv_backward
            dx = backward(dy)
            if not first:
                exchange([(dx, rank - 1)], [])                                # send_backward
        comp.wait_stream(cstream)

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
