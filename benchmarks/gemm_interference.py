#!/usr/bin/env python
"""Config 3: pipeline-parallel activation send/recv (bf16 [4,4096,8192],
256 MiB per hop, ring shift over all ranks) overlapped with a cuBLAS bf16
8192^3 GEMM on the compute stream.  Metric: GEMM slowdown =
t_gemm(with comm) / t_gemm(alone) - 1, ABAB-interleaved, median and a 95%
bootstrap CI.  The SPEC's SM-pool model predicts +30% for an NCCL-style P2P
that holds 23.1% of the SMs; the copy-engine path holds
none.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        benchmarks/gemm_interference.py --impl iccl-ce
"""
import argparse
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import random
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["iccl-ce", "iccl-sm", "iccl-auto", "nccl", "none"], required=True)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--gemms", type=int, default=4)
    ap.add_argument("--msg-mib", type=float, default=256.0,
                    help="P2P message per hop (256 = config 3's activation; 1-16 = the K6 mid-size band)")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = None
    if args.impl.startswith("iccl"):
        import paper_2510_00991_b200 as iccl
        comm = iccl.init(rank, world, local, iccl.IcclConfig.defaults(transport=args.impl.split("-")[1]))
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    nel = int(args.msg_mib * (1 << 20)) // 2
    act = torch.randint(-32768, 32767, (nel,), dtype=torch.int16, device=dev).view(torch.bfloat16)
    rcv = torch.empty_like(act)
    comp = torch.cuda.Stream(device=dev)
    cs = torch.cuda.Stream(device=dev)
    to, frm = (rank + 1) % world, (rank - 1) % world

    def comm_burst(n):
        with torch.cuda.stream(cs):
            for _ in range(n):
                if comm is not None:
                    import paper_2510_00991_b200 as iccl
                    comm.batch_isend_irecv([iccl.P2POp("isend", act, to), iccl.P2POp("irecv", rcv, frm)], stream=cs)
                elif args.impl == "nccl":
                    ops = [dist.P2POp(dist.isend, act, to), dist.P2POp(dist.irecv, rcv, frm)]
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()

    def timed_gemms():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(comp):
            e0.record(comp)
            for _ in range(args.gemms):
                torch.matmul(a, b, out=c)
            e1.record(comp)
        return e0, e1

    for _ in range(3):
        timed_gemms()
        if args.impl != "none":
            comm_burst(2)
    torch.cuda.synchronize()
    # bursts long enough to cover the GEMM window (~3.2 ms): ~4 ms of transfers
    burst = max(12, int(12 * 256 / max(args.msg_mib, 0.001) * 0.25)) if args.msg_mib < 256 else 12
    burst = min(burst, 4000)
    # attribution: SM clock and board power sampled (NVML, every ~2 ms) in
    # each phase, so a slowdown can be told apart as a clock/power effect
    # (the power cap pulls the SM clock down when the copy engines and HBM
    # draw more) or as contention at the same clock
    samp = {"A": [], "B": []}
    phase = ["-"]
    stop = [False]
    import threading
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)

        def sampler():
            import time as _t
            while not stop[0]:
                p = phase[0]
                if p in samp:
                    samp[p].append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
                _t.sleep(0.002)
        th = threading.Thread(target=sampler, daemon=True)
        th.start()
    except Exception:
        th = None
    alone, withc = [], []
    order = ["A", "B"] * args.reps
    for ph in order:
        torch.cuda.synchronize()
        dist.barrier()
        phase[0] = ph
        if ph == "B" and args.impl != "none":
            comm_burst(burst)
        e0, e1 = timed_gemms()
        torch.cuda.synchronize()
        phase[0] = "-"
        (alone if ph == "A" else withc).append(e0.elapsed_time(e1) / args.gemms)
    stop[0] = True
    if th is not None:
        th.join()
    ratios = [b_ / a_ - 1 for a_, b_ in zip(alone, withc)]
    med = statistics.median(ratios)
    rnd = random.Random(0)
    boots = sorted(statistics.median(rnd.choices(ratios, k=len(ratios))) for _ in range(2000))
    flop = 2 * 8192 ** 3
    rec = {"impl": args.impl, "rank": rank, "world": world, "gemm_ms_alone": round(statistics.median(alone), 4),
           "gemm_ms_with_comm": round(statistics.median(withc), 4), "slowdown_median": round(med, 5),
           "ci95": [round(boots[50], 5), round(boots[1949], 5)],
           "tflops_alone": round(flop / (statistics.median(alone) * 1e-3) / 1e12, 1), "msg_mib": args.msg_mib,
           "burst_ops": burst}
    for ph, lab in (("A", "alone"), ("B", "with_comm")):
        if samp[ph]:
            rec[f"sm_mhz_{lab}"] = statistics.median(x[0] for x in samp[ph])
            rec[f"power_w_{lab}"] = round(statistics.median(x[1] for x in samp[ph]), 1)
            rec[f"samples_{lab}"] = len(samp[ph])
    if comm is not None:
        rec["iccl_stats"] = comm.stats()
        comm.destroy()
    allrec = [None] * world
    dist.all_gather_object(allrec, rec)
    if rank == 0:
        for r in allrec:
            print(json.dumps(r))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
