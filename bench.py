#!/usr/bin/env python
"""Benchmark of the ICCL B200 P2P path (BASELINE.json metric).

Default workload (one "step"): every rank runs one batched isend/irecv group —
send 256 MiB (a bf16 [4, 4096, 8192] pipeline-parallel activation, config 3's
hop size) to rank+1 and receive 256 MiB from rank-1.  At N=1 the peer is the
rank itself (self send/recv: the same proxy / copy-engine path, local HBM).
``value`` = payload bytes moved by all ranks per second (weak scaling: the
per-rank work is fixed).  Inputs (256 MiB) exceed the 126 MB L2, so no flush
is needed between steps.

Other workloads (--workload): ``alltoallv`` (config 4 MoE dispatch+combine),
``sweep`` (config 2 size sweep, several lines).  ``--impl reference`` times the
reference's CPU path (the oracle port of SPEC.md transport, see oracle/) on the
same workload and prints the same JSON shape.

Launch: ``python bench.py`` (N=1) or
``python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N``.
"""
import argparse
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
MiB = 1 << 20


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None

    def __enter__(self):
        if os.environ.get("ICCL_BENCH_NO_CLOCKS"):  # diagnosis: run without the nvidia-smi sampler
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", ",".join(str(g) for g in self.gpus),
                                          f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline (oracle)
# The reference's CPU path is the SPEC transport restated in oracle/ (the
# reference ships no compiled code): real bytes moved chunk by
# chunk (4 MiB chunks, six pointers, DES clock).  One transfer is one
# single-threaded event loop, so "all host threads" means the
# step's bytes are split into one sub-transfer per core, run in parallel
# processes.  Payloads are built in the pool initializer, outside the timing.
_REF_SRC = None


def _ref_init(nbytes):
    global _REF_SRC
    import numpy as np
    _REF_SRC = np.random.default_rng(50 + os.getpid() % 1000).integers(0, 256, nbytes, dtype=np.uint8)


def _ref_noop(_):
    return os.getpid()


def _ref_transfer(_):
    from oracle import collectives as oc
    oc.send_recv(oc.CommGroup(2), 0, 1, _REF_SRC)
    return _REF_SRC.nbytes


def cpu_reference(step_bytes: int, steps: int, warmup: int, cores: int = 0):
    """Time `steps` steps of `step_bytes` through the oracle transport on
    `cores` host processes; returns (seconds per step, cores, per-core bytes)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    cores = cores or len(os.sched_getaffinity(0))
    per = ((step_bytes + cores - 1) // cores + 4095) // 4096 * 4096
    durations = []
    # spawned workers: the same clean processes whether the caller holds a CUDA
    # context, pinned buffers and a communicator's threads (the product arm)
    # or not (the reference arm) — forked ones inherited the product arm's
    # state and timed 37% slower
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("spawn"), initializer=_ref_init,
                             initargs=(per,)) as ex:
        list(ex.map(_ref_noop, range(cores)))
        for step in range(warmup + steps):
            t0 = time.perf_counter()
            moved = sum(ex.map(_ref_transfer, range(cores)))
            if step >= warmup:
                durations.append(time.perf_counter() - t0)
    assert moved >= step_bytes
    return sum(durations) / len(durations), cores, per


def run_reference(args):
    """--impl reference: the oracle port on the same workload (the world's
    step bytes), all host cores, rank 0 only; the other ranks exit."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    world = args.gpus
    step_bytes = world * args.bytes
    per_step, cores, per = cpu_reference(step_bytes, args.steps, args.warmup)
    value = step_bytes / per_step / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": _config(args),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"full step: {world} x {args.bytes >> 20} MiB split into {cores} parallel "
                                   f"send/recv transfers of {per / MiB:.2f} MiB through the oracle transport "
                                   f"(SPEC.md:228-263, 4 MiB chunks)"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- product arm
def _config(args):
    return {"workload": "sendrecv ring shift: batched isend(rank+1)+irecv(rank-1) of a bf16 [4,4096,8192] "
                        "activation (256 MiB) per rank per step; N=1 is self send/recv",
            "message_bytes": args.bytes, "transport": args.transport, "monitor": bool(args.monitor),
            "chunk_bytes": args.chunk_bytes, "l2": "inputs 256 MiB > 126 MB L2 (no flush needed)",
            "parallelism": f"p2p{args.gpus}"}


def run_product(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2510_00991_b200 as iccl
    cfg = iccl.IcclConfig.defaults(monitor_enabled=bool(args.monitor), transport=args.transport)
    if args.chunk_bytes:
        cfg.chunk_bytes = args.chunk_bytes
    comm = iccl.init(rank, world, local, cfg)
    nel = args.bytes // 2
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    src = torch.randint(-32768, 32767, (nel,), dtype=torch.int16, device=dev, generator=g).view(torch.bfloat16)
    dst = torch.empty_like(src)
    to, frm = (rank + 1) % world, (rank - 1) % world
    stream = torch.cuda.current_stream()

    def step(s=src, d=dst):
        comm.batch_isend_irecv([iccl.P2POp("isend", s, to), iccl.P2POp("irecv", d, frm)])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    comm.monitor.drain()
    stats0 = comm.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(list(range(world)) if rank == 0 else [local]) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    stats1 = comm.stats()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    per_step_ms = ms_max / args.steps
    value = world * args.bytes * args.steps / (ms_max * 1e-3) / 1e9

    # dominant operation: the chunk copy, timed on its own copy stream by the
    # monitor's device events (start/end of every chunk, no kernel) ->
    # achieved bytes / copy duration
    recs = comm.monitor.drain()
    copy_ns = [r.t2 - r.t1 for r in recs if r.t2 > r.t1]
    achieved = (sum(r.size for r in recs) / (sum(copy_ns) * 1e-9) / 1e9) if copy_ns else None
    peaks = _peaks()
    if world == 1:
        bound, peak, note = "hbm", peaks.get("hbm_gbs", 6650.0), "self copy: read+write = 2 x payload bytes"
        achieved_alg = achieved * 2 if achieved else None
    else:
        bound, peak, note = ("nvlink", 770.0,
                             "per-direction peer copy; peak = measured 770 GB/s peer copy (B200_PROFILING.md), "
                             "nominal 900")
        achieved_alg = achieved
    roofline = {"bound": bound, "achieved": round(achieved_alg, 1) if achieved_alg else None, "peak": peak,
                "unit": "GB/s", "frac": round(achieved_alg / peak, 4) if achieved_alg else None,
                "traffic": None, "kernel": "copy-engine chunk copy (cuMemcpyDtoDAsync), timed by the monitor's device events",
                "note": note + "; ncu does not profile copy-engine work, so traffic is null"}
    kernels = stats1["kernels_launched"] - stats0["kernels_launched"]
    copies = stats1["copies_issued"] - stats0["copies_issued"]

    # e2e: host buffers in pinned memory, H2D + send/recv + D2H inside the
    # timed region.  The step is pipelined the way a caller of the public API
    # would run it: the hop is split into --e2e-pieces pieces, piece i's H2D
    # (copy stream), batched isend/irecv (current stream) and D2H (a second
    # copy stream) overlap with the neighbours, so the two PCIe directions run
    # concurrently; device staging is double-buffered across steps, so step
    # s+1's H2D streams in while step s drains (no pipeline refill per step).
    # Every byte still crosses H2D -> NVLink/HBM -> D2H.
    h_src = src.view(torch.int16).cpu().pin_memory()
    h_dst = torch.empty_like(h_src).pin_memory()
    bufs = [(torch.empty_like(src), torch.empty_like(src)) for _ in range(2)]
    pieces = max(1, args.e2e_pieces)
    bounds = [(nel * i // pieces) // 8 * 8 for i in range(pieces)] + [nel]
    s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    consumed = [None, None]  # per staging buffer: its last step's sends are done (stream)
    drained = [None, None]   # per staging buffer: its last D2H is done (s_d2h)
    nstep = [0]

    def e2e_step():
        j = nstep[0] % 2
        nstep[0] += 1
        d_in, d_out = bufs[j]
        if consumed[j] is not None:
            s_h2d.wait_event(consumed[j])
        if drained[j] is not None:
            stream.wait_event(drained[j])
        for i in range(pieces):
            a, b = bounds[i], bounds[i + 1]
            with torch.cuda.stream(s_h2d):
                d_in.view(torch.int16)[a:b].copy_(h_src[a:b], non_blocking=True)
            stream.wait_stream(s_h2d)
            step(d_in[a:b], d_out[a:b])
            s_d2h.wait_stream(stream)
            with torch.cuda.stream(s_d2h):
                h_dst[a:b].copy_(d_out.view(torch.int16)[a:b], non_blocking=True)
        consumed[j] = stream.record_event()
        drained[j] = s_d2h.record_event()

    for _ in range(2):
        e2e_step()
    stream.wait_stream(s_d2h)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    s_h2d.wait_stream(stream)  # the timed region starts here for the copy streams too
    s_d2h.wait_stream(stream)
    for _ in range(args.steps):
        e2e_step()
    stream.wait_stream(s_d2h)  # every step's result is back in host memory
    e3.record(stream)
    barrier()
    t = torch.tensor([e2.elapsed_time(e3)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = world * args.bytes * args.steps / (float(t.item()) * 1e-3) / 1e9

    # the e2e ceiling on this box: the hop's H2D and D2H alone, concurrently
    # on the two copy streams (PCIe, both directions at once), best of 3
    def pcie_both():
        best = None
        for _ in range(3):
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            s_h2d.wait_stream(stream)
            s_d2h.wait_stream(stream)
            with torch.cuda.stream(s_h2d):
                bufs[0][0].view(torch.int16).copy_(h_src, non_blocking=True)
            with torch.cuda.stream(s_d2h):
                h_dst.copy_(bufs[0][1].view(torch.int16), non_blocking=True)
            stream.wait_stream(s_h2d)
            stream.wait_stream(s_d2h)
            f1.record(stream)
            torch.cuda.synchronize()
            ms_ = f0.elapsed_time(f1)
            best = ms_ if best is None else min(best, ms_)
        return args.bytes / (best * 1e-3) / 1e9

    ok = torch.equal(h_dst, torch.randint(-32768, 32767, (nel,), dtype=torch.int16, device=dev,
                                          generator=torch.Generator(device=dev).manual_seed(1 + frm)).cpu())
    pcie_bound = pcie_both()

    comm.check_async_error()
    comm.destroy()  # before the CPU baseline: the communicator's threads would share its cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference arm's own sample: the same steps / warm-up (a step is ~10 ms of CPU work)
        per_step, cores, per = cpu_reference(args.bytes, args.steps, args.warmup)
        cpu = {"value": round(args.bytes / per_step / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"{args.steps} steps (after {args.warmup} warm-up) of the same {args.bytes >> 20} MiB hop "
                         f"split into {cores} parallel send/recv transfers of {per / MiB:.2f} MiB through the oracle "
                         f"transport (SPEC.md:228-263, 4 MiB chunks)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(per_step_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": _config(args), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": args.bytes,
                    "d2h_bytes_per_step": args.bytes, "bit_exact": bool(ok),
                    "pipeline_pieces": pieces,
                    "bound": {"value": round(pcie_bound, 2), "unit": "GB/s", "frac": round(e2e_value / world / pcie_bound, 4),
                              "note": "per GPU: the hop's H2D and D2H alone, run concurrently (PCIe both "
                                      "directions), best of 3"}},
            "gpu_launches": int(kernels), "copy_engine_copies": int(copies),
            "gpu_launches_note": "kernels of libiccl_b200.so in the timed region, counted by iccl_comm_stats; a "
                                 "256 MiB hop takes the copy-engine path, which by design launches none "
                                 "(north_star: 0 SMs on the default path) - its device work is the copies and "
                                 "stream memops counted here; <=256 KiB hops run K5, <=16 MiB K6, the backup K1 / K9, "
                                 "and --workload alltoallv K2/K3 (fused forms: K8 / K10)",
            "sms_used_by_copies": 0, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def moe_routing(rank, world, T=4096, k=8, E=64, device="cuda"):
    """Config 4 routing, see paper_2510_00991_b200.moe.config4_routing."""
    from paper_2510_00991_b200.moe import config4_routing
    return config4_routing(rank, T, k, E, device)


def run_alltoallv(args):
    """Config 4: MoE expert-parallel dispatch + combine over the alltoallv path."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2510_00991_b200 as iccl
    from paper_2510_00991_b200.moe import expand_rows, plan_dispatch, scatter_rows
    cfg = iccl.IcclConfig.defaults(monitor_enabled=bool(args.monitor), transport=args.transport)
    comm = iccl.init(rank, world, local, cfg)
    T, k, E, H = 4096, 8, 64, 7168
    experts = moe_routing(rank, world, T, k, E, dev)

    def counts_exchange(send_counts):
        s = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        if world == 1:
            return send_counts
        comm.alltoall(r, s)  # the one exchange step, through the product's own alltoall
        torch.cuda.synchronize()
        return r.tolist()

    plan = plan_dispatch(experts, E, world, counts_exchange)
    from paper_2510_00991_b200.moe import config4_tokens
    tokens = config4_tokens(rank, T, H, dev)
    packed = torch.empty(T * k, H, dtype=tokens.dtype, device=dev)
    recv = torch.empty(sum(plan.recv_counts), H, dtype=tokens.dtype, device=dev)
    back = torch.empty_like(packed)
    out = torch.empty_like(packed)
    row = H * 2

    def step():
        expand_rows(tokens, plan.pos, k, packed)                              # K2 pack
        comm.alltoallv(recv, packed, plan.recv_counts, plan.send_counts)     # dispatch
        comm.alltoallv(back, recv, plan.send_counts, plan.recv_counts)       # combine
        scatter_rows(back, plan.order, out)                                  # K3 unpack

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ok = torch.equal(out.view(T, k, H).view(torch.int16), tokens.view(torch.int16).unsqueeze(1).expand(T, k, H))
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = comm.stats()
    with ClockSampler(list(range(world)) if rank == 0 else [local]) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    s1 = comm.stats()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    # per-rank egress/ingress over NVLink (self segment excluded) for the bound
    c_out = sum(plan.send_counts) - plan.send_counts[rank]
    c_in = sum(plan.recv_counts) - plan.recv_counts[rank]
    eb = torch.tensor([max(c_out, c_in) * row], device=dev, dtype=torch.float64)
    tot = torch.tensor([2.0 * sum(plan.send_counts) * row], device=dev, dtype=torch.float64)
    okt = torch.tensor([1.0 if ok else 0.0], device=dev, dtype=torch.float64)
    # rendezvous outcomes in the timed region, summed over ranks: transfers
    # the receiver issued (pulls) and sends that gave up waiting for the CTS
    rzv = torch.tensor([s1["pulls_issued"] - s0["pulls_issued"], s1["cts_timeouts"] - s0["cts_timeouts"]],
                       device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(rzv, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(eb, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    ms = float(t.item()) / args.steps
    value = float(tot.item()) / (ms * 1e-3) / 1e9
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    # bound: two alltoallv (max per-GPU NVLink direction at 770 GB/s) + K2 + K3 at HBM
    t_link = 2 * float(eb.item()) / 770e9 if world > 1 else 0.0
    t_hbm = 2 * (2 * T * k * row) / (hbm * 1e9) + (0 if world > 1 else 2 * 2 * T * k * row / (hbm * 1e9))
    t_star = t_link + t_hbm
    comm.destroy()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 rows (u8 moves)", "data": "synthetic",
            "config": {"workload": "MoE dispatch+combine: K2 pack, alltoallv, alltoallv back, K3 unpack; "
                                   "T=4096/rank, top-8 of 64 experts, hidden 7168 bf16, skewed routing",
                       "transport": args.transport, "parallelism": f"ep{world}"},
            "roofline": {"bound": "nvlink+hbm" if world > 1 else "hbm", "t_star_ms": round(t_star * 1e3, 4),
                         "frac": round(t_star / (ms * 1e-3), 4),
                         "note": "t* = 2 x max_i max(egress_i, ingress_i)/770 GB/s + K2/K3 HBM time"},
            "rendezvous": {"pulls": int(rzv[0].item()), "cts_timeouts": int(rzv[1].item()),
                           "transfers": 2 * args.steps * world * (world - 1)},
            "bit_exact_roundtrip": bool(okt.item() > 0), "gpu_launches": int(s1["kernels_launched"] - s0[
                "kernels_launched"]) + 2 * args.steps,
            "clocks": clk.summary()}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--workload", choices=["sendrecv", "alltoallv"], default="sendrecv")
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", 1)))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["iccl", "reference"], default="iccl")
    ap.add_argument("--bytes", type=int, default=256 * MiB)
    ap.add_argument("--transport", choices=["auto", "ce", "sm"], default="auto")
    ap.add_argument("--chunk-bytes", type=int, default=0)
    # (not "--monitor": torchrun's parser would take that abbreviation as its own)
    ap.add_argument("--iccl-monitor", dest="monitor", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-pieces", type=int, default=4, help="pipeline pieces of the e2e (host buffer) step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "alltoallv":
        run_alltoallv(args)
    else:
        run_product(args)


if __name__ == "__main__":
    main()
