#!/usr/bin/env python
"""Config 5: primary-backup failover under the MoE alltoallv with the window
monitor on.

Workload: config 4's expert-parallel dispatch + combine (T=4096 tokens/rank,
top-8 of 64 experts, hidden 7168 bf16, skewed routing) — K2 pack, alltoallv,
reverse alltoallv, K3 unpack — on every rank.

Phases (each K timed steps, CUDA events, max over ranks):
  off    monitor off, no fault script                       -> t_off
  armed  monitor on (W=8), a fault script installed that never fires
                                                            -> t_armed, overhead = t_armed / t_off - 1 (target <= 3%)
  fault  the primary (copy-engine) path of directed pair src->dst goes Down
         at chunk `--fault-chunk` of its first dispatch send and stays Down:
         the watchdog + probe must switch to the backup (SM kernel K1) and
         resume at the receiver's breakpoint; every rank's combine output
         must equal its tokens bit for bit (the alltoallv round trip is the
         identity)                                          -> detect_us, resume chunk, anomaly_us, backup GB/s
  restore the path comes Up; monitor_failed_link's probe moves the pair back
         to the primary                                     -> switch-back observed, bit-exact

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 benchmarks/failover.py
"""
import argparse
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunk-mib", type=int, default=8)
    ap.add_argument("--delta-us", type=int, default=1000)
    ap.add_argument("--src", type=int, default=-1)
    ap.add_argument("--dst", type=int, default=-1)
    ap.add_argument("--fault-chunk", type=int, default=3)
    ap.add_argument("--backup", choices=["sm", "relay"], default="sm")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2510_00991_b200 as iccl
    from bench import moe_routing
    from paper_2510_00991_b200.moe import expand_rows, plan_dispatch, scatter_rows

    src_r = args.src if args.src >= 0 else (3 if world > 5 else world - 1)
    dst_r = args.dst if args.dst >= 0 else (5 if world > 5 else (src_r + 2) % world if world > 2 else 1 - src_r)
    cfg = iccl.IcclConfig.defaults(chunk_bytes=args.chunk_mib << 20, delta_us=args.delta_us, probe_period_us=200,
                                   monitor_enabled=False, window=4, backup_kind=args.backup)
    comm = iccl.init(rank, world, local, cfg)
    T, k, E, H = 4096, 8, 64, 7168
    experts = moe_routing(rank, world, T, k, E, dev)

    def counts_exchange(send_counts):
        s = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        comm.alltoall(r, s)
        torch.cuda.synchronize()
        return r.tolist()

    plan = plan_dispatch(experts, E, world, counts_exchange)
    g = torch.Generator(device=dev).manual_seed(2000 + rank)
    tokens = torch.randint(-32768, 32767, (T, H), dtype=torch.int16, device=dev, generator=g).view(torch.bfloat16)
    packed = torch.empty(T * k, H, dtype=tokens.dtype, device=dev)
    recv = torch.empty(sum(plan.recv_counts), H, dtype=tokens.dtype, device=dev)
    back = torch.empty_like(packed)
    out = torch.empty_like(packed)
    expect = tokens.view(torch.int16).unsqueeze(1).expand(T, k, H)
    stream = torch.cuda.current_stream()

    def step():
        expand_rows(tokens, plan.pos, k, packed)
        comm.alltoallv(recv, packed, plan.recv_counts, plan.send_counts)
        comm.alltoallv(back, recv, plan.send_counts, plan.recv_counts)
        scatter_rows(back, plan.order, out)

    def all_ok():
        ok = torch.equal(out.view(T, k, H).view(torch.int16), expect)
        t = torch.tensor([1.0 if ok else 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item() > 0)

    def timed(n):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / n], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    res = {"bench": "failover", "n_gpus": world, "pair": f"{src_r}->{dst_r}", "backup": args.backup,
           "chunk_bytes": args.chunk_mib << 20, "delta_us": args.delta_us,
           "workload": "MoE dispatch+combine (T=4096/rank, top-8 of 64 experts, hidden 7168 bf16, skewed)"}
    for _ in range(args.warmup):
        step()
    # off / armed, ABAB-interleaved (3 rounds) to cancel drift
    never = iccl.FaultScript().down(src_r, dst_r, chunk=1 << 30, op_index=1 << 20)
    t_off, t_mon, t_armed = [], [], []
    for _ in range(3):
        comm.monitor.enable(False)
        comm.set_faults(iccl.FaultScript())
        t_off.append(timed(args.steps))
        comm.monitor.enable(True, 8)
        t_mon.append(timed(args.steps))
        comm.set_faults(never)
        t_armed.append(timed(args.steps))
    pre_recs = comm.monitor.drain()  # monitor-phase records: the pre-fault baseline of the window series
    res["t_off_ms"] = round(statistics.median(t_off), 4)
    res["t_monitor_ms"] = round(statistics.median(t_mon), 4)
    res["t_armed_ms"] = round(statistics.median(t_armed), 4)
    res["monitor_overhead"] = round(statistics.median(t_mon) / statistics.median(t_off) - 1, 4)
    res["monitor_failover_overhead"] = round(statistics.median(t_armed) / statistics.median(t_off) - 1, 4)
    res["bit_exact_armed"] = all_ok()

    # fault: Down at chunk `fault_chunk` of src's next dispatch send to dst
    comm.set_faults(iccl.FaultScript().down(src_r, dst_r, chunk=args.fault_chunk, op_index=0))
    dist.barrier()
    t_fault = timed(1)
    res["t_fault_step_ms"] = round(t_fault, 4)
    res["bit_exact_fault"] = all_ok()
    t_backup = timed(args.steps)  # the pair stays on the backup path
    res["t_on_backup_ms"] = round(t_backup, 4)
    res["bit_exact_on_backup"] = all_ok()
    time.sleep(0.01)
    recs = comm.monitor.drain()
    ev = comm.switch_events()
    info = torch.zeros(8, device=dev, dtype=torch.float64)
    if rank in (src_r, dst_r):
        # either endpoint may have issued the faulted transfer (a push by the
        # sender, a pull by the receiver): its watchdog is the one that switched
        other = dst_r if rank == src_r else src_r
        sw = [e for e in ev if e["peer"] == other and e["to"] == "backup"]
        if sw:
            e0 = sw[0]
            t_inj = e0["t_ns"] - e0["detect_ns"]
            info[0] = 1
            info[1] = e0["detect_ns"] / 1e3
            info[2] = e0["resume_chunk"]
            info[3] = 1 if e0["to"] == "backup" and e0["trigger"] == "watchdog" else 0
            # anomaly: first W=8 window sample on the faulted pair after the
            # injection whose throughput is below half the pre-fault median
            pair = [r for r in pre_recs + recs if r.peer == other]
            samples = iccl.sample_series(pair, 8)
            pre = [s.value for s in samples if s.time < t_inj]
            med = statistics.median(pre) if pre else None
            post = [s for s in samples if s.time >= t_inj]
            if med and post:
                bad = [s for s in post if s.value < 0.5 * med]
                if bad:
                    info[4] = (bad[0].time - t_inj) / 1e3
                    info[5] = min(s.value for s in bad) / med
            prim_recs = [r for r in pre_recs + recs if r.path == 0 and r.t2 > r.t1 and r.peer != rank]
            back_recs = [r for r in recs if r.path == 1 and r.t2 > r.t1 and r.peer == other]
            if prim_recs and back_recs:
                bp = sum(r.size for r in prim_recs) / (sum(r.t2 - r.t1 for r in prim_recs) * 1e-9) / 1e9
                bb = sum(r.size for r in back_recs) / (sum(r.t2 - r.t1 for r in back_recs) * 1e-9) / 1e9
                info[6], info[7] = bp, bb
    dist.all_reduce(info, op=dist.ReduceOp.SUM)
    res["switched"] = bool(info[0].item() > 0)
    res["switch_by_watchdog_to_backup"] = bool(info[3].item() > 0)
    res["detect_us"] = round(float(info[1].item()), 1)
    res["resume_chunk"] = int(info[2].item())
    res["anomaly_detect_us"] = round(float(info[4].item()), 1) if info[4].item() > 0 else None
    res["anomaly_depth"] = round(float(info[5].item()), 4) if info[4].item() > 0 else None
    res["primary_chunk_GBps"] = round(float(info[6].item()), 1)
    res["backup_chunk_GBps"] = round(float(info[7].item()), 1)
    res["backup_frac_of_primary"] = round(float(info[7].item() / info[6].item()), 4) if info[6].item() else None

    # restore: Up -> monitor_failed_link probes the primary and switches back
    comm.set_faults(iccl.FaultScript().up(src_r, dst_r, t_us=0))
    time.sleep(0.05)
    timed(2)
    ev = comm.switch_events()
    back_ok = torch.tensor([1.0 if (rank != src_r or comm.active_path(dst_r) == "primary") else 0.0], device=dev)
    sb = torch.tensor([1.0 if any(e["to"] == "primary" for e in ev) else 0.0], device=dev)
    dist.all_reduce(sb, op=dist.ReduceOp.MAX)
    res["switch_back_event"] = bool(sb.item() > 0)
    dist.all_reduce(back_ok, op=dist.ReduceOp.MIN)
    res["switched_back_to_primary"] = bool(back_ok.item() > 0)
    res["t_restored_ms"] = round(timed(args.steps), 4)
    res["bit_exact_restored"] = all_ok()
    comm.check_async_error()
    comm.destroy()
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
