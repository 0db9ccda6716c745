#!/usr/bin/env python
"""Config 4's dispatch and combine, three ways each:

  fused    K8 (iccl_dispatch_rows): each token row read once, its k routed
           copies stored straight into the owners' receive buffers over
           NVLink — no packed staging buffer
  unfused  K2 (expand form) into a packed buffer, then the copy-engine
           alltoallv (0 SMs for the transfer)
  nccl     torch gather of the routed rows + NCCL all_to_all_single

and the combine (identity experts: the received rows go straight back):

  fused    K10 (iccl_combine_rows): each token rank loads its rows from the
           expert ranks' tensors over NVLink into their (token, k) slots
  unfused  the reverse copy-engine alltoallv into a packed buffer, then K3
  nccl     NCCL all_to_all_single, then torch index_copy_

T = 4096 tokens per rank, top-8 of 64 experts, hidden 7168 bf16, skewed
routing (§8d).  One step = one dispatch; device time per step (CUDA events),
max over ranks.  Every arm's received rows are compared with the unfused
arm's, bit for bit.  Bound: t* = max over ranks of max(egress, ingress) /
770 GB/s (NVLink per direction, measured peer-copy peak).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        benchmarks/moe_dispatch.py
"""
import argparse
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--arms", default="fused,unfused,nccl")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2510_00991_b200 as iccl
    from paper_2510_00991_b200.moe import (config4_routing, config4_tokens, expand_rows, moe_combine_fused,
                                           moe_dispatch_fused, plan_dispatch, scatter_rows)
    T, k, E, H = args.tokens, 8, 64, 7168
    row = 2 * H
    comm = iccl.init(rank, world, local, iccl.IcclConfig.defaults())

    def exchange(send_counts):
        s = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        dist.all_to_all_single(r, s)
        return r.tolist()

    experts = config4_routing(rank, T, k, E, dev)
    plan = plan_dispatch(experts, E, world, exchange)
    tokens = config4_tokens(rank, T, H, dev)
    packed = torch.empty(T * k, H, dtype=tokens.dtype, device=dev)
    nrecv = sum(plan.recv_counts)
    bufs = {a: torch.zeros(nrecv, H, dtype=tokens.dtype, device=dev) for a in ("fused", "unfused", "nccl")}

    back = torch.empty(T * k, H, dtype=tokens.dtype, device=dev)
    outs = {a: torch.zeros(T * k, H, dtype=tokens.dtype, device=dev) for a in ("fused", "unfused", "nccl")}

    def combine(arm):
        if arm == "fused":
            moe_combine_fused(comm, bufs["fused"], plan, T, k, outs["fused"])
        elif arm == "unfused":
            comm.alltoallv(back, bufs["unfused"], plan.send_counts, plan.recv_counts)
            scatter_rows(back, plan.order, outs["unfused"])
        else:
            dist.all_to_all_single(back, bufs["nccl"], plan.send_counts, plan.recv_counts)
            outs["nccl"].index_copy_(0, plan.order, back)

    def step(arm):
        if arm == "fused":
            moe_dispatch_fused(comm, tokens, plan, bufs["fused"])
        elif arm == "unfused":
            expand_rows(tokens, plan.pos, k, packed)
            comm.alltoallv(bufs["unfused"], packed, plan.recv_counts, plan.send_counts)
        else:
            torch.index_select(tokens, 0, plan.token_of_row, out=packed)
            dist.all_to_all_single(bufs["nccl"], packed, plan.recv_counts, plan.send_counts)

    arms = args.arms.split(",")
    res = {"bench": "moe_dispatch", "n_gpus": world, "tokens_per_rank": T, "top_k": k, "experts": E, "hidden": H}
    eg = (sum(plan.send_counts) - plan.send_counts[rank]) * row
    ig = (sum(plan.recv_counts) - plan.recv_counts[rank]) * row
    lim = torch.tensor([max(eg, ig)], device=dev, dtype=torch.float64)
    dist.all_reduce(lim, op=dist.ReduceOp.MAX)
    t_star = float(lim.item()) / 770e9
    res["t_star_ms"] = round(t_star * 1e3, 4)
    res["max_rank_egress_or_ingress_MiB"] = round(float(lim.item()) / 2**20, 1)
    for arm in ["unfused"] + [a for a in arms if a != "unfused"]:
        for _ in range(args.warmup):
            step(arm)
        torch.cuda.synchronize()
        s0 = comm.stats()
        dist.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            step(arm)
        e1.record(st)
        torch.cuda.synchronize()
        s1 = comm.stats()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
        ok = torch.tensor([1.0 if torch.equal(bufs[arm].view(torch.int16), bufs["unfused"].view(torch.int16))
                           else 0.0], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        ms = float(t.item())
        res[arm] = {"ms_per_dispatch": round(ms, 4), "frac_of_bound": round(t_star / (ms * 1e-3), 4),
                    "bit_exact_vs_unfused": bool(ok.item() > 0)}
        if arm != "nccl":
            res[arm]["kernels_per_step"] = (s1["kernels_launched"] - s0["kernels_launched"]) / args.steps
            res[arm]["ctas_per_step"] = (s1["ctas_launched"] - s0["ctas_launched"]) / args.steps
        # the combine alone, then dispatch + combine (one MoE step without the experts)
        for name, fn in (("combine", lambda: combine(arm)), ("dispatch_combine", lambda: (step(arm), combine(arm)))):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(st)
            for _ in range(args.steps):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[arm][f"ms_per_{name}"] = round(float(t.item()), 4)
        ok = torch.equal(outs[arm].view(T, k, H).view(torch.int16),
                         tokens.view(torch.int16).unsqueeze(1).expand(T, k, H))
        okt = torch.tensor([1.0 if ok else 0.0], device=dev, dtype=torch.float64)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        res[arm]["roundtrip_bit_exact"] = bool(okt.item() > 0)
    if rank == 0:
        print(json.dumps(res), flush=True)
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
