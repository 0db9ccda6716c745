#!/usr/bin/env python
"""Standalone timing of the SM kernels (K1 copy, K2 gather, K3 scatter) at the
BASELINE shapes, each against its roofline, plus a bit-exact check.

The product path parks its side streams on stream memory operations, which
ncu's serialised replay cannot profile through; this script launches the
same kernels through the same C ABI (``iccl_copy_sm`` / ``iccl_gather_rows``
/ ``iccl_scatter_rows``) with no memops, so it is the ncu target:

    ncu --set full --clock-control none -k regex:iccl_ -c 6 python benchmarks/kernels.py --reps 1

Shapes:
* K1 local: 256 MiB (bf16 [4,4096,8192] PP activation) HBM->HBM, 2 x bytes of
  HBM traffic; sm_cap 16 (the backup default) and 148 (one CTA per SM).
* K1 peer (2 GPUs): 256 MiB cuda:0 -> cuda:1 over NVLink, bound = 770 GB/s
  measured peer-copy peak.
* K2 / K3: MoE pack / unpack, 32768 rows x 14336 B (T=4096, top-8, hidden
  7168 bf16) = 448 MiB each way, 2 x bytes of HBM traffic (+8 B index/row).
"""
import argparse
import ctypes as C
import json
import os

# one hardware queue per stream: a stream parked on a stream-memory wait must not
# stall the library's other streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MiB = 1 << 20


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def timed(fn, reps, stream):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3  # s per launch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="", help="comma list of k1_local,k1_peer,k1_pull,k2,k3,k8")
    ap.add_argument("--quick", action="store_true", help="small shapes (compute-sanitizer runs)")
    args = ap.parse_args()
    from paper_2510_00991_b200 import gather_rows, scatter_rows
    from paper_2510_00991_b200._lib import lib
    hbm = peaks().get("hbm_gbs", 6546.6)
    only = set(args.only.split(",")) if args.only else None
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    sh = C.c_void_p(int(s.cuda_stream))
    out = []
    n = (16 if args.quick else 256) * MiB
    g = torch.Generator(device="cuda").manual_seed(1)
    src = torch.randint(-128, 127, (n,), dtype=torch.int8, device="cuda", generator=g)

    def k1(dst, ctas):
        rc = lib.iccl_copy_sm(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), n, ctas, sh)
        assert rc == 0, rc

    if not only or "k1_local" in only:
        dst = torch.empty_like(src)
        for ctas in (16, 148):
            t = timed(lambda: k1(dst, ctas), args.reps, s)
            ok = torch.equal(dst, src)
            ach = 2 * n / t / 1e9
            out.append({"kernel": "K1 iccl_copy_tma local", "bytes": n, "ctas": ctas, "us": round(t * 1e6, 2),
                        "payload_GBps": round(n / t / 1e9, 1), "achieved_GBps": round(ach, 1), "peak": hbm,
                        "bound": "hbm (r+w = 2 x bytes)", "frac": round(ach / hbm, 4), "bit_exact": ok})
        del dst
    if (not only or "k1_peer" in only) and torch.cuda.device_count() > 1:
        dst = torch.empty(n, dtype=torch.int8, device="cuda:1")
        _ = src[:16].to("cuda:1")  # torch enables peer access 0 -> 1
        torch.cuda.synchronize()
        for ctas in (8, 16, 32, 148):
            t = timed(lambda: k1(dst, ctas), args.reps, s)
            ok = torch.equal(dst.cpu(), src.cpu())
            ach = n / t / 1e9
            out.append({"kernel": "K1 iccl_copy_tma peer 0->1", "bytes": n, "ctas": ctas, "us": round(t * 1e6, 2),
                        "achieved_GBps": round(ach, 1), "peak": 770.0, "bound": "nvlink (measured peer copy)",
                        "frac": round(ach / 770.0, 4), "nominal_frac": round(ach / 900.0, 4), "bit_exact": ok})
        del dst
    if (not only or "k1_pull" in only) and torch.cuda.device_count() > 1:
        # pull: cuda:0 reads cuda:1's memory (the SM backup of a receiver-issued transfer)
        rsrc = src.to("cuda:1")
        dst = torch.empty_like(src)
        torch.cuda.synchronize()
        for name, fn, ctas_list in (("K1 iccl_copy_tma pull 1->0", lib.iccl_copy_sm, (16, 148)),):
            for ctas in ctas_list:
                def run(fn=fn, ctas=ctas):
                    assert fn(C.c_void_p(rsrc.data_ptr()), C.c_void_p(dst.data_ptr()), n, ctas, sh) == 0
                t = timed(run, max(1, args.reps // 4), s)
                ok = torch.equal(dst, src)
                ach = n / t / 1e9
                out.append({"kernel": name, "bytes": n, "ctas": ctas, "us": round(t * 1e6, 2),
                            "achieved_GBps": round(ach, 1), "peak": 770.0, "bound": "nvlink (measured peer copy)",
                            "frac": round(ach / 770.0, 4), "bit_exact": ok})
        del dst, rsrc
    T, k, H = (256 if args.quick else 4096), 8, 7168
    row = H * 2
    rows = T * k
    if not only or "k2" in only or "k3" in only:
        tok = torch.randint(-32768, 32767, (T, H), dtype=torch.int16, device="cuda", generator=g)
        idx = torch.randint(0, T, (rows,), dtype=torch.int64, device="cuda", generator=g)
        packed = torch.empty(rows, H, dtype=torch.int16, device="cuda")
        if not only or "k2" in only:
            t = timed(lambda: gather_rows(tok, idx, packed), args.reps, s)
            ok = torch.equal(packed, tok[idx])
            alg = 2 * rows * row + rows * 8
            out.append({"alg_bytes": "T*k rows read (L2 may serve repeats) + T*k written + 8 B/row index",
                        "kernel": "K2 iccl_gather_rows", "rows": rows, "row_bytes": row, "us": round(t * 1e6, 2),
                        "achieved_GBps": round(alg / t / 1e9, 1), "peak": hbm, "bound": "hbm",
                        "frac": round(alg / t / 1e9 / hbm, 4), "bit_exact": ok})
        if not only or "k2" in only:
            # expand form (what moe_dispatch runs): each token read once, written k times
            from paper_2510_00991_b200 import expand_rows
            order = torch.randperm(rows, device="cuda", generator=g)
            pos = torch.empty_like(order)
            pos[order] = torch.arange(rows, device="cuda")
            t = timed(lambda: expand_rows(tok, pos, k, packed), args.reps, s)
            ok = torch.equal(packed, tok[torch.div(order, k, rounding_mode="floor")])
            alg = T * row + rows * row + rows * 8
            out.append({"kernel": "K2 iccl_expand_rows", "rows": rows, "row_bytes": row, "us": round(t * 1e6, 2),
                        "achieved_GBps": round(alg / t / 1e9, 1), "peak": hbm, "bound": "hbm",
                        "alg_bytes": "T rows read + T*k rows written + 8 B/row index",
                        "frac": round(alg / t / 1e9 / hbm, 4), "bit_exact": ok})
        if not only or "k3" in only:
            perm = torch.randperm(rows, device="cuda", generator=g)
            back = torch.empty_like(packed)
            t = timed(lambda: scatter_rows(packed, perm, back), args.reps, s)
            exp = torch.empty_like(packed)
            exp[perm] = packed
            ok = torch.equal(back, exp)
            alg = 2 * rows * row + rows * 8
            out.append({"kernel": "K3 iccl_scatter_rows", "rows": rows, "row_bytes": row, "us": round(t * 1e6, 2),
                        "achieved_GBps": round(alg / t / 1e9, 1), "peak": hbm, "bound": "hbm",
                        "frac": round(alg / t / 1e9 / hbm, 4), "bit_exact": ok})
    if not only or "k8" in only:
        # K8 (fused dispatch) on one rank: every routed row stays local, so
        # the kernel is K2's expand plus K8's handshake words (no peer flags)
        import paper_2510_00991_b200 as iccl
        from paper_2510_00991_b200.moe import DispatchPlan, moe_dispatch_fused
        tok = torch.randint(-32768, 32767, (T, H), dtype=torch.int16, device="cuda", generator=g)
        order = torch.randperm(rows, device="cuda", generator=g)
        pos = torch.empty_like(order)
        pos[order] = torch.arange(rows, device="cuda")
        comm = iccl.Communicator(0, 1, 0, iccl.IcclConfig.defaults())
        plan = DispatchPlan(order, torch.div(order, k, rounding_mode="floor"), pos, [rows], [rows])
        recv = torch.empty(rows, H, dtype=torch.int16, device="cuda")
        t = timed(lambda: moe_dispatch_fused(comm, tok, plan, recv), args.reps, s)
        ok = torch.equal(recv, tok[torch.div(order, k, rounding_mode="floor")])
        comm.destroy()
        alg = T * row + rows * row + rows * 8
        out.append({"kernel": "K8 iccl_dispatch_push (1 rank: all rows local)", "rows": rows, "row_bytes": row,
                    "us": round(t * 1e6, 2), "achieved_GBps": round(alg / t / 1e9, 1), "peak": hbm, "bound": "hbm",
                    "alg_bytes": "T rows read + T*k rows written + 8 B/row index",
                    "frac": round(alg / t / 1e9 / hbm, 4), "bit_exact": ok})
    for r in out:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
