"""Diagnostic: 2-rank ring exchange (bench.py's step) with monitor records per
chunk (issuer side, push / pull), to see whether the two directions overlap."""
import os, sys, json
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
import paper_2510_00991_b200 as iccl
mon = int(os.environ.get("DIAG_MON", "1"))
comm = iccl.init(rank, world, rank, iccl.IcclConfig.defaults(monitor_enabled=bool(mon)))
n = 128 << 20
src = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device=dev)
dst = torch.empty_like(src)
to, frm = (rank + 1) % world, (rank - 1) % world
def step():
    comm.batch_isend_irecv([iccl.P2POp("isend", src, to), iccl.P2POp("irecv", dst, frm)])
for _ in range(3):
    step()
torch.cuda.synchronize(); dist.barrier()
comm.monitor.drain()
s = torch.cuda.current_stream()
times = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); step(); e1.record(s)
    torch.cuda.synchronize()
    times.append(round(e0.elapsed_time(e1) * 1e3, 1))
recs = comm.monitor.drain()
t0 = min(r.t1 for r in recs) if recs else 0
out = {"rank": rank, "step_us": times, "stats": comm.stats(),
       "recs": [(r.peer, r.chunk, r.path, r.op_seq, round((r.t1 - t0) / 1e3, 1), round((r.t2 - t0) / 1e3, 1)) for r in recs]}
print(json.dumps(out), flush=True)
comm.destroy()
dist.barrier()
