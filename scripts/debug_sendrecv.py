"""Debug: the test_pair_sendrecv_bytes sequence with progress prints (2 ranks, torchrun)."""
import faulthandler, os, sys, threading, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("gloo")
import paper_2510_00991_b200 as iccl
faulthandler.dump_traceback_later(40, exit=True)
ll = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pinned = len(sys.argv) > 2 and sys.argv[2] == "pinned"
comm = iccl.init(rank, world, rank, iccl.IcclConfig.defaults(sm_small_bytes=ll))
works = []
def watch():
    while True:
        time.sleep(5)
        st = []
        for w in works:
            try:
                s = iccl._lib.XferState()
                iccl._lib.lib.iccl_req_state(comm._h, iccl._lib.C.c_uint64(w.req), iccl._lib.C.byref(s))
                st.append((s.total_chunks, s.posted, s.done, s.active_path))
            except Exception as e:
                st.append(str(e))
        err = iccl._lib.C.c_int()
        iccl._lib.lib.iccl_comm_get_async_error(comm._h, iccl._lib.C.byref(err))
        print(f"[r{rank}] watch stats={comm.stats()} works={st} async={err.value} "
              f"last={iccl._lib.lib.iccl_get_last_error()}", flush=True)
threading.Thread(target=watch, daemon=True).start()
sizes = [8, 4097, 3 * (1 << 20) + 5, 64 << 20]
for i, n in enumerate(sizes):
    for off in (0, 3):
        src = np.random.default_rng(1000 + i).integers(0, 256, n + off, dtype=np.uint8)
        if rank == 0:
            print(f"[r0] to_dev {n}+{off}", flush=True)
            t = (torch.from_numpy(src.copy()).pin_memory().to(dev, non_blocking=True) if pinned
                 else torch.from_numpy(src.copy()).to(dev))
            print(f"[r0] send {n}+{off}", flush=True)
            works.append(comm.isend(t[off:], 1))
        else:
            r = torch.zeros(n + off, dtype=torch.uint8, device=dev)
            print(f"[r1] recv {n}+{off}", flush=True)
            works.append(comm.irecv(r[off:], 0))
            torch.cuda.synchronize()
            ok = np.array_equal(r[off:].cpu().numpy(), src[off:])
            print(f"[r1] got {n}+{off} ok={ok}", flush=True)
torch.cuda.synchronize()
print(f"[r{rank}] done", flush=True)
comm.destroy()
