"""Helpers for the GPU parity tests: seeded payloads and a multi-process
launcher (one process per rank, as in production).  Ranks map to GPUs
round-robin (rank % device_count), so every multi-rank test also runs on a
one-GPU box: CUDA IPC, the copy engines, stream memops and the SM kernels
all work between processes that share a device (a "peer" copy is then a
local HBM copy)."""
import os
import socket
import traceback

import numpy as np


def payload(nbytes: int, seed: int) -> np.ndarray:
    """Uniform random bytes (viewed as fp32 they include NaN/Inf/denormal
    patterns: parity is raw-byte)."""
    return np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8)


def to_dev(a: np.ndarray, device):
    import torch
    return torch.from_numpy(a.copy()).to(device)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, outdir, kwargs):
    import faulthandler
    import sys
    import torch
    import torch.distributed as dist
    # a hung rank leaves its Python stacks behind for the parent's error report
    log = open(os.path.join(outdir, f"rank{rank}.log"), "w")
    sys.stdout = sys.stderr = log
    faulthandler.dump_traceback_later(kwargs.pop("_hang_s", 100), exit=True, file=log)
    try:
        dev = rank % torch.cuda.device_count()  # ranks share GPUs when there are fewer GPUs than ranks
        torch.cuda.set_device(dev)
        store = dist.TCPStore("127.0.0.1", port, world, rank == 0, wait_for_workers=True)
        from paper_2510_00991_b200 import Communicator, IcclConfig
        cfg = IcclConfig.defaults(**kwargs.pop("config", {}))
        comm = Communicator(rank, world, dev, cfg, store=store)
        comm._test_store = store  # scenarios may barrier through it
        res = fn(comm, rank, world, **kwargs)
        torch.cuda.synchronize()
        comm.destroy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **(res or {}))
    except Exception:
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as fh:
            fh.write(traceback.format_exc())
        raise


def run_ranks(world: int, fn, tmpdir, timeout: float = 120.0, **kwargs):
    """Run fn(comm, rank, world, **kwargs) -> dict of numpy arrays on `world`
    GPUs, one process each; returns the per-rank dicts.  A rendezvous port
    taken between free_port() and the bind is retried once."""
    try:
        return _run_ranks(world, fn, tmpdir, timeout, **kwargs)
    except AssertionError as e:
        if "EADDRINUSE" not in str(e):
            raise
        for f in os.listdir(str(tmpdir)):
            if f.startswith("rank"):
                os.remove(os.path.join(str(tmpdir), f))
        return _run_ranks(world, fn, tmpdir, timeout, **kwargs)


def _run_ranks(world: int, fn, tmpdir, timeout: float = 120.0, **kwargs):
    import torch.multiprocessing as mp
    port = free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, str(tmpdir), dict(kwargs))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
    errs = []
    for r, p in enumerate(procs):
        if p.is_alive():
            p.kill()
            errs.append(f"rank {r} timed out")
        ef = os.path.join(str(tmpdir), f"rank{r}.err")
        if os.path.exists(ef):
            errs.append(open(ef).read())
        if p.exitcode not in (0, None) and not os.path.exists(ef):
            lf = os.path.join(str(tmpdir), f"rank{r}.log")
            errs.append(f"rank {r} exit code {p.exitcode}:\n" + (open(lf).read()[-6000:] if os.path.exists(lf) else ""))
    if errs:
        raise AssertionError("\n".join(errs))
    return [dict(np.load(os.path.join(str(tmpdir), f"rank{r}.npz"))) for r in range(world)]


def dev_of(rank: int):
    """The GPU rank `rank` runs on (round-robin over the visible GPUs)."""
    import torch
    return torch.device("cuda", rank % torch.cuda.device_count())


def fault_delta_us(world: int) -> int:
    """Watchdog delta for the failover tests.  On separate GPUs 300 us.  When
    ranks share a GPU, their processes' kernels and copies are time-sliced:
    a rank spinning in a kernel (K7, an LL receive, a device sleep) holds the
    GPU for whole time slices, so an innocent chunk (and its CTS probe) can
    wait milliseconds — delta must exceed that or innocent stalls switch."""
    import torch
    return 300 if torch.cuda.device_count() >= world else 20_000
