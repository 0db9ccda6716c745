"""The "iccl" torch.distributed backend: registration on
CPU; on >= 2 GPUs, torch's own P2P / all-to-all calls routed through the
ICCL path and checked byte for byte against the oracle's delivered bytes."""
import os
import traceback

import numpy as np
import pytest

from gpu_helpers import free_port, payload


def test_backend_registers():
    import torch.distributed as dist
    from paper_2510_00991_b200 import backend
    backend.register()
    backend.register()  # idempotent
    assert "iccl" in dist.Backend.backend_list
    assert dist.Backend.ICCL == "iccl"
    assert issubclass(backend.IcclProcessGroup, dist.ProcessGroup)


def _rank_main(rank, world, port, outdir):
    try:
        import torch
        import torch.distributed as dist
        import paper_2510_00991_b200.backend  # noqa: F401
        torch.cuda.set_device(rank % torch.cuda.device_count())
        dist.init_process_group("iccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        dev = torch.device("cuda", rank % torch.cuda.device_count())
        res = {}
        # batched P2P in a ring, ops issued in an order that would deadlock if
        # the backend serialised them on one stream
        n = 3 * (1 << 20) + 5
        src = torch.from_numpy(payload(n, seed=300 + rank)).to(dev)
        dst = torch.zeros(n, dtype=torch.uint8, device=dev)
        ops = [dist.P2POp(dist.isend, src, (rank + 1) % world), dist.P2POp(dist.irecv, dst, (rank - 1) % world)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        torch.cuda.synchronize()
        res["ring"] = dst.cpu().numpy()
        # blocking send / recv, both orders
        small = torch.from_numpy(payload(4099, seed=400 + rank)).to(dev)
        got = torch.zeros(4099, dtype=torch.uint8, device=dev)
        if rank == 0:
            dist.send(small, 1)
            dist.recv(got, 1)
        elif rank == 1:
            dist.recv(got, 0)
            dist.send(small, 0)
        torch.cuda.synchronize()
        res["pingpong"] = got.cpu().numpy()
        # all_to_all_single with uneven splits (MoE dispatch shape, row = 14336 B)
        rng = np.random.default_rng(9)
        splits = [[int(x) for x in rng.integers(0, 40, world)] for _ in range(world)]
        row = 7168
        inp = torch.from_numpy(payload(sum(splits[rank]) * row * 2, seed=500 + rank)).to(dev).view(
            torch.bfloat16).view(-1, row)
        out = torch.empty(sum(splits[i][rank] for i in range(world)), row, dtype=torch.bfloat16, device=dev)
        dist.all_to_all_single(out, inp, [splits[i][rank] for i in range(world)], splits[rank])
        torch.cuda.synchronize()
        res["a2a"] = out.view(torch.uint8).cpu().numpy().reshape(-1)
        res["splits"] = np.array(splits)
        dist.barrier()
        dist.destroy_process_group()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    except Exception:
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as fh:
            fh.write(traceback.format_exc())
        raise


@pytest.mark.gpu
def test_backend_p2p_and_alltoall(tmp_path):
    import torch
    import torch.multiprocessing as mp
    from oracle import collectives as oc
    world = max(2, torch.cuda.device_count())
    port = free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = [open(tmp_path / f"rank{r}.err").read() for r in range(world) if (tmp_path / f"rank{r}.err").exists()]
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    n = 3 * (1 << 20) + 5
    for r in range(world):
        assert np.array_equal(res[r]["ring"], payload(n, seed=300 + (r - 1) % world))
    assert np.array_equal(res[0]["pingpong"], payload(4099, seed=401))
    assert np.array_equal(res[1]["pingpong"], payload(4099, seed=400))
    splits = res[0]["splits"].tolist()
    row = 7168 * 2
    send = [payload(sum(splits[i]) * row, seed=500 + i) for i in range(world)]
    exp = oc.expected_alltoallv(send, splits, row)
    for r in range(world):
        assert np.array_equal(res[r]["a2a"], exp[r])
