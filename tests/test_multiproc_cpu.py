"""World-size-2 host-side checks on CPU with the gloo backend: the unique-id
bootstrap through the TCPStore, and the alltoallv semantics the product
mirrors (torch all_to_all_single) against the oracle's delivered bytes, with
the MoE routing counts exchanged like the product's counts-exchange step."""
import os
import socket

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # 1. unique-id exchange (the product's bootstrap, comm._exchange_uid)
    from paper_2510_00991_b200.comm import _exchange_uid
    uid = _exchange_uid(rank, world, dist.distributed_c10d._get_default_store())
    raw = torch.tensor(list(bytes(uid.internal)), dtype=torch.uint8)
    allraw = [torch.zeros_like(raw) for _ in range(world)]
    dist.all_gather(allraw, raw)
    same = all(torch.equal(allraw[0], r) for r in allraw)
    # 2. MoE routing (config 4 recipe) + counts exchange + torch alltoallv
    T, k, E, H = 64, 8, 16, 32
    g = torch.Generator().manual_seed(0)
    p = torch.arange(1, E + 1, dtype=torch.float64) ** -0.8
    p = p[torch.randperm(E, generator=g)]
    g = torch.Generator().manual_seed(1000 + rank)
    experts = torch.multinomial(p.expand(T, E), k, replacement=False, generator=g)
    dest = (experts // (E // world)).reshape(-1)
    order = torch.sort(experts.reshape(-1), stable=True).indices
    send_counts = torch.bincount(dest, minlength=world)
    recv_counts = torch.zeros_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    g = torch.Generator().manual_seed(2000 + rank)
    tokens = torch.randint(0, 256, (T, H), dtype=torch.uint8, generator=g)
    packed = tokens[order // k]
    out = torch.zeros(int(recv_counts.sum()), H, dtype=torch.uint8)
    dist.all_to_all_single(out, packed, recv_counts.tolist(), send_counts.tolist())
    np.savez(os.path.join(outdir, f"r{rank}.npz"), same=same, packed=packed.numpy(), out=out.numpy(),
             send=send_counts.numpy())
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_alltoallv_semantics(tmp_path):
    import torch.multiprocessing as mp
    port = _port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn", join=True)
    res = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(2)]
    assert all(bool(r["same"]) for r in res)
    from oracle import collectives as oc
    splits = [[int(x) for x in r["send"]] for r in res]
    send = [r["packed"].reshape(-1) for r in res]
    exp = oc.expected_alltoallv(send, splits, 32)
    got_oracle = oc.alltoallv(oc.CommGroup(2, chunk_size=256), send, splits, oc.counts_T(splits), 32)
    for r in range(2):
        assert np.array_equal(res[r]["out"].reshape(-1), exp[r])
        assert np.array_equal(got_oracle[r], exp[r])
