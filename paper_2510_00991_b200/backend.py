"""torch.distributed backend "iccl" over the B200 P2P path.

The paper's integration mode is a drop-in communication library under
Megatron: pipeline-parallel activations move with
``batch_isend_irecv`` / ``send`` / ``recv`` and MoE dispatch / combine with
``all_to_all_single``.  Registering this backend routes exactly those calls
through ``libiccl_b200.so`` unchanged::

    import paper_2510_00991_b200.backend  # registers "iccl"
    dist.init_process_group("iccl", ...)   # or backend="cuda:iccl,cpu:gloo"
    dist.batch_isend_irecv([...]); dist.all_to_all_single(out, inp, osplit, isplit)

Stream model (NCCL-like): each op is enqueued on a side stream that first
waits for the caller's current stream; ``Work.wait()`` makes the caller's
current stream wait for the op, ``Work.synchronize()`` waits on the host.
torch only hands batched P2P to a Python backend op by op (no coalescing),
so sends to peer p and receives from p get their own streams: FIFO matching
per ordered pair is preserved and no op ever waits behind an op for another
peer (no cross-pair cycles, whatever order the ranks issue them in).

Only the P2P path is implemented; reductions / gathers raise
``NotImplementedError`` (DP/TP collectives are out of scope —
pair this backend with NCCL or gloo for them, e.g. ``"cuda:iccl"`` in a
subgroup).
"""
from __future__ import annotations

from datetime import timedelta
from typing import Dict, List, Optional, Tuple

import torch
import torch.distributed as dist

from .comm import Communicator
from .config import IcclConfig

BACKEND_NAME = "iccl"


class IcclWork(dist._Work):
    """Completion handle of one op: an event on the op's side stream."""

    def __init__(self, stream: torch.cuda.Stream, tensors: List[torch.Tensor], result=None):
        super().__init__()
        self._event = torch.cuda.Event()
        self._event.record(stream)
        self._tensors = tensors  # keep buffers alive until the op completes
        self._result = result if result is not None else tensors

    def wait(self, timeout: timedelta = timedelta(0)) -> bool:
        torch.cuda.current_stream().wait_event(self._event)
        return True

    def is_completed(self) -> bool:
        return self._event.query()

    def synchronize(self) -> None:
        self._event.synchronize()

    def result(self):
        return self._result


class IcclProcessGroup(dist.ProcessGroup):
    """Python ProcessGroup whose P2P and all-to-all ops run on the ICCL path."""

    def __init__(self, store, rank: int, size: int, timeout: timedelta, config: Optional[IcclConfig] = None):
        super().__init__(rank, size)
        self._dev = torch.cuda.current_device()
        self.comm = Communicator(rank, size, self._dev, config or IcclConfig.defaults(), store=store)
        self._streams: Dict[Tuple[str, int], torch.cuda.Stream] = {}

    # -- streams --------------------------------------------------------------
    def _stream(self, kind: str, peer: int) -> torch.cuda.Stream:
        key = (kind, peer)
        s = self._streams.get(key)
        if s is None:
            s = torch.cuda.Stream(device=self._dev)
            self._streams[key] = s
        return s

    def _enter(self, kind: str, peer: int, tensors: List[torch.Tensor]) -> torch.cuda.Stream:
        s = self._stream(kind, peer)
        s.wait_stream(torch.cuda.current_stream())
        for t in tensors:
            t.record_stream(s)
        return s

    # -- P2P ----------------------------------------------------------------------
    def send(self, tensors: List[torch.Tensor], dst: int, tag: int = 0) -> IcclWork:
        s = self._enter("send", dst, tensors)
        for t in tensors:
            self.comm.isend(t, dst, stream=s)
        return IcclWork(s, tensors)

    def recv(self, tensors: List[torch.Tensor], src: int, tag: int = 0) -> IcclWork:
        s = self._enter("recv", src, tensors)
        for t in tensors:
            self.comm.irecv(t, src, stream=s)
        return IcclWork(s, tensors)

    # -- all-to-all ------------------------------------------------------------------
    def alltoall_base(self, output: torch.Tensor, input: torch.Tensor, output_split_sizes: List[int],
                      input_split_sizes: List[int], opts=None) -> IcclWork:
        s = self._enter("a2a", -1, [output, input])
        n = self.size()
        osp = list(output_split_sizes) or None
        isp = list(input_split_sizes) or None
        if input.dim() == 0 or output.dim() == 0:
            raise ValueError("all_to_all_single needs at least 1-d tensors")
        if n == 1:
            with torch.cuda.stream(s):
                output.copy_(input)
        else:
            self.comm.alltoallv(output, input, osp, isp, stream=s)
        return IcclWork(s, [output, input], [output])

    def alltoall(self, output_tensors: List[torch.Tensor], input_tensors: List[torch.Tensor], opts=None) -> IcclWork:
        """List form: rank i's input_tensors[j] lands in rank j's output_tensors[i]."""
        n = self.size()
        s = self._enter("a2a", -1, list(output_tensors) + list(input_tensors))
        self.comm.group_start()
        try:
            for k in range(n):
                to, frm = (self.rank() + k) % n, (self.rank() - k) % n
                if output_tensors[frm].numel():
                    self.comm.irecv(output_tensors[frm], frm, stream=s)
                if input_tensors[to].numel():
                    self.comm.isend(input_tensors[to], to, stream=s)
        finally:
            self.comm.group_end()
        return IcclWork(s, list(output_tensors) + list(input_tensors), list(output_tensors))

    def barrier(self, opts=None) -> IcclWork:
        """Every rank exchanges one 16-byte word with every other over the path."""
        n = self.size()
        inp = torch.zeros(max(n, 1), 16, dtype=torch.uint8, device=self._dev)
        out = torch.empty_like(inp)
        w = self.alltoall_base(out, inp, [], []) if n > 1 else IcclWork(torch.cuda.current_stream(), [inp])
        w.synchronize()
        return w

    def getBackendName(self) -> str:
        return BACKEND_NAME

    def shutdown(self) -> None:
        torch.cuda.synchronize(self._dev)
        self.comm.destroy()

    # -- out of scope ------------------------------------------------
    def _unsupported(self, *a, **k):
        raise NotImplementedError("the iccl backend implements the P2P path only (send/recv, batch_isend_irecv, "
                                  "all_to_all); use nccl or gloo for reductions and gathers")

    allreduce = allgather = broadcast = reduce = reduce_scatter = gather = scatter = _unsupported


def _create(store, rank: int, size: int, timeout: timedelta) -> IcclProcessGroup:
    return IcclProcessGroup(store, rank, size, timeout)


def register() -> None:
    """Register the "iccl" backend with torch.distributed (idempotent)."""
    if BACKEND_NAME not in dist.Backend.backend_list:
        dist.Backend.register_backend(BACKEND_NAME, _create, devices=["cuda"])


register()
