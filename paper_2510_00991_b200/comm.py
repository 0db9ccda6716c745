"""Communicator: the Python surface of the ICCL B200 P2P path.

Mirrors the reference's API surface: ``init`` builds the
CommGroup; ``send`` / ``recv`` are send_message /
send_recv; ``alltoall`` is SPEC.md:427-435;
``isend`` / ``irecv`` / ``batch_isend_irecv`` / ``alltoallv`` follow
torch.distributed's shapes; ``switch_qp`` is SPEC.md:255-263;
``set_faults`` installs a FaultScript; ``monitor`` is the
window monitor.

Tensors are the buffer type.  Every call is stream-ordered on the caller's
current CUDA stream (or ``stream=``): the data move starts when the stream
reaches the op and the stream does not run past the op until the bytes have
landed, exactly like NCCL ops.  All data movement is done by
``libiccl_b200.so``; nothing here touches tensor contents.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from ._lib import Fault as _CFault, SwitchEvent, UniqueId, XferState, lib
from .config import IcclConfig
from .errors import GroupTooSmall, InvalidArgument, ZeroLengthMessage, raise_for
from .faults import FaultScript
from .monitor import Monitor, detect_lagging_rank

PATHS = {"primary": 0, "backup": 1, 0: 0, 1: 1, "ToPrimary": 0, "ToBackup": 1}


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_tensor(t: torch.Tensor, what: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgument(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise InvalidArgument(f"{what} must be contiguous")


class Work:
    """Handle of an isend / irecv, like torch.distributed's Work."""

    def __init__(self, comm: "Communicator", req: int, stream: torch.cuda.Stream, tensor: torch.Tensor):
        self.comm = comm
        self.req = req
        self.stream = stream
        self.tensor = tensor  # keep the buffer alive until completion

    def is_completed(self) -> bool:
        done = C.c_int()
        raise_for(lib.iccl_req_test(self.comm._h, C.c_uint64(self.req), C.byref(done)), "iccl_req_test")
        return bool(done.value)

    def wait(self, timeout_s: Optional[float] = None) -> bool:
        """Make the current stream wait for the op (device-side), like NCCL
        Work.wait.  With ``timeout_s`` the host also waits for completion and
        raises IcclTimeout past the deadline (iccl_req_wait)."""
        cur = torch.cuda.current_stream()
        if cur != self.stream:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            cur.wait_event(ev)
        if timeout_s is not None:
            self.synchronize(timeout_s)
        return True

    def state(self) -> dict:
        """TransferState: the six progress pointers of this
        op, its chunk count, active path and switch count (iccl_req_state)."""
        st = XferState()
        raise_for(lib.iccl_req_state(self.comm._h, C.c_uint64(self.req), C.byref(st)), "iccl_req_state")
        return {f: getattr(st, f) for f, _ in XferState._fields_}

    def synchronize(self, timeout_s: float = 60.0) -> None:
        """Host-side wait for completion (iccl_req_wait)."""
        raise_for(lib.iccl_req_wait(self.comm._h, C.c_uint64(self.req), int(timeout_s * 1e6)), "iccl_req_wait")


@dataclass
class P2POp:
    """torch.distributed.P2POp shape: op is 'isend'/'irecv' (or the Communicator
    methods themselves)."""

    op: object
    tensor: torch.Tensor
    peer: int


def _exchange_uid(rank: int, world: int, store) -> UniqueId:
    uid = UniqueId()
    if world == 1:
        raise_for(lib.iccl_get_unique_id(C.byref(uid)), "iccl_get_unique_id")
        return uid
    key = "iccl_b200_uid"
    if rank == 0:
        raise_for(lib.iccl_get_unique_id(C.byref(uid)), "iccl_get_unique_id")
        store.set(key, bytes(uid.internal))
    else:
        raw = store.get(key)
        C.memmove(C.addressof(uid), raw, min(len(raw), C.sizeof(uid)))
    return uid


def _default_store(rank: int, world: int):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.distributed_c10d._get_default_store()
    addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
    port = int(os.environ.get("MASTER_PORT", "29512")) + 17
    return dist.TCPStore(addr, port, world, rank == 0, wait_for_workers=False)


class Communicator:
    """One rank of an ICCL communicator over the GPUs of one B200 box."""

    def __init__(self, rank: int, world_size: int, device: Optional[int] = None,
                 config: Optional[IcclConfig] = None, store=None, uid: Optional[UniqueId] = None):
        if device is None:
            device = torch.cuda.current_device()
        self.rank, self.world_size, self.device = int(rank), int(world_size), int(device)
        self.config = (config or IcclConfig.defaults()).validate()
        torch.cuda.set_device(self.device)
        if uid is None:
            uid = _exchange_uid(self.rank, self.world_size, store or (
                None if world_size == 1 else _default_store(rank, world_size)))
        h = C.c_void_p()
        cfg = self.config.to_c()
        raise_for(lib.iccl_comm_init_rank(C.byref(h), self.world_size, uid, self.rank, self.device, C.byref(cfg)),
                  "iccl_comm_init_rank")
        self._h = h
        self._group = 0
        self._keep: List[torch.Tensor] = []
        self.monitor = Monitor(self, self.config.monitor_window)

    # -- lifecycle -----------------------------------------------------------
    def destroy(self) -> None:
        if self._h:
            raise_for(lib.iccl_comm_destroy(self._h), "iccl_comm_destroy")
            self._h = None

    def abort(self) -> None:
        if self._h:
            lib.iccl_comm_abort(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    def check_async_error(self) -> None:
        err = C.c_int()
        lib.iccl_comm_get_async_error(self._h, C.byref(err))
        raise_for(err.value, "async")

    # -- memory registration (MemoryRegion) -----------------------
    def register(self, tensor: torch.Tensor) -> int:
        """Register ``tensor``'s allocation for zero-copy transfers (User Buffer
        Registration): exported over CUDA IPC once and cached.
        Unexportable memory raises UnregisteredRegion.  Returns
        the registration handle (the allocation's buffer id)."""
        _check_tensor(tensor, "registered tensor")
        h = C.c_uint64()
        raise_for(lib.iccl_register(self._h, C.c_void_p(tensor.data_ptr()), tensor.numel() * tensor.element_size(),
                                    C.byref(h)), "iccl_register")
        return h.value

    def deregister(self, handle: int) -> None:
        """Drop a registration; peers that mapped the allocation close their
        mappings.  No op in flight may still use the buffer."""
        raise_for(lib.iccl_deregister(self._h, C.c_uint64(int(handle))), "iccl_deregister")

    # -- point to point (send_message / send_recv) ---------------------------------
    def isend(self, tensor: torch.Tensor, peer: int, stream: Optional[torch.cuda.Stream] = None) -> Work:
        _check_tensor(tensor, "send tensor")
        if tensor.numel() == 0:
            raise ZeroLengthMessage("send of an empty tensor (SPEC.md:236)")
        req = C.c_uint64()
        s = stream or torch.cuda.current_stream()
        raise_for(lib.iccl_send(self._h, C.c_void_p(tensor.data_ptr()), tensor.numel() * tensor.element_size(),
                                int(peer), C.c_void_p(int(s.cuda_stream)), C.byref(req)), "iccl_send")
        return Work(self, req.value, s, tensor)

    def irecv(self, tensor: torch.Tensor, peer: int, stream: Optional[torch.cuda.Stream] = None) -> Work:
        _check_tensor(tensor, "recv tensor")
        if tensor.numel() == 0:
            raise ZeroLengthMessage("recv into an empty tensor (SPEC.md:236)")
        req = C.c_uint64()
        s = stream or torch.cuda.current_stream()
        raise_for(lib.iccl_recv(self._h, C.c_void_p(tensor.data_ptr()), tensor.numel() * tensor.element_size(),
                                int(peer), C.c_void_p(int(s.cuda_stream)), C.byref(req)), "iccl_recv")
        return Work(self, req.value, s, tensor)

    def send(self, tensor: torch.Tensor, peer: int, stream: Optional[torch.cuda.Stream] = None) -> None:
        self.isend(tensor, peer, stream)

    def recv(self, tensor: torch.Tensor, peer: int, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        self.irecv(tensor, peer, stream)
        return tensor

    send_message = send  # SPEC.md:228 name

    def group_start(self) -> None:
        raise_for(lib.iccl_group_start(self._h), "iccl_group_start")

    def group_end(self) -> None:
        raise_for(lib.iccl_group_end(self._h), "iccl_group_end")

    def batch_isend_irecv(self, ops: Sequence[P2POp], stream: Optional[torch.cuda.Stream] = None) -> List[Work]:
        """All ops of the list form one group (torch.distributed.batch_isend_irecv)."""
        works = []
        self.group_start()
        try:
            for op in ops:
                kind = op.op if isinstance(op.op, str) else getattr(op.op, "__name__", "")
                if kind in ("isend", "send"):
                    works.append(self.isend(op.tensor, op.peer, stream))
                elif kind in ("irecv", "recv"):
                    works.append(self.irecv(op.tensor, op.peer, stream))
                else:
                    raise InvalidArgument(f"unknown P2P op {op.op!r}")
        finally:
            self.group_end()
        return works

    # -- all-to-all --------------------------------------------------------------
    def alltoallv(self, output: torch.Tensor, input: torch.Tensor, output_split_sizes: Optional[Sequence[int]] = None,
                  input_split_sizes: Optional[Sequence[int]] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """torch ``all_to_all_single`` semantics: splits along dim 0 in rows;
        rank i's input rows for j land in rank j's output at rank i's offset.
        Zero-count pairs are skipped."""
        _check_tensor(input, "input")
        _check_tensor(output, "output")
        n = self.world_size
        if input.dim() == 0 or output.dim() == 0:
            raise InvalidArgument("alltoallv needs at least 1-d tensors")
        row = input[0].numel() * input.element_size() if input.shape[0] else (
            output[0].numel() * output.element_size() if output.shape[0] else 1)
        if input_split_sizes is None:
            if input.shape[0] % n:
                raise InvalidArgument("input rows not divisible by world size")
            input_split_sizes = [input.shape[0] // n] * n
        if output_split_sizes is None:
            if output.shape[0] % n:
                raise InvalidArgument("output rows not divisible by world size")
            output_split_sizes = [output.shape[0] // n] * n
        if len(input_split_sizes) != n or len(output_split_sizes) != n:
            raise InvalidArgument("split lists must have world_size entries")
        if sum(input_split_sizes) > input.shape[0] or sum(output_split_sizes) > output.shape[0]:
            raise InvalidArgument("splits exceed the tensor")
        Arr = C.c_size_t * n
        sc = Arr(*[int(x) for x in input_split_sizes])
        rc = Arr(*[int(x) for x in output_split_sizes])
        sd, rd, a, b = Arr(), Arr(), 0, 0
        for i in range(n):
            sd[i], rd[i] = a, b
            a += sc[i]
            b += rc[i]
        s = stream or torch.cuda.current_stream()
        raise_for(lib.iccl_alltoallv(self._h, C.c_void_p(input.data_ptr()), sc, sd, C.c_void_p(output.data_ptr()),
                                     rc, rd, int(row), C.c_void_p(int(s.cuda_stream))), "iccl_alltoallv")
        return output

    def alltoall(self, output: torch.Tensor, input: torch.Tensor,
                 stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Uniform alltoall: GroupTooSmall below 2 ranks."""
        if self.world_size < 2:
            raise GroupTooSmall(f"alltoall needs >= 2 ranks, have {self.world_size}")
        if input.numel() == 0:
            return output  # nbytes_per_pair = 0 completes immediately
        return self.alltoallv(output, input, None, None, stream)

    # -- primary / backup paths -------------------------------------------------------
    def switch_qp(self, peer: int, direction) -> None:
        """Receiver-driven switch of the path to ``peer``:
        'ToBackup' / 'ToPrimary' (or 'backup' / 'primary')."""
        raise_for(lib.iccl_path_switch(self._h, int(peer), PATHS[direction]), "iccl_path_switch")

    switch_path = switch_qp

    def active_path(self, peer: int) -> str:
        p = C.c_int()
        raise_for(lib.iccl_path_active(self._h, int(peer), C.byref(p)), "iccl_path_active")
        return "primary" if p.value == 0 else "backup"

    def set_chunk_bytes(self, chunk_bytes: int) -> None:
        """Chunk size of the transfers this rank issues from now on (the
        SPEC's chunk_size; config.chunk_bytes at init)."""
        raise_for(lib.iccl_comm_set_chunk_bytes(self._h, int(chunk_bytes)), "iccl_comm_set_chunk_bytes")
        self.config.chunk_bytes = int(chunk_bytes)

    def set_faults(self, script: FaultScript) -> None:
        script.validate(self.world_size)
        arr = (_CFault * max(1, len(script.entries)))()
        for i, e in enumerate(script.entries):
            arr[i].src, arr[i].dst, arr[i].path, arr[i].up = e.src, e.dst, e.path, int(e.up)
            arr[i].trigger_kind, arr[i].op_index, arr[i].chunk, arr[i].t_us = e.trigger_kind, e.op_index, e.chunk, e.t_us
        raise_for(lib.iccl_fault_set(self._h, arr, len(script.entries)), "iccl_fault_set")

    def switch_events(self) -> List[dict]:
        buf = (SwitchEvent * 1024)()
        n = C.c_int()
        raise_for(lib.iccl_switch_events(self._h, buf, 1024, C.byref(n)), "iccl_switch_events")
        return [dict(t_ns=buf[i].t_ns, peer=buf[i].peer, to="primary" if buf[i].to_path == 0 else "backup",
                     resume_chunk=buf[i].resume_chunk, trigger=("api", "watchdog", "probe")[buf[i].trigger],
                     detect_ns=buf[i].detect_ns) for i in range(n.value)]

    # -- observability -----------------------------------------------------------
    def stats(self) -> dict:
        """Work this rank issued: SM kernels launched (K1, K5, K6) and their
        CTAs, copy-engine copies and payload bytes; transfers issued as the
        receiver (pulls), sends whose wait for the receiver timed out, and
        issued transfers not yet retired by the proxy / watchdog."""
        from ._lib import Stats
        s = Stats()
        raise_for(lib.iccl_comm_stats(self._h, C.byref(s)), "iccl_comm_stats")
        return dict(kernels_launched=s.kernels_launched, ctas_launched=s.ctas_launched, copies_issued=s.copies_issued,
                    bytes_issued=s.bytes_issued, pulls_issued=s.pulls_issued, cts_timeouts=s.cts_timeouts,
                    pending_xfers=s.pending_xfers)

    def op_counts(self) -> dict:
        arr = (C.c_uint64 * self.world_size)()
        raise_for(lib.iccl_comm_op_counts(self._h, arr, self.world_size), "iccl_comm_op_counts")
        return {r: int(arr[r]) for r in range(self.world_size)}

    def detect_lagging_rank(self, threshold: int = 1) -> Optional[int]:
        return detect_lagging_rank(self.op_counts(), threshold)


def init(rank: Optional[int] = None, world_size: Optional[int] = None, device: Optional[int] = None,
         config: Optional[IcclConfig] = None, store=None) -> Communicator:
    """Build the communicator (CommGroup).  Defaults come from
    torch.distributed when it is initialised, else RANK / WORLD_SIZE /
    LOCAL_RANK from the environment (torchrun)."""
    import torch.distributed as dist
    if rank is None:
        rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else int(os.environ.get("RANK", 0))
    if world_size is None:
        world_size = (dist.get_world_size() if dist.is_available() and dist.is_initialized()
                      else int(os.environ.get("WORLD_SIZE", 1)))
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    return Communicator(rank, world_size, device, config, store)
