"""MoE expert-parallel dispatch / combine over the alltoallv path (config 4).

dispatch: route every (token, expert) pair to the rank owning the expert —
K2 packs the routed rows by destination rank (``iccl_gather_rows``), the
alltoallv moves them, received rows arrive grouped by source rank.
combine: the reverse alltoallv with the same counts, then K3 scatters the
rows back to (token, k) order (``iccl_scatter_rows``).  The routing metadata
(a 32 K-entry argsort) is computed with torch; the bytes move only through
libiccl_b200.so kernels and copy engines.  PAPER.md:157, 864-868.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import torch

from ._lib import lib
from .errors import InvalidArgument, raise_for


def _sh(stream: Optional[torch.cuda.Stream]) -> C.c_void_p:
    s = stream or torch.cuda.current_stream()
    return C.c_void_p(int(s.cuda_stream))


def gather_rows(src: torch.Tensor, idx: torch.Tensor, out: Optional[torch.Tensor] = None, ctas: int = 0,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """out[i] = src[idx[i]] (K2)."""
    if idx.dtype != torch.int64 or not idx.is_cuda:
        raise InvalidArgument("idx must be a CUDA int64 tensor")
    n = idx.numel()
    if out is None:
        out = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row = src[0].numel() * src.element_size() if src.shape[0] else out[0].numel() * out.element_size()
    raise_for(lib.iccl_gather_rows(C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(idx.data_ptr()),
                                   n, row, int(ctas), _sh(stream)), "iccl_gather_rows")
    return out


def expand_rows(src: torch.Tensor, pos: torch.Tensor, k: int, out: torch.Tensor, ctas: int = 0,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """out[pos[t*k + j]] = src[t] for j < k (K2, expand form: every source row
    read once and written k times — the dispatch pack without the gather's
    k-fold re-reads)."""
    if pos.dtype != torch.int64 or not pos.is_cuda or pos.numel() != src.shape[0] * k:
        raise InvalidArgument("pos must be a CUDA int64 tensor of src rows x k entries")
    row = out[0].numel() * out.element_size() if out.shape[0] else 16
    raise_for(lib.iccl_expand_rows(C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(pos.data_ptr()),
                                   src.shape[0], int(k), row, int(ctas), _sh(stream)), "iccl_expand_rows")
    return out


def scatter_rows(src: torch.Tensor, idx: torch.Tensor, out: torch.Tensor, ctas: int = 0,
                 stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """out[idx[i]] = src[i] (K3)."""
    if idx.dtype != torch.int64 or not idx.is_cuda:
        raise InvalidArgument("idx must be a CUDA int64 tensor")
    n = idx.numel()
    row = out[0].numel() * out.element_size()
    raise_for(lib.iccl_scatter_rows(C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(idx.data_ptr()),
                                    n, row, int(ctas), _sh(stream)), "iccl_scatter_rows")
    return out


def config4_routing(rank: int, T: int = 4096, k: int = 8, E: int = 64, device="cuda") -> torch.Tensor:
    """BASELINE config 4's routing: expert popularity
    p_e ~ (e+1)^-0.8, permuted by seed 0; top-k experts per token by
    multinomial sampling with seed 1000 + rank.  Returns [T, k] int64."""
    g = torch.Generator().manual_seed(0)
    p = torch.arange(1, E + 1, dtype=torch.float64) ** -0.8
    p = p[torch.randperm(E, generator=g)]
    g = torch.Generator().manual_seed(1000 + rank)
    return torch.multinomial(p.expand(T, E), k, replacement=False, generator=g).to(device)


def config4_tokens(rank: int, T: int = 4096, H: int = 7168, device="cuda") -> torch.Tensor:
    """Config 4's token payload: uniform random int16 bits (seed 2000 + rank)
    viewed as bf16 [T, H], so every bit pattern (NaN, Inf, denormals) occurs."""
    g = torch.Generator(device=device).manual_seed(2000 + rank)
    return torch.randint(-32768, 32767, (T, H), dtype=torch.int16, device=device, generator=g).view(torch.bfloat16)


@dataclass
class DispatchPlan:
    order: torch.Tensor          # [T*k] int64: flattened (token, k) index of each packed row
    token_of_row: torch.Tensor   # [T*k] int64: token index of each packed row
    pos: torch.Tensor            # [T*k] int64: packed row of each flattened (token, k) pair (inverse of order)
    send_counts: List[int]       # rows to each rank
    recv_counts: List[int]       # rows from each rank


def plan_dispatch(expert_ids: torch.Tensor, n_experts: int, world: int, counts_exchange) -> DispatchPlan:
    """expert_ids: [T, k] int64 on the GPU.  Experts are laid out contiguously
    per rank (n_experts / world each).  ``counts_exchange(send_counts) ->
    recv_counts`` is the one exchange step of the alltoallv."""
    T, k = expert_ids.shape
    per_rank = n_experts // world
    flat = expert_ids.reshape(-1)
    dest = torch.div(flat, per_rank, rounding_mode="floor")
    # stable sort by (destination rank, expert) keeps token order inside a segment
    key = flat
    order = torch.sort(key, stable=True).indices
    counts = torch.bincount(dest, minlength=world).tolist()
    recv = counts_exchange(counts)
    pos = torch.empty_like(order)
    pos[order] = torch.arange(order.numel(), device=order.device)
    return DispatchPlan(order, torch.div(order, k, rounding_mode="floor"), pos, counts, recv)


def moe_dispatch(comm, tokens: torch.Tensor, plan: DispatchPlan, packed: Optional[torch.Tensor] = None,
                 recv: Optional[torch.Tensor] = None, stream=None):
    """tokens [T, H] -> rows received from every rank, grouped by source."""
    if packed is None:
        packed = torch.empty((plan.order.numel(),) + tuple(tokens.shape[1:]), dtype=tokens.dtype, device=tokens.device)
    expand_rows(tokens, plan.pos, plan.order.numel() // tokens.shape[0], packed, stream=stream)
    if recv is None:
        recv = torch.empty((sum(plan.recv_counts),) + tuple(tokens.shape[1:]), dtype=tokens.dtype,
                           device=tokens.device)
    comm.alltoallv(recv, packed, plan.recv_counts, plan.send_counts, stream=stream)
    return packed, recv


def moe_dispatch_fused(comm, tokens: torch.Tensor, plan: DispatchPlan, recv: Optional[torch.Tensor] = None,
                       stream=None) -> torch.Tensor:
    """The same result as :func:`moe_dispatch` (rows received from every
    rank, grouped by source) in one kernel, K8 (``iccl_dispatch_rows``): each
    token row is read once and each of its k routed copies is stored straight
    into the receive buffer of the rank that owns it — over NVLink, with no
    packed staging buffer.  Pairs armed for failover take
    the unfused form inside the library, with the same result."""
    if not tokens.is_cuda or not tokens.is_contiguous():
        raise InvalidArgument("tokens must be a contiguous CUDA tensor")
    T = tokens.shape[0]
    k = plan.pos.numel() // T if T else 1
    row = tokens[0].numel() * tokens.element_size() if T else 16
    if recv is None:
        recv = torch.empty((sum(plan.recv_counts),) + tuple(tokens.shape[1:]), dtype=tokens.dtype,
                           device=tokens.device)
    n = len(plan.send_counts)
    Arr = C.c_size_t * n
    sc = Arr(*[int(x) for x in plan.send_counts])
    rc = Arr(*[int(x) for x in plan.recv_counts])
    raise_for(lib.iccl_dispatch_rows(comm._h, C.c_void_p(tokens.data_ptr()), T, int(k),
                                     C.c_void_p(plan.pos.data_ptr()), sc, C.c_void_p(recv.data_ptr()), rc, int(row),
                                     _sh(stream)), "iccl_dispatch_rows")
    return recv


def moe_combine(comm, expert_out: torch.Tensor, plan: DispatchPlan, T: int, k: int,
                back: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None, stream=None):
    """Reverse alltoallv with the same counts, then K3 puts every row back at
    its (token, k) slot: out [T, k, H]."""
    if back is None:
        back = torch.empty((sum(plan.send_counts),) + tuple(expert_out.shape[1:]), dtype=expert_out.dtype,
                           device=expert_out.device)
    comm.alltoallv(back, expert_out, plan.send_counts, plan.recv_counts, stream=stream)
    if out is None:
        out = torch.empty((T * k,) + tuple(expert_out.shape[1:]), dtype=expert_out.dtype, device=expert_out.device)
    scatter_rows(back, plan.order, out, stream=stream)
    return out.view(T, k, *expert_out.shape[1:])


def moe_combine_fused(comm, expert_out: torch.Tensor, plan: DispatchPlan, T: int, k: int,
                      out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """The same result as :func:`moe_combine` in one kernel on the receiving
    side, K10 (``iccl_combine_rows``): every row this rank routed out comes
    back straight from the expert rank's tensor (NVLink loads) into its
    (token, k) slot of ``out`` [T, k, ...] — no packed staging buffer.  Pairs
    armed for failover take the unfused form inside the library."""
    if not expert_out.is_cuda or not expert_out.is_contiguous():
        raise InvalidArgument("expert_out must be a contiguous CUDA tensor")
    shape = tuple(expert_out.shape[1:])
    if out is None:
        out = torch.empty((T * k,) + shape, dtype=expert_out.dtype, device=expert_out.device)
    row = out[0].numel() * out.element_size() if out.shape[0] else 16
    n = len(plan.send_counts)
    Arr = C.c_size_t * n
    sc = Arr(*[int(x) for x in plan.recv_counts])   # rows this rank returns to each rank
    rc = Arr(*[int(x) for x in plan.send_counts])   # rows it gets back (the packed layout `order` indexes)
    src = expert_out.data_ptr() if expert_out.numel() else out.data_ptr()
    raise_for(lib.iccl_combine_rows(comm._h, C.c_void_p(src), sc, C.c_void_p(out.data_ptr()),
                                    C.c_void_p(plan.order.data_ptr()), rc, int(row), _sh(stream)),
              "iccl_combine_rows")
    return out.view(T, k, *shape)
