"""Row-sharded (data-parallel) plumbing around librqlp.

A is split by rows over the ranks of a torch.distributed group; every exchange step of the
method (Gram of each CholeskyQR pass, the power-step A^T V, the projection B = V^T A) is a
row-sum done inside librqlp with ncclAllReduce on the compute stream.  This module only does the
host-side plumbing: the row partition, the NCCL unique-id bootstrap over torch.distributed (any
backend, gloo included) and the max-over-ranks reduction bench.py uses for timing.
"""
from __future__ import annotations

import ctypes

import torch

UID_BYTES = 128


def row_block(m_global: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous row block [r0, r1) of rank `rank` (the first m % world ranks get one
    extra row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m_global, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def exchange_unique_id(group=None, make_id=None) -> bytes:
    """Rank 0 of `group` creates the 128-byte ncclUniqueId (librqlp's rqlp_get_unique_id) and
    broadcasts it; every rank returns the same bytes.  Works with gloo (CPU tensors) and nccl."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if make_id is None:
        from . import _capi

        def make_id():
            buf = ctypes.create_string_buffer(UID_BYTES)
            rc = _capi.load().rqlp_get_unique_id(buf)
            if rc != 0:
                raise RuntimeError(f"rqlp_get_unique_id rc={rc}")
            return buf.raw
    if rank == 0:
        raw = make_id()
        t = torch.frombuffer(bytearray(raw), dtype=torch.uint8).clone()
    else:
        t = torch.zeros(UID_BYTES, dtype=torch.uint8)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().tolist())


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a host scalar over the group (bench.py: the slowest rank's time)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    dev = device if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
