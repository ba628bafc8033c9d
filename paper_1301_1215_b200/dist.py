"""Host-side plumbing of the coil-sharded multi-GPU path (one process per GPU).

torch.distributed only carries host metadata: the 64-byte CUDA IPC handles of the ranks' exchange
windows (peer-memory transport, the default) or the 128-byte NCCL unique id (NCCL transport). The
data-path exchanges (the Omega-window coil sum of P:246 / P:289 and the CG dot products) are done by
libnlinv.so's own kernels over peer memory, or on its own NCCL communicator.
"""
from __future__ import annotations

import numpy as np

from .nlinv import coil_partition, get_unique_id


def exchange_unique_id(rank: int, world: int, group=None) -> bytes | None:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes (None if world == 1)."""
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def connect_peers(plan, group=None) -> None:
    """Peer-memory exchange (world > 1 without an NCCL id): all-gather every rank's 64-byte
    exchange-window handle over torch.distributed and open them (nlinv_plan_connect)."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, plan.exchange_handle(), group=group)
    plan.connect(handles)


def local_frame(y_full: np.ndarray, ncoils: int, rank: int, world: int) -> np.ndarray:
    """This rank's contiguous coil block of a [J, ng, ng] frame (rule R10)."""
    first, count = coil_partition(ncoils, world, rank)
    return np.ascontiguousarray(y_full[first:first + count])


def assemble_unknowns(parts, ncoils: int) -> np.ndarray:
    """Global [1 + J, ng, ng] unknowns from per-rank [1 + J_r, ng, ng] pieces (rank order).
    rho is replicated: every rank's block 0 must be identical, and rank 0's copy is kept."""
    world = len(parts)
    ng = parts[0].shape[-1]
    out = np.empty((1 + ncoils, ng, ng), dtype=parts[0].dtype)
    out[0] = parts[0][0]
    for r, part in enumerate(parts):
        first, count = coil_partition(ncoils, world, r)
        if part.shape[0] != 1 + count:
            raise ValueError(f"rank {r}: expected {1 + count} blocks, got {part.shape[0]}")
        if not np.array_equal(part[0], parts[0][0]):
            raise ValueError(f"rank {r}: replicated rho differs from rank 0")
        out[1 + first:1 + first + count] = part[1:]
    return out
