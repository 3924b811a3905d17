"""Host-side plumbing of the multi-GPU migration path (one process per GPU).

Each GPU is one Symphony node (reference: one NodeManager per node,
/root/reference/proj/src/simcore.cpp:31-33); sessions shard across nodes and
the only exchange is point-to-point per-session migration
(simcore.cpp:132-141), so there is no collective on the data path. What the
ranks do exchange, once, over torch.distributed is control metadata: CUDA IPC
handles of every rank's page pool, so a migration kernel on the source GPU
can store straight into the receiver's pages over NVLink. Timing is reduced
as the max over ranks.

Backend-agnostic (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np


def ring_peer(rank: int, world: int) -> int:
    """Receiver of `rank`'s session in the ring migration (config 3)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return (rank + 1) % world


def ring_source(rank: int, world: int) -> int:
    """Whose session `rank` receives."""
    return (rank - 1) % world


def session_seed(rank: int) -> int:
    return 100 + rank


def session_layout(rank: int, pool_pages: int, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Deterministic page placement of a rank's pool: its own session's pages
    (src ids) and the region it receives a peer's session into (dst ids).
    Any rank can recompute any other rank's layout from the rank id alone,
    which is how a sender addresses the receiver's pages."""
    if 2 * n > pool_pages:
        raise ValueError("pool must hold two sessions")
    perm = np.random.default_rng(session_seed(rank)).permutation(pool_pages).astype(np.uint32)
    return perm[:n], perm[n:2 * n]


@dataclass
class PeerPool:
    rank: int
    handle: bytes
    num_pages: int
    page_bytes: int


def exchange_pool_handles(dist, rank: int, handle: bytes, num_pages: int, page_bytes: int) -> List[PeerPool]:
    """all_gather of every rank's (IPC handle, pool geometry)."""
    world = dist.get_world_size()
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, bytes(handle), int(num_pages), int(page_bytes)))
    pools = [PeerPool(*g) for g in gathered]
    for i, p in enumerate(pools):
        if p.rank != i:
            raise RuntimeError(f"rank {i} reported as {p.rank}")
        if p.page_bytes != page_bytes:
            raise RuntimeError("page size differs across ranks")
    return pools


def max_over_ranks(dist, value: float, device=None) -> float:
    """Max of a per-rank float (device time) across the job."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
