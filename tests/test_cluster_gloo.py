"""Multi-rank host logic of the migration path, world size 2 over gloo (CPU).

Covers what bench.py --gpus N does around the kernels: ring partner
assignment, the IPC-handle exchange (all_gather_object), the page placement
each sender recomputes for its receiver, and max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2412_16434_b200 import cluster


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        handle = bytes([rank + 1]) * 64
        pools = cluster.exchange_pool_handles(dist, rank, handle, 1000 + rank, 65536)
        peer = cluster.ring_peer(rank, world)
        src = cluster.ring_source(rank, world)
        # the sender's view of the receiver's dst region == the receiver's own
        _, recv_dst = cluster.session_layout(peer, 64, 20)
        mine_src, mine_dst = cluster.session_layout(rank, 64, 20)
        t = cluster.max_over_ranks(dist, 10.0 * (rank + 1))
        results[rank] = dict(handles=[p.handle[0] for p in pools], pages=[p.num_pages for p in pools], peer=peer,
                             src=src, recv_dst=recv_dst.tolist(), mine_dst=mine_dst.tolist(),
                             overlap=len(set(mine_src.tolist()) & set(mine_dst.tolist())), tmax=t)
    finally:
        dist.destroy_process_group()


def test_two_rank_ring_exchange():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        res = dict(results)
    for r in range(world):
        assert res[r]["handles"] == [1, 2]
        assert res[r]["pages"] == [1000, 1001]
        assert res[r]["peer"] == (r + 1) % world and res[r]["src"] == (r - 1) % world
        assert res[r]["overlap"] == 0
        assert res[r]["tmax"] == 20.0
    # rank 0 addresses rank 1's receive region exactly as rank 1 lays it out
    assert res[0]["recv_dst"] == res[1]["mine_dst"]
    assert res[1]["recv_dst"] == res[0]["mine_dst"]


def test_ring_assignment_is_a_permutation():
    for world in (1, 2, 4, 8):
        peers = [cluster.ring_peer(r, world) for r in range(world)]
        assert sorted(peers) == list(range(world))
        assert all(cluster.ring_source(p, world) == r for r, p in enumerate(peers))
    with pytest.raises(ValueError):
        cluster.ring_peer(3, 2)
    with pytest.raises(ValueError):
        cluster.session_layout(0, 10, 6)
