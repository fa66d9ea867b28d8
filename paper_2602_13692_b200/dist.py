"""Multi-GPU plumbing: one replica per process (rank r holds replica r).

`connect()` all-gathers every rank's CUDA-IPC handle blob (HBM pool + barrier
mailbox, `ta_export_pool_handle`) over torch.distributed and maps every peer with
`ta_import_peer_pool`.  This is host-side setup only; the per-tick data path is
NVLink peer loads/stores and device-side flag barriers inside libta.
"""
from __future__ import annotations


def exchange(mine, rank: int, world: int, group=None):
    """All-gather (replica, handle) pairs; returns {replica: handle} of the peers."""
    import torch.distributed as dist
    got = [None] * world
    dist.all_gather_object(got, (rank, mine), group=group)
    out = {}
    for rep, h in got:
        if rep in out:
            raise RuntimeError(f"replica {rep} announced twice")
        if rep != rank:
            out[rep] = h
    if len(out) != world - 1:
        raise RuntimeError("missing peers in the handle exchange")
    return out


def connect(pool, group=None):
    """Map every other rank's pool and mailbox into `pool` (collective)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if pool.R != world or pool.here != 1:
        raise ValueError("multi-GPU mode needs n_replicas == world size and one replica per rank")
    peers = exchange(pool.export_handle(), pool.first, world, group)
    for rep in sorted(peers):
        pool.import_peer(rep, peers[rep])
    dist.barrier(group)
    return sorted(peers)
