"""Host-side multi-process plumbing on CPU: the handle exchange of paper_2602_13692_b200.dist
over a world-size-2 gloo group (no GPU: handles are opaque bytes here)."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_13692_b200.dist import exchange
    peers = exchange(bytes([rank]) * 192, rank, world)
    q.put((rank, {k: v[:1] for k, v in peers.items()}))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_handle_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, peers in got.items():
        assert sorted(peers) == [r for r in range(world) if r != rank]
        assert all(peers[r] == bytes([r]) for r in peers)
