"""K3 partitioner (CPU, gloo, world_size 2): cyclic deal + all-gather reassembles the map exactly."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_04550_b200 import shard


def test_cyclic_deal_roundtrip():
    for P in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            parts = [np.arange(P)[shard.shard_indices(P, r, world)] for r in range(world)]
            assert sum(p.size for p in parts) == P
            assert all(p.size == shard.shard_count(P, r, world) for r, p in enumerate(parts))
            if P:
                assert np.array_equal(shard.assemble(parts, P), np.arange(P))


def _worker(rank, world, port, P, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    zs = np.exp(1j * np.linspace(0, 6, P)) * np.linspace(1, 2, P)
    calls = []

    def fake_sigma(z):  # stands in for core.smin_many on a CPU-only box
        calls.append(z.size)
        return np.abs(z) ** 2 + 0.5 * z.real
    vals = shard.sharded_sigma(zs, fake_sigma)
    q.put((rank, calls, vals))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("P", [1001, 8])
def test_gloo_world2_gather(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, P, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    zs = np.exp(1j * np.linspace(0, 6, P)) * np.linspace(1, 2, P)
    want = np.abs(zs) ** 2 + 0.5 * zs.real
    for rank, calls, vals in out:
        assert calls == [shard.shard_count(P, rank, 2)]  # each rank evaluated only its shard
        assert np.array_equal(vals, want)                 # and holds the full map after the gather
