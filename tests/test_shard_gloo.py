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


class _Grid:  # minimal ComplexGrid stand-in (points, shape) for the CPU test
    def __init__(self, ny, nx):
        self.shape = (ny, nx)
        x, y = np.linspace(-1, 1, nx), np.linspace(-2, 2, ny)
        self._p = x[None, :] + 1j * y[:, None]

    def points(self):
        return self._p


def _worker_restricted(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _Grid(9, 13)
    region = (np.arange(9 * 13).reshape(9, 13) * 7919) % 5 == 0
    calls = []

    def fake_sigma(z):
        calls.append(z.size)
        return np.abs(z) + 0.25 * z.imag
    vals = shard.sharded_restricted_sigma(g, region, fake_sigma)
    q.put((rank, calls, vals, region))
    dist.destroy_process_group()


def test_gloo_world2_restricted_map():
    """Guided mode across ranks: the region's points are dealt cyclically in row-major
    order (pseudospec core.py:204), each rank evaluates only its share, NaN elsewhere (core.py:203)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_restricted, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _Grid(9, 13)
    for rank, calls, vals, region in out:
        k = int(region.sum())
        assert calls == [shard.shard_count(k, rank, 2)]
        want = np.full(g.shape, np.nan)
        z = g.points()[region]
        want[region] = np.abs(z) + 0.25 * z.imag
        assert np.array_equal(np.isnan(vals), ~region)
        assert np.array_equal(vals[region], want[region])


def _worker_batch(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mats = [np.full((2, 2), float(i)) for i in range(7)]
    got = shard.sharded_matrix_batch(mats, None, evaluate_field=lambda A, g: float(A[0, 0]) * 10)
    maps = {i: np.full((3, 4), v) + np.arange(12).reshape(3, 4) for i, v in got.items()}
    full = shard.gather_matrix_maps(maps, len(mats), (3, 4))
    q.put((rank, (got, full)))
    dist.destroy_process_group()


def test_gloo_world2_matrix_batch():
    """C5-style batches: matrix i goes to rank i mod N, each map computed exactly once."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_batch, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = {r: v[0] for r, v in res.items()}
    assert sorted(out[0]) == [0, 2, 4, 6] and sorted(out[1]) == [1, 3, 5]
    assert all(v == 10 * i for part in out.values() for i, v in part.items())
    # the final gather: rank 0 holds every map in matrix order, the other rank nothing
    assert res[1][1] is None
    want = np.stack([np.full((3, 4), 10.0 * i) + np.arange(12).reshape(3, 4) for i in range(7)])
    assert np.array_equal(res[0][1], want)


def _worker_dynamic(rank, world, port, q):
    import time

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = [3, 40, 5, 1, 22, 8, 30, 2, 2, 15, 9]
    order = shard.lpt_order(costs)
    mats = [np.full((2, 2), float(i)) for i in range(len(costs))]

    def slow_eval(A, g):  # cost-proportional work, so the queue really interleaves the two ranks
        time.sleep(0.01 * costs[int(A[0, 0])])
        return float(A[0, 0]) * 10
    got = shard.dynamic_matrix_batch(mats, None, evaluate_field=slow_eval, order=order, key="t/pass0")
    again = shard.dynamic_matrix_batch(mats, None, evaluate_field=lambda A, g: 1.0, order=order, key="t/pass1")
    maps = {i: np.full((3, 4), v) + np.arange(12).reshape(3, 4) for i, v in got.items()}
    full = shard.gather_matrix_maps(maps, len(mats), (3, 4))
    q.put((rank, (got, sorted(again), full)))
    dist.destroy_process_group()


def test_lpt_order_and_local_queue():
    assert shard.lpt_order([3, 40, 5, 40, 0]) == [1, 3, 2, 0, 4]
    c = shard.LocalCounter()
    assert list(shard.dynamic_items([4, 2, 9], "k", c)) == [4, 2, 9]
    assert list(shard.dynamic_items([4, 2, 9], "k", c)) == []  # the key's pass is exhausted
    assert list(shard.dynamic_items([4, 2, 9], "k2", c)) == [4, 2, 9]


def test_gloo_world2_dynamic_matrix_batch():
    """C5 batches across ranks: ranks pull whole matrices from the process group's store
    counter in LPT order; every matrix is computed exactly once, both ranks get work, each pass (key) is an
    independent queue, and the gather reassembles any ownership in matrix order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dynamic, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 11
    got = {r: v[0] for r, v in res.items()}
    assert sorted(list(got[0]) + list(got[1])) == list(range(n))  # exactly once
    assert got[0] and got[1]
    assert sorted(res[0][1] + res[1][1]) == list(range(n))        # a fresh key is a fresh queue
    assert all(v == 10 * i for part in got.values() for i, v in part.items())
    assert res[1][2] is None
    want = np.stack([np.full((3, 4), 10.0 * i) + np.arange(12).reshape(3, 4) for i in range(n)])
    assert np.array_equal(res[0][2], want)
