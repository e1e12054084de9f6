"""K3 — grid partitioner across the GPUs of one box (replaces pseudospec/core.py:186-195, the
ProcessPoolExecutor over row blocks).

Points of the (compacted) row-major point list are dealt cyclically, point p -> rank p mod N:
σ_min cost is spatially correlated (slow clusters outside the spectrum), so contiguous row
blocks (core.py:189) would unbalance the ranks, while a cyclic deal spreads every region over
all of them. Each rank evaluates its shard with its own device; the only exchange is the final
gather of the σ map (NCCL all-gather over NVLink on GPUs; gloo in the CPU tests). Values are
bitwise identical to the single-GPU map because every σ depends only on (A, z).
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_indices(P: int, rank: int, world: int) -> np.ndarray:
    """Indices of the points owned by `rank` under the cyclic deal."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return np.arange(rank, P, world, dtype=np.int64)


def shard_count(P: int, rank: int, world: int) -> int:
    return (P - rank + world - 1) // world if P > rank else 0


def assemble(parts: list[np.ndarray], P: int) -> np.ndarray:
    """Inverse of the cyclic deal: parts[r] holds the values of shard_indices(P, r, world)."""
    world = len(parts)
    out = np.empty(P, dtype=parts[0].dtype if parts else float)
    for r, vals in enumerate(parts):
        out[r::world] = vals
    return out


def gather_values(local: np.ndarray, P: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's shard values (float64) and reassemble the full length-P array.

    Shards differ in length by at most one; they are padded to the same length for the
    collective. Works with the gloo (CPU tensors) and nccl (CUDA tensors) backends."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    m = (P + world - 1) // world
    buf = torch.full((m,), float("nan"), dtype=torch.float64, device=device)
    buf[: local.size] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64)).to(buf.device)
    out = torch.empty(world * m, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    out = out.cpu().numpy().reshape(world, m)
    parts = [out[r, : shard_count(P, r, world)] for r in range(world)]
    return assemble(parts, P)


def sharded_sigma(zs: np.ndarray, evaluate: Callable[[np.ndarray], np.ndarray], group=None,
                  device=None) -> np.ndarray:
    """σ at every z of zs on this process group: evaluate the local cyclic shard, all-gather."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    zs = np.asarray(zs, dtype=complex).ravel()
    local = evaluate(zs[shard_indices(zs.size, rank, world)])
    return gather_values(np.asarray(local, dtype=np.float64), zs.size, group=group, device=device)


def sharded_full_pseudospectrum(A, grid, group=None, label: str = "matrix"):
    """full_pseudospectrum (core.py:177-195) across the ranks of `group`, one GPU per rank."""
    import torch
    from . import core
    dev = torch.device("cuda", torch.cuda.current_device())
    vals = sharded_sigma(grid.points().ravel(), lambda z: core.smin_many(A, z, label=label, device=dev.index),
                         group=group, device=dev)
    return core.SigmaField(grid, vals.reshape(grid.shape))


def sharded_restricted_sigma(grid, region: np.ndarray, evaluate: Callable[[np.ndarray], np.ndarray],
                             group=None, device=None) -> np.ndarray:
    """restricted_field's values (core.py:198-208) across the ranks of `group`: the region's points in
    row-major order (core.py:204) are dealt cyclically, evaluated per rank and all-gathered; every
    other grid point is NaN (core.py:203). Same bits as the single-GPU restricted map."""
    region = np.asarray(region, dtype=bool)
    if region.shape != tuple(grid.shape):
        raise ValueError(f"region shape {region.shape} != grid shape {tuple(grid.shape)}")
    idx = np.flatnonzero(region.ravel())
    out = np.full(region.size, np.nan)
    if idx.size:
        out[idx] = sharded_sigma(grid.points().ravel()[idx], evaluate, group=group, device=device)
    return out.reshape(grid.shape)


def sharded_hybrid_pseudospectrum(bundle, A, grid, eps: float, group=None, probe_seed: int = 0,
                                  stride: int = 4, label: str = "matrix"):
    """hybrid_pseudospectrum (pipeline.py:273-297) across the ranks of `group` (guided
    mode): every rank runs the predictor (K2) on its own GPU. That pass is deterministic, so all
    ranks hold the same region without exchanging anything. Only the restricted σ sweep (K1) is
    sharded, and its values are all-gathered."""
    import time

    import torch
    from . import core, pipeline
    if bundle.tau_star is None:
        raise core.ParameterError("model bundle carries no calibrated threshold")
    if eps <= 0:
        raise core.ParameterError(f"eps must be positive, got {eps}")
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    prob, n_evals = pipeline.hierarchical_predict(bundle, A, grid, stride=stride, probe_seed=probe_seed)
    region = pipeline.predicted_region(prob, bundle.tau_star)
    t_nn = time.perf_counter() - t0
    t0 = time.perf_counter()
    vals = sharded_restricted_sigma(grid, region, lambda z: core.smin_many(A, z, label=label, device=dev.index),
                                    group=group, device=dev)
    t_restricted = time.perf_counter() - t0
    fld = core.SigmaField(grid, vals)
    fld.eps = eps
    return pipeline.HybridResult(field=fld, region=region, prob_field=prob, t_nn=t_nn,
                                 t_restricted=t_restricted, nn_evaluations=n_evals)


def sharded_matrix_batch(matrices, grid, evaluate_field: Callable | None = None, group=None):
    """σ maps of a batch of matrices on one grid (BASELINE C5: 64 matrices, 1024^2 grid each), matrices
    dealt cyclically over the ranks of `group` (matrix i -> rank i mod N). Each rank
    evaluates whole maps for its matrices; the maps stay on the rank that computed them, so the
    result is {matrix index: SigmaField} for this rank's share and nothing is exchanged.
    `evaluate_field(A, grid)` defaults to core.full_pseudospectrum."""
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if evaluate_field is None:
        from . import core
        evaluate_field = core.full_pseudospectrum
    return {i: evaluate_field(matrices[i], grid) for i in shard_indices(len(matrices), rank, world).tolist()}


# ------------------------------------------------------------------ matrix batches: LPT dynamic queue
# C5's matrices differ in cost by 250x (4 ms .. 1.05 s per 1024^2 map on one B200, tools/c5_balance.py): the
# share of grid points outside the pseudospectrum (bisection engine) sets a matrix's cost. Dealing whole
# matrices cyclically makes the slowest rank's sum the job time (modelled efficiency 0.65 / 0.47 / 0.37 at
# N = 2 / 4 / 8 over the 64 measured maps), and splitting every matrix over the ranks multiplies each
# launch's latency-bound tail (0.84 / 0.65 / 0.48). So ranks pull whole matrices from one shared counter in
# longest-first (LPT) order of a cheap cost estimate: modelled 1.00 / 0.998 / 0.982 with the estimate below
# (tools/c5_costmodel.py). The counter lives in the process group's store (host side); the data path has no
# collective.
SPLIT_STRIDE = 16  # cost-estimate subgrid: every 16th grid point each way (4,096 points of a 1024^2 grid)
# Cost model fitted by tools/c5_costmodel.py over the 64 C5 maps (rank correlation 0.98 with the measured
# device time): ms ~ 0.407 (subgrid bisection points) + 0.0111 (subgrid Lanczos points); only the ratio
# matters for the order.
BIS_WEIGHT, LAN_WEIGHT = 1.0, 0.0273


def batch_cost_estimates(matrices, grid, stride: int = SPLIT_STRIDE, device=None) -> np.ndarray:
    """Per-matrix cost estimate: the engine split (core.engine_split, one classification test per point) on
    a coarse subgrid. Deterministic, so every rank computes the same estimates and order without exchange."""
    from . import core
    sub = np.ascontiguousarray(grid.points()[::stride, ::stride].ravel())
    est = np.empty(len(matrices))
    for i, A in enumerate(matrices):
        nb, nl = core.engine_split(A, sub, device=device)
        est[i] = BIS_WEIGHT * nb + LAN_WEIGHT * nl
    return est


def lpt_order(costs) -> list[int]:
    """Longest-processing-time-first order (ties by index)."""
    return sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))


class LocalCounter:
    """Single-process stand-in for the store's atomic counter."""

    def __init__(self):
        self._v = {}

    def add(self, key, amount):
        self._v[key] = self._v.get(key, 0) + amount
        return self._v[key]


def default_store():
    """The process group's key-value store (TCPStore under torchrun), or a local counter without one."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        from torch.distributed import distributed_c10d
        return distributed_c10d._get_default_store()
    return LocalCounter()


def dynamic_items(order, key: str, store=None):
    """Yield the items of `order` this rank pulls from the shared counter `key` (each item goes to exactly
    one rank: the store's add is atomic). Every pass over a batch needs a fresh key."""
    store = default_store() if store is None else store
    while True:
        k = int(store.add(key, 1)) - 1
        if k >= len(order):
            return
        yield order[k]


def dynamic_matrix_batch(matrices, grid, evaluate_field: Callable | None = None, order=None, key: str = "psb/batch",
                         store=None, device=None) -> dict:
    """σ maps of a batch of matrices on one grid (BASELINE C5), matrices pulled by the ranks from a shared
    LPT-ordered queue. Returns {matrix index: SigmaField} for the matrices this rank computed; the maps stay
    on their rank (gather_matrix_maps collects them). `order` defaults to lpt_order(batch_cost_estimates(...))."""
    if evaluate_field is None:
        from . import core

        def evaluate_field(A, g):
            return core.full_pseudospectrum(A, g, device=device)
    if order is None:
        order = lpt_order(batch_cost_estimates(matrices, grid, device=device))
    return {i: evaluate_field(matrices[i], grid) for i in dynamic_items(order, key, store)}


def gather_matrix_maps(maps: dict, count: int, shape, dst: int = 0, group=None, device=None):
    """The batch's final gather (north star: "no NCCL except a final gather of the sigma_min map"): every
    rank's maps ({matrix index: (ny, nx) float64 values or SigmaField}, from sharded_matrix_batch or
    dynamic_matrix_batch - any ownership) to rank `dst`, which returns the full (count, ny, nx) stack; the
    other ranks return None. Two collectives: the per-rank map counts, then one all-gather of every rank's
    maps padded with NaN to the largest share, each with its matrix indices (-1 = padding). Works with gloo
    (CPU tensors) and nccl (CUDA tensors, `device`)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ny, nx = shape
    mine = sorted(maps)
    cnt = torch.tensor([len(mine)], dtype=torch.int64, device=device)
    cnts = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    per = max(1, int(cnts.max().item()))
    buf = torch.full((per, ny, nx), float("nan"), dtype=torch.float64, device=device)
    idx = torch.full((per,), -1, dtype=torch.int64, device=device)
    for k, i in enumerate(mine):
        v = maps[i]
        v = v.values if hasattr(v, "values") else v
        buf[k] = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(buf.device)
        idx[k] = int(i)
    out = torch.empty((world * per, ny, nx), dtype=torch.float64, device=device)
    oidx = torch.empty(world * per, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    dist.all_gather_into_tensor(oidx, idx, group=group)
    if rank != dst:
        return None
    out = out.cpu().numpy()
    oidx = oidx.cpu().numpy()
    full = np.full((count, ny, nx), np.nan)
    seen = np.zeros(count, dtype=bool)
    for k, i in enumerate(oidx.tolist()):
        if i >= 0:
            if seen[i]:
                raise ValueError(f"matrix {i} held by more than one rank")
            full[i] = out[k]
            seen[i] = True
    if not seen.all():
        raise ValueError(f"matrices missing from the gather: {np.flatnonzero(~seen).tolist()}")
    return full
