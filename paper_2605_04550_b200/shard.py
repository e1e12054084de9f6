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


def gather_matrix_maps(maps: dict, count: int, shape, dst: int = 0, group=None, device=None):
    """The batch's final gather (north star: "no NCCL except a final gather of the sigma_min map"): every
    rank's maps from sharded_matrix_batch ({matrix index: (ny, nx) float64 values}) to rank `dst`, which
    returns the full (count, ny, nx) stack; the other ranks return None. One collective of the largest
    share per rank (ranks hold ceil(count/N) or floor(count/N) maps, padded with NaN to the same size).
    Works with gloo (CPU tensors) and nccl (CUDA tensors, `device`)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    per = (count + world - 1) // world
    ny, nx = shape
    mine = shard_indices(count, rank, world)
    buf = torch.full((per, ny, nx), float("nan"), dtype=torch.float64, device=device)
    for k, i in enumerate(mine.tolist()):
        v = maps[i]
        v = v.values if hasattr(v, "values") else v
        buf[k] = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(buf.device)
    out = torch.empty((world * per, ny, nx), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    if rank != dst:
        return None
    out = out.cpu().numpy().reshape(world, per, ny, nx)
    full = np.empty((count, ny, nx))
    for r in range(world):
        idx = shard_indices(count, r, world)
        full[idx] = out[r, : idx.size]
    return full
