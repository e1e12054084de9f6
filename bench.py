#!/usr/bin/env python3
"""bench.py — throughput of the σ_min(zI - A) grid evaluator (the BASELINE.json metric).

Headline workload (BASELINE.json configs[4], the config the 1/2/4/8-GPU metric is
quoted on): 64 seeded noisy banded Toeplitz matrices, n=4000, (kl,ku)=(3,3), complex128, a full
1024 x 1024 grid each. One step = one pass over the whole batch (64 x 1,048,576 σ_min) by all GPUs
together ("scaling": "strong"): the ranks pull whole matrices from one counter in the process group's
store, in longest-first order of a subgrid cost estimate (shard.dynamic_matrix_batch; the matrices'
costs differ 250x, so a fixed deal would leave most GPUs idle behind the slowest). The matrices are
independent objects: no data-path collective; each rank keeps the σ maps it computed. A
pass takes as long as its busiest rank's device time (max over ranks per pass).

--config C1..C4 are the single-matrix configs (secondary lines). Their fixed grid is dealt cyclically
(point p -> rank p mod N, shard.py) and the σ map is all-gathered over NCCL inside every step, the
path's only exchange ("scaling": "strong").

--gpus N without torchrun re-executes this script under `torch.distributed.run` with N ranks
(one process per GPU, rendezvous on 127.0.0.1).

Keys beyond the driver contract:
  roofline          the dominant kernel of the step (largest CUDA-event window) against its bound;
                    every window is taken from events recorded on that kernel's own stream, with no
                    host round trip inside. Bisection/classification: FP64 (peak = DFMA
                    microbenchmark measured in this run; MEASURED_PEAKS.json has no FP64 figure);
                    Lanczos: HBM (peak = MEASURED_PEAKS hbm_gbs).
  lu_solve_model    SURVEY §8(d)'s algorithmic per-z model (LU + k(z) inverse-Lanczos steps, band bytes)
  cpu_baseline      the oracle port (numpy zgesdd per shift = the reference's computation,
                    pseudospec/core.py:141-168) on a bounded sample, rank 0 at N=1 only
  e2e               the same metric through the public API (full_pseudospectrum with host arrays:
                    band, axes H2D and the σ map D2H inside the timed region)
--impl reference runs the reference's CPU computation on all host cores instead (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sigma_min(zI-A) grid points/sec at 1/2/4/8 B200; % of per-z FP64/HBM roofline"
UNIT = "points/s"
WORKLOAD = {
    "C5": "C5: 64 seeded noisy banded Toeplitz n=4000 (3,3) complex128, full 1024x1024 grid per matrix; "
          "one step = one pass over the whole batch (64 x 1,048,576 sigma_min) on all GPUs together",
    "C4": "C4: convection-diffusion n=2000 Pe=50 (1,1), fixed 512x512 grid dealt over the GPUs",
    "C3": "C3: complex banded Toeplitz n=1000 (2,3), fixed 256x256 grid dealt over the GPUs",
    "C2": "C2: Grcar n=400 (1,3), fixed 200x200 grid over [-1,3]x[-3.5,3.5] dealt over the GPUs",
    "C1": "C1: Grcar n=100 (1,3), fixed 50x50 grid over [-1,3]x[-3.5,3.5] dealt over the GPUs",
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", help="workload C1..C5; C5 (BASELINE configs[4]) is the headline")
    ap.add_argument("--matrices", type=int, default=0,
                    help="C5 development runs: the first M matrices of the batch (default: all 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-guided", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--dist-selftest", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- launcher
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: run this script as N ranks (one per GPU) on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator log (nranks) for the driver
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9
                          for i, v in enumerate(r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU legs
def host_info() -> dict:
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')}"
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "blas": blas, "numpy": np.__version__}


def _dense(cfg, m=0):
    A = cfg.matrix(m).todense()
    return A.real.copy() if np.all(A.imag == 0) else A


def _oracle_chunk(args):
    A, zs, threads = args
    from oracle.sigma_oracle import smin_restated
    return smin_restated(A, zs, threads=threads)


def _reference_chunk(args):
    """The reference package's own smin_many (baseline/_ref, stock code path; real A only). BLAS threads are
    set explicitly: forked pool children inherit the parent's initialised OpenBLAS, so OPENBLAS_NUM_THREADS
    set after numpy's import would not reach them (SURVEY §0.6's 8 x 8 oversubscription)."""
    A, zs, threads = args
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    from threadpoolctl import threadpool_limits

    from pseudospec import core as rcore
    with threadpool_limits(threads):
        return rcore.smin_many(A, zs, chunk=1)


def _reference_available() -> bool:
    return (ROOT / "baseline" / "_ref" / "pseudospec" / "core.py").exists()


def cpu_rate(fn, A_dense, zs, procs: int, blas_threads: int, pool=None) -> tuple[float, float]:
    """pts/s of `fn` over zs: on `pool` (a process pool of `procs` workers, each with `blas_threads` BLAS
    threads) or in-process."""
    t0 = time.perf_counter()
    if procs <= 1 or pool is None:
        fn((A_dense, zs, blas_threads))
    else:
        chunks = [c for c in np.array_split(zs, procs) if c.size]
        list(pool.map(fn, [(A_dense, c, blas_threads) for c in chunks]))
    dt = time.perf_counter() - t0
    return zs.size / dt, dt


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU computation of the path on the host cores, rank 0 only.
    Real A (C1, C2, C4): the reference package's own smin_many from baseline/_ref, one process per core
    (OPENBLAS_NUM_THREADS=1: SURVEY §0.6's best reference configuration). Complex A (C3, C5): the reference
    casts A to real (core.py:112-119), so the oracle port (the same zgesdd call without the cast) runs.
    n=4000 (C5) takes ~75 s per shift on one core, so its step is one shift on all cores' BLAS threads."""
    if rank != 0:
        return
    from paper_2605_04550_b200 import configs
    cfg = configs.CONFIGS[args.config]
    A = _dense(cfg)
    cores = os.cpu_count() or 1
    real = not np.iscomplexobj(A)
    fn, kind = (_reference_chunk, "reference") if real and _reference_available() else (_oracle_chunk, "port")
    if args.config == "C5":
        per_step, procs, blas = 1, 1, cores
    else:
        per_step, procs, blas = {"C1": 40, "C2": 4, "C3": 1, "C4": 1}[args.config] * cores, cores, 1
    rng = np.random.default_rng(7)
    pts = cfg.grid.points().ravel()
    pool = None
    if procs > 1:  # one pool for the whole run (worker start-up and imports stay out of the steps)
        from concurrent.futures import ProcessPoolExecutor
        pool = ProcessPoolExecutor(max_workers=procs)
    times, npts = [], 0
    try:
        for _ in range(args.warmup):
            cpu_rate(fn, A, pts[rng.choice(pts.size, per_step, replace=False)], procs, blas, pool)
        for _ in range(args.steps):
            zs = pts[rng.choice(pts.size, per_step, replace=False)]
            _, dt = cpu_rate(fn, A, zs, procs, blas, pool)
            times.append(dt)
            npts += zs.size
    finally:
        if pool is not None:
            pool.shutdown()
    value = npts / sum(times)
    how = (f"{per_step} random grid shift(s) per step of the {args.config} grid, "
           + ("pseudospec.core.smin_many (baseline/_ref, unmodified)" if kind == "reference"
              else "numpy zgesdd per shift (oracle port of pseudospec/core.py:141-168, complex A kept)")
           + (f" in {procs} processes, OPENBLAS_NUM_THREADS=1" if procs > 1 else f", {blas} BLAS threads"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded BASELINE config)",
        "config": {"workload": WORKLOAD[args.config], "sample_points_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": how, **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_line(cfg, name) -> dict:
    """The oracle port on a bounded sample (~10-30 s), rank 0 at N=1."""
    A = _dense(cfg)
    pts = cfg.grid.points().ravel()
    rng = np.random.default_rng(11)
    cores = os.cpu_count() or 1
    if name == "C5":  # ~75 s per shift on one core: one shift on all cores' BLAS threads
        ns, threads = 1, cores
    else:
        ns, threads = {"C1": 2500, "C2": 200, "C3": 12, "C4": 3}[name], 1
    zs = pts[rng.choice(pts.size, ns, replace=False)]
    rate, dt = cpu_rate(_oracle_chunk, A, zs, 1, threads)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{ns} random shift(s) of the {name} grid, numpy zgesdd per shift (the reference's "
                      f"pseudospec/core.py:141-168 computation), {threads} BLAS thread(s), {dt:.1f} s",
            **host_info()}


# ----------------------------------------------------------------------------- our arm
def run_guided(name, cfg, args) -> dict:
    """The MLP-guided run (pipeline.py:273-297): hierarchical prediction (K2), 5x5-dilated region, restricted
    σ sweep on the device-side selection (K1). C1/C2 (BASELINE configs[1]) use the bundle the reference
    trained and calibrated on a Grcar family (tests/golden/model_grcar.npz, eps 0.01); C4 (configs[3])
    the one it trained on a convection-diffusion family (model_c4.npz), in the exact power-of-two units
    oracle/make_guided_c4.py explains. Reports the reference's timing split and its metrics against the
    full map (pipeline.py:300-331)."""
    import torch

    from paper_2605_04550_b200 import core, pipeline
    grid = cfg.grid
    if name == "C4":
        mz = np.load(ROOT / "tests" / "golden" / "model_c4.npz")
        bundle = pipeline.load_npz(ROOT / "tests" / "golden" / "model_c4.npz")
        S, eps = float(mz["scale"]), float(mz["eps"])
        A0 = cfg.matrix(0)
        Ab = core.BandMatrix(A0.band * S, A0.kl, A0.ku)
        grid = core.make_grid(grid.x_min * S, grid.x_max * S, grid.y_min * S, grid.y_max * S, grid.nx, grid.ny)
        units = f"A and z scaled by {S:g} (exact power of two)"
    else:
        bundle = pipeline.load_npz(ROOT / "tests" / "golden" / "model_grcar.npz")
        Ab, eps, units = cfg.matrix(0), 0.01, "as configured"
    res = None
    t_nn, t_r = [], []
    pipeline.clear_feature_cache()
    t_cold = None
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        res = pipeline.hybrid_pseudospectrum(bundle, Ab, grid, eps=eps)  # the band form: no dense n x n per call
        if t_cold is None:
            t_cold = res.t_nn  # host global_features computed in this call
        if it >= args.warmup:
            t_nn.append(res.t_nn)
            t_r.append(res.t_restricted)
    full = core.full_pseudospectrum(Ab, grid)
    truth = full.values <= eps
    region = res.region
    tp = int((region & truth).sum())
    dil = core.dilate(truth, 3)
    recall = float((region & dil).sum() / dil.sum()) if dil.sum() else 1.0
    coverage = float(tp / truth.sum()) if truth.sum() else 1.0
    same = bool(np.array_equal(res.field.values[region], full.values[region]))
    tn, tr = float(np.median(t_nn)), float(np.median(t_r))
    return {"eps": eps, "units": units, "tau_star": bundle.tau_star, "nn_evaluations": int(res.nn_evaluations),
            "grid_fraction": float(region.mean()), "t_nn_s": tn, "t_nn_cold_s": t_cold,
            "t_restricted_s": tr, "t_hybrid_s": tn + tr,
            "grid_points_per_s": grid.size / (tn + tr), "recall": recall, "coverage": coverage,
            "restricted_equals_full_bitwise": same,
            "note": "t_nn: median over timed calls, host global_features served from the per-matrix cache; "
                    "t_nn_cold_s: the first call, which computes them (host eig/svd, O(n^3))"}


def lu_solve_model(n, kl, ku, s, fp64_tf, hbm_gbs) -> dict:
    """F(z) = F_LU + k(z) F_it, F_LU = n p (8(p+q)+6), F_pair = n (8p + 8(p+q) + 6),
    F_it = 2 F_pair + 40 n, B_band = 16 n (2p+q+1); t_roof(z) = max(F/P_FP64, B_band/BW). k(z) is recorded by
    K1 for the engine-L points (mean k below); engine-B points carry no Lanczos count, so the model is
    evaluated over engine-L points, where the kernel runs exactly this algorithm."""
    p, q = kl, ku
    f_lu = n * p * (8 * (p + q) + 6)
    f_it = 2 * n * (8 * p + 8 * (p + q) + 6) + 40 * n
    b_band = 16 * n * (2 * p + q + 1)
    kbar = s["lanczos_iters"] / s["n_lanczos"] if s["n_lanczos"] else 0.0
    f = f_lu + kbar * f_it
    t = max(f / (fp64_tf * 1e12), b_band / (hbm_gbs * 1e9))
    return {"F_LU": f_lu, "F_it": f_it, "B_band": b_band, "k_mean_engine_L": kbar, "flops_per_point": f,
            "bound": "fp64" if f / (fp64_tf * 1e12) >= b_band / (hbm_gbs * 1e9) else "hbm",
            "roof_points_per_s_per_gpu": 1.0 / t}


def _sum_stats(stats: list[dict]) -> dict:
    keys = ["n_points", "n_lanczos", "n_bisect", "lanczos_iters", "pd_tests", "flops_bisect", "flops_lanczos",
            "bytes_lanczos", "ms_bisect", "ms_lanczos", "ms_total", "ms_classify", "flops_classify", "ms_fallback",
            "launches"]
    return {k: sum(s[k] for s in stats) for k in keys}


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2605_04550_b200 import _lib, configs, core, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    h = _lib.handle(local_rank)
    name = args.config
    cfg = configs.CONFIGS[name]
    grid = cfg.grid
    batch = cfg.batch > 1
    pts = grid.points().ravel()
    if batch:
        # One step = one pass over the batch, all ranks together: ranks pull whole matrices (every rank
        # evaluates the full grid of the matrices it pulls) from the process group's store counter in
        # longest-first order of a subgrid cost estimate (shard.py). No data-path collective.
        nmat = min(args.matrices, cfg.batch) if args.matrices > 0 else cfg.batch
        mine = pts
        mats = [cfg.matrix(m) for m in range(nmat)]
        t_plan = time.perf_counter()
        costs = shard.batch_cost_estimates(mats, grid, device=local_rank)
        order = shard.lpt_order(costs)
        plan_s = time.perf_counter() - t_plan
        store = shard.default_store()
    else:
        mine = np.ascontiguousarray(pts[rank::world])
        A0 = cfg.matrix(0)

        def matrix_of(step):
            return 0, A0
    P = mine.size
    d_zs = torch.from_numpy(np.ascontiguousarray(mine).view(np.float64).copy()).to(dev)
    d_out = torch.empty(P, dtype=torch.float64, device=dev)
    d_iters = torch.empty(P, dtype=torch.int32, device=dev)
    d_status = torch.empty(P, dtype=torch.int8, device=dev)
    m_pad = (pts.size + world - 1) // world
    gather_in = torch.full((m_pad,), float("nan"), dtype=torch.float64, device=dev) if (world > 1 and not batch) else None
    gathered = torch.empty(world * m_pad, dtype=torch.float64, device=dev) if gather_in is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # a dedicated stream (not the legacy default one, whose handle is 0 and would make the library fall back
    # to its own unordered stream): the L2 flush, the step's kernels and the timing events are then ordered
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    def step():
        rc = h.lib.psb_smin_points_device(h.h, C.c_void_p(d_zs.data_ptr()), P, None,
                                          C.c_void_p(d_out.data_ptr()), C.c_void_p(d_iters.data_ptr()),
                                          C.c_void_p(d_status.data_ptr()), C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"psb_smin_points_device failed: {h.error()}")
        if gathered is not None:  # the path's one exchange: the σ map all-gathered over NCCL
            gather_in[:P].copy_(d_out)
            dist.all_gather_into_tensor(gathered, gather_in)

    def barrier():
        if world > 1:
            dist.barrier()

    def timed_item(A):
        """One matrix's sweep: the band resident on the device and L2 flushed first (outside the events)."""
        with h.lock:
            core._set_matrix(h, A)
        flush.random_(0, 255)  # evict L2 (256 MiB > 126 MB) between timed sweeps, outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        st_ = h.stats()
        assert (d_status.cpu().numpy() <= 2).all(), "non-converged points in a timed sweep"
        return e0.elapsed_time(e1), st_

    sampler = ClockSampler(local_rank)  # covers warm-up, the timed steps and the e2e leg
    sampler.start()
    time.sleep(0.3)
    stats, step_ms, pass_items = [], [], []
    if batch:
        def run_pass(key):
            """This rank's share of one pass: [(matrix, device ms, stats)] of the matrices it pulled."""
            return [(m, *timed_item(mats[m])) for m in shard.dynamic_items(order, key, store)]

        for w in range(max(args.warmup, 0)):
            run_pass(f"bench/warmup{w}")
            barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            items = run_pass(f"bench/step{k}")
            barrier()
            pass_items.append(items)
            step_ms.append(float(sum(ms_ for _, ms_, _ in items)))  # this rank's device time in the pass
            stats.extend(st_ for _, _, st_ in items)
        torch.cuda.synchronize()
        # the step (pass) takes as long as its busiest rank: max over ranks per pass
        tp = torch.tensor(step_ms, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        ms = float(tp.mean().item())
        units = nmat * P  # points every rank together finishes per step
    else:
        with h.lock:
            core._set_matrix(h, matrix_of(0)[1])
        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize()
        assert (d_status.cpu().numpy() <= 2).all(), "non-converged points in the benchmark step"
        barrier()
        torch.cuda.synchronize()
        A0m = matrix_of(0)[1]
        for _ in range(args.steps):
            ms_, st_ = timed_item(A0m)
            barrier()
            step_ms.append(ms_)
            stats.append(st_)
        torch.cuda.synchronize()
        barrier()
        # max over ranks of the summed step time (each rank runs the same number of steps)
        t = torch.tensor([float(np.sum(step_ms))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item()) / args.steps
        units = pts.size
    value = units / (ms * 1e-3)

    # ---- e2e through the public API, host buffers, copies inside the timed region
    e2e_ms, h2d, d2h = [], 0, 0
    if not args.no_e2e and batch:
        # one pass over the batch through the public API (host band and axes in, the σ map and status out, per
        # matrix), the same queue and order; the pass ends when the last rank finishes (max over ranks)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for m in shard.dynamic_items(order, "bench/e2e", store):
            core.full_pseudospectrum(mats[m], grid, device=local_rank)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = sum(A.band.size * 16 + (grid.nx + grid.ny) * 8 for A in mats)  # the whole batch, every rank's share
        d2h = nmat * grid.size * 9  # σ (f64) + status (i8) of every map
    elif not args.no_e2e:
        A = matrix_of(0)[1]
        for it in range(args.warmup + args.steps):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if world == 1:
                core.full_pseudospectrum(A, grid, device=local_rank)
            else:
                shard.sharded_full_pseudospectrum(A, grid)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            if it >= args.warmup:
                e2e_ms.append(dt)
        band_bytes = A.band.size * 16
        if world == 1:
            h2d = band_bytes + (grid.nx + grid.ny) * 8
            d2h = grid.size * 9  # σ (f64) + status (i8)
        else:
            h2d = band_bytes + P * 16 + m_pad * 8  # band, this rank's shifts, its padded shard for the gather
            d2h = P * (8 + 4 + 1) + world * m_pad * 8  # its σ / iters / status, the gathered map
    clocks = sampler.stop()
    e2e_value = None
    if e2e_ms:
        te = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = units / (float(te.item()) * 1e-3)

    # ---- roofline of the dominant kernel (largest CUDA-event window of the step)
    S = _sum_stats(stats)
    fp64_peak = h.fp64_peak()
    hbm_peak = 6455.9
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            hbm_peak = float(json.loads(mp.read_text())["hbm_gbs"])
        except Exception:
            pass
    K = args.steps

    def kern(bound, work, ms_sum, kname):
        ms_k = ms_sum / K
        if bound == "fp64":
            ach = work / (ms_sum * 1e-3) / 1e12 if ms_sum > 0 else 0.0
            d = {"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s"}
        else:
            ach = work / (ms_sum * 1e-3) / 1e9 if ms_sum > 0 else 0.0
            d = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s"}
        d.update({"frac": ach / d["peak"], "ms": ms_k, "kernel": kname,
                  "work_per_launch": work / K})
        return d

    kerns = {
        "bisect": kern("fp64", S["flops_bisect"], S["ms_bisect"], "k_bisect (engine B, mode 1)"),
        "lanczos": kern("hbm", S["bytes_lanczos"], S["ms_lanczos"], "k_lanczos (engine L)"),
        "classify": kern("fp64", S["flops_classify"], S["ms_classify"], "k_bisect (mode 0, classification)"),
    }
    dom = max(kerns, key=lambda k: kerns[k]["ms"])
    roof = dict(kerns[dom])
    ms_local = float(np.mean(step_ms))
    assert roof["ms"] <= ms_local * 1.001 + 1e-3, f"kernel window {roof['ms']} ms > step {ms_local} ms"
    roof["share_of_step"] = roof["ms"] / ms_local
    # the engines overlap inside a step, so their windows sum to more than the step; ncu serialises them:
    # the window's share of the summed windows is the figure to hold against profiles/*_launches.csv
    roof["share_of_serialised_kernels"] = roof["ms"] / max(1e-12, sum(k["ms"] for k in kerns.values()))
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(name, {}).get(dom)
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    n_, kl_, ku_ = (cfg.matrix(0).n, cfg.matrix(0).kl, cfg.matrix(0).ku)
    flops_pt = (S["flops_bisect"] + S["flops_lanczos"] + S["flops_classify"]) / max(1, S["n_points"])
    roof_pts = fp64_peak * 1e12 / flops_pt if flops_pt > 0 else None
    model = lu_solve_model(n_, kl_, ku_, S, fp64_peak, hbm_peak)
    model["frac_of_roof"] = value / (model["roof_points_per_s_per_gpu"] * world)

    guided = None
    if rank == 0 and world == 1 and name in ("C1", "C2", "C4") and not args.no_guided:
        guided = run_guided(name, cfg, args)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(cfg, name)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded BASELINE config, no dataset)",
            "config": {"workload": WORKLOAD[name], "grid": f"{grid.ny}x{grid.nx}",
                       "points_per_gpu": units / world if batch else P,
                       "points_per_step": units,
                       **({"matrices": nmat,
                           "matrices_rank0_per_pass": [len(it) for it in pass_items],
                           "schedule": "ranks pull whole matrices from one store counter in longest-first order "
                                       "of a cost estimate (engine split on every 16th grid point each way); "
                                       "no data-path collective; a pass takes its busiest rank's device time",
                           "plan_s": plan_s} if batch else {}),
                       "sharding": ("whole matrices per rank, LPT dynamic queue (shard.dynamic_matrix_batch)"
                                    if batch else "cyclic point p -> rank p mod N; sigma map all-gathered over "
                                                  "NCCL inside every step"),
                       "l2": "flushed before every timed matrix sweep (256 MiB write, outside the events)",
                       "parallelism": f"dp{world}"},
            "roofline": roof,
            "roofline_kernels": kerns,
            "per_z_fp64_roofline": {"executed_flops_per_point": flops_pt,
                                    "points_per_s": roof_pts * world if roof_pts else None,
                                    "frac": value / (roof_pts * world) if roof_pts else None},
            "lu_solve_model": model,
            "phases_ms": ([{"matrix": m, "sweep": round(ms_, 3),
                            **{k[3:]: round(st_[k], 3) for k in ("ms_classify", "ms_bisect", "ms_lanczos", "ms_fallback")}}
                           for m, ms_, st_ in pass_items[0]] if batch else
                          [{"step": round(step_ms[i], 3),
                            **{k[3:]: round(st_[k], 3) for k in ("ms_total", "ms_classify", "ms_bisect", "ms_lanczos",
                                                               "ms_fallback")}}
                           for i, st_ in enumerate(stats)]),
            "engines": {"lanczos_points": S["n_lanczos"] // K, "bisect_points": S["n_bisect"] // K,
                        "lanczos_steps": S["lanczos_iters"] // K, "pd_tests": S["pd_tests"] // K},
            "gpu_launches": int(S["launches"]),
            "clocks": clocks,
        }
        if e2e_value is not None:
            line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                           "api": ("core.full_pseudospectrum per matrix, matrices from the LPT queue (one pass)"
                                   if batch else "core.full_pseudospectrum" if world == 1
                                   else "shard.sharded_full_pseudospectrum")}
        if cpu:
            line["cpu_baseline"] = cpu
        if guided:
            line["guided"] = guided
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launcher self-test
def run_dist_selftest(rank, world):
    """CPU check of the multi-rank plumbing (gloo): cyclic deal, all-gather, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2605_04550_b200 import configs, shard
    grid = configs.CONFIGS["C1"].grid
    zs = grid.points().ravel()
    vals = shard.sharded_sigma(zs, lambda z: np.abs(z) + rank * 0.0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"selftest": True, "world": world, "max_over_ranks": float(t.item()),
                          "gather_ok": bool(np.array_equal(vals, np.abs(zs)))}), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"[bench] note: WORLD_SIZE={world} ranks, --gpus {args.gpus}; reporting n_gpus={world}",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if args.dist_selftest:
        dist.init_process_group("gloo")
        try:
            run_dist_selftest(rank, world)
        finally:
            dist.destroy_process_group()
        return
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
