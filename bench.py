#!/usr/bin/env python3
"""bench.py — throughput of the σ_min(zI - A) grid evaluator (the BASELINE.json metric).

Workload (BASELINE.json configs[1]): Grcar n=400, full 200 x 200 grid over
[-1,3] x [-3.5,3.5]; one step = one full-grid σ_min sweep (40,000 shifts, every value checked
by the parity suite against the reference's zgesdd). With N GPUs (torchrun, one rank per GPU)
the grid is widened to 200 x 200N over the same box and its points are dealt cyclically
(point p -> rank p mod N): per-GPU work is fixed (weak scaling), and the σ map is gathered to
rank 0 over NCCL at the end of every step — the only exchange in the path.

Keys beyond the driver contract:
  roofline      the dominant kernel of the step against its bound: the bisection engine is
                FP64-bound (peak = DFMA microbenchmark measured in this run, MEASURED_PEAKS.json
                has no FP64 figure); the Lanczos engine is HBM-bound (peak = MEASURED_PEAKS hbm_gbs)
  cpu_baseline  the oracle port (numpy zgesdd per shift = the reference's own computation,
                pseudospec/core.py:141-168) on a bounded sample, 1 thread, rank 0 at N=1 only
  e2e           the same metric through the public API (full_pseudospectrum / smin_many with
                host arrays: H2D of the shifts and D2H of the σ map inside the timed region)
--impl reference runs the oracle port on all host cores instead (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
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
WORKLOAD = "C2: Grcar n=400 (kl,ku)=(1,3), full 200x200 grid over [-1,3]x[-3.5,3.5], sigma_min at every point"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", help="workload (C1..C4); C2 is the headline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-guided", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

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
def _oracle_chunk(args):
    A, zs = args
    from oracle.sigma_oracle import smin_restated
    return smin_restated(A, zs)


def cpu_oracle_rate(A_dense, zs, cores: int) -> tuple[float, float]:
    """pts/s of the oracle port (reference computation) over zs with `cores` processes."""
    t0 = time.perf_counter()
    if cores <= 1:
        _oracle_chunk((A_dense, zs))
    else:
        from concurrent.futures import ProcessPoolExecutor
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        chunks = np.array_split(zs, cores * 2)
        with ProcessPoolExecutor(max_workers=cores) as ex:
            list(ex.map(_oracle_chunk, [(A_dense, c) for c in chunks]))
    dt = time.perf_counter() - t0
    return zs.size / dt, dt


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU computation (oracle port) on all host cores."""
    if rank != 0:
        return
    from paper_2605_04550_b200 import configs
    cfg = configs.CONFIGS[args.config]
    A = cfg.matrix(0).todense()
    if not np.iscomplexobj(A) or np.all(A.imag == 0):
        A = A.real.copy()
    cores = os.cpu_count() or 1
    per_step = {"C1": 40, "C2": 12, "C3": 1, "C4": 1}.get(args.config, 4) * cores
    rng = np.random.default_rng(7)
    pts = cfg.grid.points().ravel()
    for _ in range(args.warmup):
        cpu_oracle_rate(A, pts[rng.choice(pts.size, max(cores, per_step // 4), replace=False)], cores)
    times, npts = [], 0
    for _ in range(args.steps):
        zs = pts[rng.choice(pts.size, per_step, replace=False)]
        _, dt = cpu_oracle_rate(A, zs, cores)
        times.append(dt)
        npts += zs.size
    value = npts / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE config)",
        "config": {"workload": WORKLOAD if args.config == "C2" else args.config,
                   "sample_points_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{per_step} random grid shifts per step of the {args.config} grid, "
                                   f"numpy zgesdd per shift (pseudospec/core.py:141-168) in "
                                   f"{cores} processes, OPENBLAS_NUM_THREADS=1"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_guided(cfg, grid, args) -> dict:
    """BASELINE C2's MLP-guided run (pipeline.py:273-297): hierarchical prediction (K2) with the bundle
    the reference trained and calibrated (tests/golden/model_grcar.npz), 5x5-dilated region, restricted
    σ sweep (K1). Reports the reference's own timing split (t_nn incl. the host O(n^3) global_features,
    t_restricted) and its metrics against the full map (pipeline.py:300-331)."""
    import torch

    from paper_2605_04550_b200 import core, pipeline
    bundle = pipeline.load_npz(ROOT / "tests" / "golden" / "model_grcar.npz")
    A = cfg.matrix(0).todense().real
    eps = 0.01
    res = None
    t_nn, t_r = [], []
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        res = pipeline.hybrid_pseudospectrum(bundle, A, grid, eps=eps)
        if it >= args.warmup:
            t_nn.append(res.t_nn)
            t_r.append(res.t_restricted)
    gf_t = time.perf_counter()
    pipeline.global_features(A)
    gf_t = time.perf_counter() - gf_t
    full = core.full_pseudospectrum(cfg.matrix(0), grid)
    truth = full.values <= eps
    region = res.region
    tp = int((region & truth).sum())
    dil = core.dilate(truth, 3)
    recall = float((region & dil).sum() / dil.sum()) if dil.sum() else 1.0
    coverage = float(tp / truth.sum()) if truth.sum() else 1.0
    same = bool(np.array_equal(res.field.values[region], full.values[region]))
    tn, tr = float(np.median(t_nn)), float(np.median(t_r))
    return {"eps": eps, "tau_star": bundle.tau_star, "nn_evaluations": int(res.nn_evaluations),
            "grid_fraction": float(region.mean()), "t_nn_s": tn, "t_global_features_host_s": gf_t,
            "t_restricted_s": tr, "t_hybrid_s": tn + tr,
            "grid_points_per_s": grid.size / (tn + tr), "recall": recall, "coverage": coverage,
            "restricted_equals_full_bitwise": same,
            "note": "t_nn includes the host O(n^3) global_features (eig/svd, SURVEY 8f row 1)"}


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2605_04550_b200 import _lib, configs, core

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    h = _lib.handle(local_rank)
    cfg = configs.CONFIGS[args.config]
    A = cfg.matrix(0)
    g0 = cfg.grid
    grid = core.make_grid(g0.x_min, g0.x_max, g0.y_min, g0.y_max, g0.nx * world, g0.ny)
    pts = grid.points().ravel()
    mine = np.ascontiguousarray(pts[rank::world])
    P = mine.size
    with h.lock:
        core._set_matrix(h, A)
    d_zs = torch.from_numpy(mine.view(np.float64).copy()).to(dev)
    d_out = torch.empty(P, dtype=torch.float64, device=dev)
    d_iters = torch.empty(P, dtype=torch.int32, device=dev)
    d_status = torch.empty(P, dtype=torch.int8, device=dev)
    gathered = torch.empty(world * P, dtype=torch.float64, device=dev) if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        rc = h.lib.psb_smin_points_device(h.h, C.c_void_p(d_zs.data_ptr()), P, None,
                                          C.c_void_p(d_out.data_ptr()), C.c_void_p(d_iters.data_ptr()),
                                          C.c_void_p(d_status.data_ptr()), C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"psb_smin_points_device failed: {h.error()}")
        if world > 1:
            dist.all_gather_into_tensor(gathered, d_out)

    def barrier():
        if world > 1:
            dist.barrier()

    sampler = ClockSampler(local_rank)  # covers warm-up, the timed steps and the e2e leg
    sampler.start()
    time.sleep(0.3)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    # correctness guard on the timed configuration: every point converged
    st = d_status.cpu().numpy()
    assert (st <= 2).all(), "non-converged points in the benchmark step"

    stats = []
    step_ms = []
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.random_(0, 255)  # evict L2 (256 MiB > 126 MB) between timed steps, outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        stats.append(h.stats())
    torch.cuda.synchronize()
    barrier()

    ms_local = float(np.mean(step_ms))
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * P / (ms * 1e-3)

    # ---- e2e through the public API, host buffers, copies inside the timed region
    e2e_ms = []
    for it in range(args.warmup + args.steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            fld = core.full_pseudospectrum(A, grid)
        else:
            out = core.smin_many(A, mine)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if it >= args.warmup:
            e2e_ms.append(dt)
    clocks = sampler.stop()
    te = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * P / (float(te.item()) * 1e-3)
    # grid path: the two axes (shifts are formed on the device); sharded path: this rank's shifts
    h2d = (grid.nx + grid.ny) * 8 if world == 1 else P * 16
    d2h = (grid.size * 9) if world == 1 else P * 9       # sigma (f64) + status (i8)

    # ---- roofline of the dominant kernel
    s = stats[-1]
    fp64_peak = h.fp64_peak()
    hbm_peak = 6455.9
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            hbm_peak = float(json.loads(mp.read_text())["hbm_gbs"])
        except Exception:
            pass
    kern = {
        "bisect": {"bound": "fp64", "achieved": s["flops_bisect"] / (s["ms_bisect"] * 1e-3) / 1e12,
                   "peak": fp64_peak, "unit": "TFLOP/s", "ms": s["ms_bisect"]},
        "lanczos": {"bound": "hbm", "achieved": s["bytes_lanczos"] / (s["ms_lanczos"] * 1e-3) / 1e9
                    if s["ms_lanczos"] > 0 else 0.0, "peak": hbm_peak, "unit": "GB/s", "ms": s["ms_lanczos"]},
    }
    for v in kern.values():
        v["frac"] = v["achieved"] / v["peak"] if v["peak"] else None
    dom = "bisect" if s["ms_bisect"] >= s["ms_lanczos"] else "lanczos"
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    roof = dict(kern[dom])
    roof["kernel"] = f"k_{dom}"
    roof["traffic"] = traffic
    # per-z FP64 roofline of the whole step (north star): G*P_FP64 / mean flops per point
    flops_pt = (s["flops_bisect"] + s["flops_lanczos"]) / max(1, s["n_points"])
    roof_pts = fp64_peak * 1e12 / flops_pt if flops_pt > 0 else None

    guided = None
    if rank == 0 and world == 1 and args.config in ("C1", "C2") and not args.no_guided:
        guided = run_guided(cfg, grid, args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Ad = A.todense()
        Ad = Ad.real.copy() if np.all(Ad.imag == 0) else Ad
        rng = np.random.default_rng(11)
        ns = {"C1": 2500, "C2": 200, "C3": 12, "C4": 3}.get(args.config, 8)
        zs = pts[rng.choice(pts.size, ns, replace=False)]
        rate, dt = cpu_oracle_rate(Ad, zs, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{ns} random shifts of the {args.config} grid, numpy zgesdd per shift "
                         f"(the reference's pseudospec/core.py:141-168 computation), 1 thread, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded BASELINE config, no dataset)",
            "config": {"workload": WORKLOAD if args.config == "C2" else cfg.description,
                       "grid": f"{grid.ny}x{grid.nx}", "points_per_gpu": P, "points_total": world * P,
                       "sharding": "cyclic point p -> rank p mod N; sigma map all-gathered over NCCL each step",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": f"dp{world}"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "core.full_pseudospectrum" if world == 1 else "core.smin_many (rank shard)"},
            "roofline": roof,
            "roofline_kernels": kern,
            "per_z_fp64_roofline": {"points_per_s": roof_pts * world if roof_pts else None,
                                    "frac": value / (roof_pts * world) if roof_pts else None,
                                    "flops_per_point": flops_pt},
            "engines": {"lanczos_points": s["n_lanczos"], "bisect_points": s["n_bisect"],
                        "lanczos_steps": s["lanczos_iters"], "pd_tests": s["pd_tests"]},
            # per step: the classification kernel, then engine L and engine B when they have points
            "gpu_launches": int(sum(1 + (s_["grid_lanczos"] > 0) + (s_["grid_bisect"] > 0) for s_ in stats)),
            "clocks": clocks,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if guided:
            line["guided"] = guided
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
