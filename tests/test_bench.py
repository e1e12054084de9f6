"""bench.py plumbing on CPU: the --gpus N self-launch under torch.distributed.run (gloo self-test of the
cyclic deal, all-gather and max-over-ranks), and the reference arm's JSON line."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_bench_self_launches_ranks():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dist-selftest"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1  # rank 0 alone prints
    assert lines[0] == {"selftest": True, "world": 2, "max_over_ranks": 2.0, "gather_ok": True}


def test_reference_arm_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _json_lines(r.stdout)
    assert line["impl"] == "reference" and line["unit"] == "points/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["kind"] in ("reference", "port")


@pytest.mark.gpu
def test_bench_line_on_gpu():
    """One short C1 bench run on the GPU: a well-formed line whose dominant kernel window fits inside the step
    (the events bracket each launch on its own stream), with the library's own launch count."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "C1", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-guided"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _json_lines(r.stdout)
    assert line["metric"].startswith("sigma_min") and line["value"] > 0 and line["n_gpus"] == 1
    roof = line["roofline"]
    assert 0 < roof["share_of_step"] <= 1.001 and roof["frac"] > 0
    assert line["gpu_launches"] >= 3 * 2
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["engines"]["lanczos_points"] + line["engines"]["bisect_points"] == 2500


@pytest.mark.gpu
def test_bench_c5_batch_pass_on_gpu():
    """The headline's step structure on a 4-matrix batch: one pass covers every matrix once (the LPT queue),
    the e2e leg declares the whole batch's copies, and the per-matrix sweeps sum to the pass."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--matrices", "4", "--steps", "1", "--warmup", "1",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _json_lines(r.stdout)
    cfg = line["config"]
    assert cfg["matrices"] == 4 and cfg["points_per_step"] == 4 * 1024 * 1024
    assert sorted(p["matrix"] for p in line["phases_ms"]) == [0, 1, 2, 3]
    assert sum(p["sweep"] for p in line["phases_ms"]) == pytest.approx(line["ms_per_step"], rel=1e-3)
    assert line["e2e"]["d2h_bytes_per_step"] == 4 * 1024 * 1024 * 9 and line["e2e"]["value"] > 0
    assert 0 < line["roofline"]["share_of_step"] <= 1.001
