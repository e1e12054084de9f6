"""Field / mask CSV writers: libpsb200.so's host writers against the
reference's own bytes (tests/golden/io_writers.npz, made by oracle/make_golden.py io) and the
f-string restatement (oracle/io_oracle.py). Host-only: no GPU needed."""

import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle.io_oracle import field_csv_bytes, mask_csv_bytes
from paper_2605_04550_b200 import configs, core, io

GOLD = Path(__file__).resolve().parent / "golden"


def _field(grid, values):
    return core.SigmaField(grid, values)


def test_demo01_csv_byte_identical_to_shipped_golden(tmp_path):
    z = np.load(GOLD / "io_writers.npz")
    assert bool(z["demo01_matches_shipped"])
    vals = np.load(GOLD / "demo01_field.npz")["values"]
    g = configs.make_grid(-1.5, 1.5, -1.5, 1.5, 120, 120)
    p = tmp_path / "demo.csv"
    io.write_field_csv(p, _field(g, vals))
    assert hashlib.sha256(p.read_bytes()).hexdigest() == str(z["demo01_sha256"])


def test_special_values_match_reference_bytes(tmp_path):
    from oracle.make_golden import special_field_values
    z = np.load(GOLD / "io_writers.npz")
    g = configs.make_grid(-2.0, 7.5, -0.3, 1e-3, 7, 6)
    p = tmp_path / "s.csv"
    io.write_field_csv(p, _field(g, special_field_values()))
    assert p.read_bytes() == z["special_csv"].tobytes()


def test_mask_matches_reference_bytes(tmp_path):
    z = np.load(GOLD / "io_writers.npz")
    g = configs.make_grid(-1.0, 3.0, -3.5, 3.5, 11, 9)
    p = tmp_path / "m.csv"
    io.write_mask_csv(p, z["mask"], g)
    assert p.read_bytes() == z["mask_csv"].tobytes()


@pytest.mark.parametrize("nthreads", [1, 3, 0])
def test_random_bit_patterns_match_restatement(tmp_path, nthreads):
    rng = np.random.default_rng(17 + nthreads)
    ny, nx = 37, 23
    bits = rng.integers(0, 2**63, size=(ny, nx), dtype=np.uint64) | (rng.integers(0, 2, (ny, nx)).astype(np.uint64) << 63)
    vals = np.abs(bits.view(np.float64))  # every exponent, NaN payloads, inf, subnormals
    vals[0, :5] = [0.0, np.nan, -np.nan, np.inf, 1e-310]
    g = configs.make_grid(-1e-3, 2.5e7, -np.pi, np.e, nx, ny)
    p = tmp_path / "r.csv"
    io.write_field_csv(p, _field(g, vals), nthreads=nthreads)
    assert p.read_bytes() == field_csv_bytes(g.xs(), g.ys(), vals)
    m = rng.random((ny, nx)) < 0.5
    q = tmp_path / "rm.csv"
    io.write_mask_csv(q, m, g, nthreads=nthreads)
    assert q.read_bytes() == mask_csv_bytes(g.xs(), g.ys(), m)


def test_nan_field_and_large_grid_row_order(tmp_path):
    g = configs.make_grid(0.0, 1.0, 0.0, 1.0, 300, 70)  # > one 16-row block per thread
    vals = np.full(g.shape, np.nan)
    vals[::7, ::3] = np.linspace(1e-12, 10.0, vals[::7, ::3].size).reshape(vals[::7, ::3].shape)
    p = tmp_path / "n.csv"
    io.write_field_csv(p, _field(g, vals), nthreads=4)
    assert p.read_bytes() == field_csv_bytes(g.xs(), g.ys(), vals)


def test_writer_errors(tmp_path):
    g = configs.make_grid(0.0, 1.0, 0.0, 1.0, 4, 3)
    with pytest.raises(core.ParameterError):
        io.write_mask_csv(tmp_path / "x.csv", np.zeros((4, 3), bool), g)
    with pytest.raises(OSError):
        io.write_field_csv(tmp_path / "no_such_dir" / "x.csv", _field(g, np.ones(g.shape)))
