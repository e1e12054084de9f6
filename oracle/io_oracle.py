"""ORACLE (test infrastructure only): restatement of the reference's CSV writers,
pseudospec/io.py:92-102 (write_field_csv) and io.py:105-115 (write_mask_csv) — one Python
f-string per grid point, row-major order. Pinned by tests/golden/io_writers.npz (the reference's
own output bytes, and the shipped demos/output_01_field.csv by sha256)."""

from __future__ import annotations

import numpy as np


def field_csv_bytes(xs, ys, values) -> bytes:
    with np.errstate(divide="ignore", invalid="ignore"):
        logs = np.log10(values)
    rows = ["x,y,log10_smin\n"]
    for i in range(len(ys)):
        for j in range(len(xs)):
            rows.append(f"{xs[j]:.17g},{ys[i]:.17g},{logs[i, j]:.17g}\n")
    return "".join(rows).encode()


def mask_csv_bytes(xs, ys, mask) -> bytes:
    mask = np.asarray(mask, dtype=bool)
    rows = ["x,y,flag\n"]
    for i in range(len(ys)):
        for j in range(len(xs)):
            rows.append(f"{xs[j]:.17g},{ys[i]:.17g},{int(mask[i, j])}\n")
    return "".join(rows).encode()
