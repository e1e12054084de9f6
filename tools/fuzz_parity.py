"""Randomised parity sweep (development tool): random banded matrices of many shapes, sizes, scales
and structures (constant diagonals, noisy Toeplitz, general, real/complex, near-singular shifts)
against the oracle restatement (numpy zgesdd), floored gate 1e-9 relative at 1e-5 ||A||_2."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from oracle.sigma_oracle import floored_rel_err, smin_restated
from paper_2605_04550_b200 import core

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
big = len(sys.argv) > 3 and sys.argv[3] == 'big'  # include n = 1100 (the n >= 1000 engine split)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 150
worst, fails, t0 = 0.0, 0, time.time()
for t in range(N):
    n = int(rng.choice([2, 3, 5, 8, 17, 40, 90, 160, 300, 700] + ([1100] if big else [])))
    wide = rng.random() < 0.15  # runtime-shape kernels (bands beyond the exact-shape table)
    kmax = min(16, n - 1) if wide else min(5, n - 1)
    kl, ku = int(rng.integers(0, kmax + 1)), int(rng.integers(0, kmax + 1))
    cplx = rng.random() < 0.5
    kind = rng.choice(["toeplitz", "noisy", "general"])
    scale = 10.0 ** rng.uniform(-3, 6)
    c = rng.standard_normal(kl + ku + 1) + (1j * rng.standard_normal(kl + ku + 1) if cplx else 0)
    A = np.zeros((n, n), complex if cplx else float)
    for d in range(-kl, ku + 1):
        m = n - abs(d)
        if m <= 0:
            continue
        if kind == "general":
            v = rng.standard_normal(m) + (1j * rng.standard_normal(m) if cplx else 0)
        else:
            v = np.full(m, c[d + kl]) + (1e-3 * rng.standard_normal(m) if kind == "noisy" else 0)
        A += np.diag(v, d)
    A *= scale
    ev = np.linalg.eigvals(A)
    box = (ev.real.min() - 1, ev.real.max() + 1, ev.imag.min() - 1, ev.imag.max() + 1)
    zs = (rng.uniform(box[0], box[1], 24) + 1j * rng.uniform(box[2], box[3], 24))
    zs = np.concatenate([zs, ev[: min(4, n)] * (1 + 1e-9)])  # near-singular shifts
    got = core.smin_many(A, zs)
    want = smin_restated(A, zs)
    e = floored_rel_err(got, want, 1e-5 * np.linalg.norm(A, 2))
    worst = max(worst, float(e.max()))
    if e.max() > 1e-9:
        fails += 1
        i = int(np.argmax(e))
        print(f"FAIL t={t} n={n} kl={kl} ku={ku} cplx={cplx} kind={kind} scale={scale:.2e} z={zs[i]} got={got[i]:.6e} want={want[i]:.6e} err={e[i]:.2e}", flush=True)
print(f"fuzz: {N} matrices, worst floored rel err {worst:.2e}, failures {fails}, {time.time() - t0:.0f}s")
