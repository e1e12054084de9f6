"""K1 parity on the GPU (-m gpu): σ_min from libpsb200.so against the reference's zgesdd fixtures.

Gate: |σ - σ_ref| <= 1e-9 * max(σ_ref, 1e-5 ||A||_2); ε-masks identical
except where |σ_ref - ε| is inside that band; plus the reference's own test forms
(tests/test_core.py:96-152, tests/test_acceptance.py:53-85,145-157 of the reference).
"""

import numpy as np
import pytest

from oracle.sigma_oracle import floored_rel_err
from paper_2605_04550_b200 import _lib, configs, core

pytestmark = pytest.mark.gpu
TOL = 1e-9


def check(got, want, norm2, what):
    floor = 1e-5 * norm2
    e = floored_rel_err(got, want, floor)
    assert np.all(np.isfinite(got)), what
    assert e.max() <= TOL, f"{what}: worst floored rel err {e.max():.3e} at {int(np.argmax(e))}"
    return e.max()


def masks_agree(got, want, norm2, eps_levels):
    band = TOL * np.maximum(want, 1e-5 * norm2)
    for eps in eps_levels:
        m_got, m_want = got <= eps, want <= eps
        diff = m_got != m_want
        assert not np.any(diff & (np.abs(want - eps) > band)), f"mask mismatch at eps={eps}"


def test_c1_full_grid_and_eps_masks(gpu, gold):
    z = gold("c1_full.npz")
    cfg = configs.CONFIGS["C1"]
    fld = core.full_pseudospectrum(cfg.matrix(), cfg.grid)
    check(fld.values, z["values"], float(z["norm2"]), "C1")
    masks_agree(fld.values, z["values"], float(z["norm2"]), [10.0 ** -k for k in range(1, 9)])
    st = core.last_stats()
    assert st["n_lanczos"] > 0 and st["n_bisect"] > 0 and st["n_lanczos"] + st["n_bisect"] == 2500


def test_demo01_golden_including_exact_zeros(gpu, gold):
    """demos/output_01_field.csv: nilpotent shift n=32, 120x120; 85 points with σ_ref = 0."""
    want = gold("demo01_field.npz")["values"]
    A = np.diag(np.ones(31), k=-1)
    fld = core.full_pseudospectrum(A, core.make_grid(-1.5, 1.5, -1.5, 1.5, 120, 120))
    check(fld.values, want, 1.0, "demo01")
    masks_agree(fld.values, want, 1.0, [1e-2, 1e-4, 1e-8])


@pytest.mark.parametrize("name", ["c2_sample", "c3_sample", "c4_sample", "c3_wide", "c4_wide"])
def test_config_samples(gpu, gold, name):
    """Seeded grid subsets; *_wide are SURVEY 8(c)'s sizes (C3 1,024 points, C4 256)."""
    z = gold(f"{name}.npz")
    cfg = configs.CONFIGS[name.split("_")[0].upper()]
    got, it, st = core.smin_many(cfg.matrix(), z["zs"], return_info=True)
    check(got, z["sigma"], float(z["norm2"]), name)
    # the points themselves and their engines: batch-invariant (same bits in a different order)
    perm = np.random.default_rng(0).permutation(got.size)
    assert np.array_equal(core.smin_many(cfg.matrix(), z["zs"][perm]), got[perm])


def test_c5_sample(gpu, gold):
    z = gold("c5_sample.npz")
    cfg = configs.CONFIGS["C5"]
    for r, m in enumerate(z["matrices"]):
        got = core.smin_many(cfg.matrix(int(m)), z["zs"][r])
        check(got, z["sigma"][r], float(z["norm2"][r]), f"C5[{m}]")


def test_c5_stratified(gpu, gold):
    """C5 pinned on meaningful points (oracle/make_golden.py gen_c5_strat): 4 of the 64 matrices x 64 grid
    shifts chosen from full C5 maps by what they exercise - general-band bisection points above the parity
    floor, points straddling the engine split, points within 20% of an eps level, Lanczos points above
    the floor - each against the restated zgesdd. Every engine must be pinned on many of them."""
    z = gold("c5_strat.npz")
    cfg = configs.CONFIGS["C5"]
    worst, above, by_engine = 0.0, 0, {0: 0, 1: 0}
    for r, m in enumerate(z["matrices"]):
        A = cfg.matrix(int(m))
        want = z["sigma"][r]
        n2 = float(z["norm2"][r])
        got, it, st = core.smin_many(A, z["zs"][r], return_info=True)
        worst = max(worst, check(got, want, n2, f"C5 strat[{m}]"))
        live = want >= 1e-5 * n2
        above += int(live.sum())
        for e in (0, 1):
            by_engine[e] += int((live & (st == e)).sum())
        masks_agree(got, want, n2, [1e-1, 1e-2, 1e-3])
    print(f"\n[parity] C5 stratified: {above} points above the floor (engine L {by_engine[0]}, engine B "
          f"{by_engine[1]}), worst floored rel err {worst:.3g} (gate {TOL})")
    assert above >= 64 * len(z["matrices"]) - 8
    assert by_engine[1] >= 64 and by_engine[0] >= 32


def test_small_random_reference_acceptance_form(gpu, gold):
    """tests/test_acceptance.py:53-70: |got - want| / max(1, want) < 1e-10 over random banded A."""
    z = gold("small_random.npz")
    worst = 0.0
    for t in range(len(z["A"])):
        n = int(z["n"][t])
        got = core.smin_many(z["A"][t][:n, :n], z["zs"][t])
        worst = max(worst, float(np.max(np.abs(got - z["sigma"][t]) / np.maximum(1.0, z["sigma"][t]))))
    assert worst < 1e-10


def test_normality_identity(gpu):
    """tests/test_acceptance.py:73-85: symmetric A -> σ_min = dist(z, spectrum) within 1e-8."""
    rng = np.random.default_rng(20)
    zs = core.make_grid(-3, 3, -3, 3, 10, 10).points().ravel()
    worst = 0.0
    for _ in range(5):
        M = rng.standard_normal((12, 12))
        A = (M + M.T) / 2
        lam = np.linalg.eigvalsh(A)
        d = np.abs(zs[:, None] - lam[None, :]).min(axis=1)
        worst = max(worst, float(np.abs(core.smin_many(A, zs) - d).max()))
    assert worst < 1e-8


def test_identity_and_singular_shift(gpu):
    g = core.make_grid(0, 2, -1, 1, 3, 3)
    fld = core.full_pseudospectrum(np.eye(2), g)
    assert np.allclose(fld.values, np.abs(g.points() - 1.0), atol=1e-12)
    assert core.smin_at(np.diag(np.ones(3), -1), 0.0) == pytest.approx(0.0, abs=1e-15)
    assert core.smin_at(np.eye(2), 3.0) == pytest.approx(2.0, abs=1e-12)


def test_shift_covariance(gpu):
    A = configs.grcar_band(40).todense().real
    for c in (0.7, -1.3, 2.0):
        z = 0.4 + 0.9j
        assert abs(core.smin_at(A + c * np.eye(40), z + c) - core.smin_at(A, z)) < 1e-10


def test_restricted_equals_full_bitwise(gpu):
    cfg = configs.CONFIGS["C1"]
    A = cfg.matrix()
    full = core.full_pseudospectrum(A, cfg.grid)
    rng = np.random.default_rng(5)
    region = rng.uniform(size=cfg.grid.shape) < 0.2
    res = core.restricted_field(A, cfg.grid, region)
    assert np.array_equal(res.values[region], full.values[region])
    assert np.all(np.isnan(res.values[~region]))
    empty = core.restricted_field(A, cfg.grid, np.zeros(cfg.grid.shape, bool))
    assert np.all(np.isnan(empty.values))


def test_batch_order_and_pointwise_invariance_bitwise(gpu):
    """Values depend only on (A, z): pointwise == batched, any order, any batch, any call."""
    A = configs.CONFIGS["C2"].matrix()
    zs = configs.CONFIGS["C2"].grid.points().ravel()[::97]
    base = core.smin_many(A, zs)
    perm = np.random.default_rng(1).permutation(zs.size)
    assert np.array_equal(core.smin_many(A, zs[perm]), base[perm])
    assert np.array_equal(core.smin_many(A, zs), base)
    for i in range(0, zs.size, 50):
        assert core.smin_at(A, zs[i]) == base[i]
    parts = np.concatenate([core.smin_many(A, zs[i:i + 37]) for i in range(0, zs.size, 37)])
    assert np.array_equal(parts, base)


def test_engines_agree_where_both_apply(gpu):
    """Forcing all points through either engine gives the same σ (points with σ >= tau*S)."""
    A = configs.CONFIGS["C1"].matrix()
    zs = configs.CONFIGS["C1"].grid.points().ravel()
    auto, _, st = core.smin_many(A, zs, return_info=True)
    sel = zs[st == 1][:300]
    lan = core.smin_many(A, sel, opts=_lib.make_opts(force_engine=1))
    bis = core.smin_many(A, sel, opts=_lib.make_opts(force_engine=2))
    assert np.max(np.abs(lan - bis) / bis) < 1e-10


def test_c2_full_grid_properties(gpu):
    """Full-size (40,000-point) checks: all converged; σ is 1-Lipschitz in z; bounded by ||zI-A||."""
    cfg = configs.CONFIGS["C2"]
    A = cfg.matrix()
    vals, iters, st = core.smin_many(A, cfg.grid.points().ravel(), return_info=True)
    assert np.all(st <= 2)
    v = vals.reshape(cfg.grid.shape)
    dx = cfg.grid.xs()[1] - cfg.grid.xs()[0]
    dy = cfg.grid.ys()[1] - cfg.grid.ys()[0]
    assert np.all(np.abs(np.diff(v, axis=1)) <= dx * (1 + 1e-9) + 1e-12)
    assert np.all(np.abs(np.diff(v, axis=0)) <= dy * (1 + 1e-9) + 1e-12)
    assert np.all(v >= 0) and np.all(v <= np.abs(cfg.grid.points()) + 4.0)


def test_edge_cases(gpu):
    assert core.smin_many(np.eye(3), np.zeros(0, complex)).shape == (0,)
    assert core.smin_at(np.array([[0.0, 1.0], [0.0, 0.0]]), 0.0) == 0.0
    dense16 = np.random.default_rng(3).standard_normal((16, 16))  # kl = ku = 15 (runtime-shape kernels)
    zs = np.array([0.3 + 0.1j, -2 + 1j, 5j])
    from oracle.sigma_oracle import smin_restated
    check(core.smin_many(dense16, zs), smin_restated(dense16, zs), np.linalg.norm(dense16, 2), "dense16")
    diag = np.diag(np.arange(1.0, 6.0))  # kl = ku = 0
    assert np.allclose(core.smin_many(diag, [2.5 + 0j, 10j]),
                       [0.5, np.abs(10j - np.arange(1, 6)).min()], rtol=1e-12)


def test_no_state_leaks_between_calls(gpu):
    """Scratch buffers are reused across calls: a forced-engine call, another matrix, or a smaller batch
    must not change the next call's bits (regression: a stale per-point marker once did)."""
    A = configs.CONFIGS["C1"].matrix()
    zs = configs.CONFIGS["C1"].grid.points().ravel()
    base, _, st = core.smin_many(A, zs, return_info=True)
    core.smin_many(A, zs[st == 1], opts=_lib.make_opts(force_engine=2))
    core.smin_many(configs.CONFIGS["C4"].matrix(), configs.CONFIGS["C4"].grid.points().ravel()[:64])
    core.smin_many(A, zs[:7], opts=_lib.make_opts(force_engine=1))
    assert np.array_equal(core.smin_many(A, zs), base)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_bisection_near_threshold_full_grid(gpu, name):
    """Engine B against engine L on every point of a full grid that a low split (tau = 5e-4) moves
    to bisection. Engine L is accurate there (fixtures <= 1e-11); engine B's squared-form error is
    c eps / (2 r^2) at r = sigma / T(z) with c <= 1.5 measured, i.e. <= 3.3e-10 at
    r = tau. Regression: a secant probe inside the rounding band of sigma^2 once ended the
    multisection at the midpoint of the still-wide bracket (errors up to 2e-6 at such points)."""
    cfg = configs.CONFIGS[name]
    A = cfg.matrix()
    zs = cfg.grid.points().ravel()
    ref, _, st0 = core.smin_many(A, zs, opts=_lib.make_opts(tau=1e-2), return_info=True)
    got, _, st = core.smin_many(A, zs, opts=_lib.make_opts(tau=5e-4), return_info=True)
    moved = (st0 == 0) & (st == 1)
    assert moved.sum() > 100
    e = np.abs(got[moved] - ref[moved]) / ref[moved]
    assert e.max() <= 1e-9, f"{name}: worst {e.max():.3e}"


def test_launch_shapes_are_bitwise_neutral(gpu, tmp_path):
    """Launch shape and lane scheduling must not change a single bit (every sigma is a function of (A, z)).
    C5's full 1024x1024 grid of matrix 0 (about 300k bisection points, 740k engine-L points) takes the long
    general-band path: engine L on a third of the SMs with its step iterations deferred until 16 lanes hold
    a factored point, engine B as one full-occupancy launch. The knobs (read at handle creation, so each run
    is a subprocess) switch that back to engine L on every SM with undeferred steps and the two-launch
    engine B (second launch queued behind engine L), and to one launch without the expansion."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); from paper_2605_04550_b200 import configs, core; "
            "c = configs.CONFIGS['C5']; np.save(sys.argv[1], core.smin_many(c.matrix(0), c.grid.points().ravel()))")
    knobs = ("PSB_NOBEXP", "PSB_BFULL", "PSB_DEFER", "PSB_LFRAC")
    outs = []
    for env_extra, name in (({}, "product.npy"), ({"PSB_BFULL": "0", "PSB_DEFER": "0"}, "two.npy"),
                            ({"PSB_BFULL": "0", "PSB_NOBEXP": "1", "PSB_DEFER": "8"}, "one.npy")):
        env = {k: v for k, v in os.environ.items() if k not in knobs}
        env.update(env_extra)
        path = tmp_path / name
        subprocess.run([sys.executable, "-c", code, str(path)], check=True, env=env,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


def test_general_band_long_list_shapes_and_parity(gpu, tmp_path):
    """A mid-size noisy (2,2) band (general-band kernels, runtime knobs as above) on a 400x400 grid: enough
    bisection points for the long-list launch shape (engine L on a third of the SMs plus its queued second
    launch, engine B as one launch, step deferral). The map must equal the one computed with those shapes
    switched off, bit for bit, and a seeded sample of it must match zgesdd."""
    import os
    import subprocess
    import sys
    from oracle.sigma_oracle import smin_restated
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); from paper_2605_04550_b200 import core\n"
        "rng = np.random.default_rng(5); n = 300\n"
        "c = rng.standard_normal(5) + 1j * rng.standard_normal(5)\n"
        "A = sum(np.diag(np.full(n - abs(d), c[d + 2]) + 1e-3 * (rng.standard_normal(n - abs(d)) + 1j * "
        "rng.standard_normal(n - abs(d))), d) for d in range(-2, 3))\n"
        "r = np.abs(c).sum(); g = core.make_grid(-1.2 * r, 1.2 * r, -1.2 * r, 1.2 * r, 400, 400)\n"
        "f = core.full_pseudospectrum(A, g); st = core.last_stats()\n"
        "np.savez(sys.argv[1], A=A, zs=g.points().ravel(), v=f.values.ravel(), nb=st['n_bisect'], nl=st['n_lanczos'])\n")
    knobs = ("PSB_NOBEXP", "PSB_BFULL", "PSB_DEFER", "PSB_LFRAC")
    outs = []
    for env_extra, name in (({}, "product.npz"), ({"PSB_BFULL": "0", "PSB_DEFER": "0"}, "plain.npz")):
        env = {k: v for k, v in os.environ.items() if k not in knobs}
        env.update(env_extra)
        path = tmp_path / name
        subprocess.run([sys.executable, "-c", code, str(path)], check=True, env=env,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
        outs.append(np.load(path))
    a, b = outs
    assert int(a["nb"]) >= 256 * 148 and int(a["nl"]) > 0, (int(a["nb"]), int(a["nl"]))
    assert np.array_equal(a["v"], b["v"])
    idx = np.random.default_rng(9).choice(a["v"].size, 48, replace=False)
    worst = check(a["v"][idx], smin_restated(a["A"], a["zs"][idx]), np.linalg.norm(a["A"], 2), "general long list")
    print(f"[general long list] nB {int(a['nb'])}, nL {int(a['nl'])}, worst floored rel err {worst:.2e}")


def test_partly_constant_band_long_boundary(gpu):
    """A band that is diagonal-constant only over its second half: the constant interior is long
    enough to detect but its boundary (60 rows) exceeds the per-thread slot budget, so the general
    kernels run. Against the oracle at points on both sides of the engine split."""
    from oracle.sigma_oracle import smin_restated
    A = configs.grcar_band(120).todense().real.copy()
    rng = np.random.default_rng(11)
    for i in range(60):
        for j in range(max(0, i - 1), min(120, i + 4)):
            A[i, j] += 0.3 * rng.standard_normal()
    zs = np.concatenate([core.make_grid(-1, 3, -3.5, 3.5, 6, 6).points().ravel(), [0.5 + 1.2j, 2.9 + 0.1j]])
    check(core.smin_many(A, zs), smin_restated(A, zs), np.linalg.norm(A, 2), "partly constant band")


@pytest.mark.parametrize("offdiag", [0.0, 1e-6])
def test_clustered_small_sigma_lanczos_fallback(gpu, offdiag):
    """A tight cluster at sigma_min below the engine split: a diagonal (runtime-shape kernels) or
    nearly diagonal tridiagonal band with entries 734.5 + 0.31 N(0,1), shifted next to the cluster.
    Inverse Lanczos stagnates (regression: the old stop rule ended 8.5e-9 off, found by
    tools/fuzz_parity.py); points that hit kmax are retried on engine B where the squared form is
    accurate. sigma = min_j |z - a_jj| for the diagonal case."""
    from oracle.sigma_oracle import smin_restated
    rng = np.random.default_rng(4)
    n = 160
    a = 734.5 + 0.31 * rng.standard_normal(n)
    A = np.diag(a) + offdiag * (np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))
    zs = np.array([734.5318694864126 - 0.7180989702498619j, a[7] + 0.5j, a[3] - 0.9j, 734.0 + 0.3j])
    got = core.smin_many(A, zs)
    want = smin_restated(A, zs)
    if offdiag == 0.0:
        assert np.allclose(want, np.abs(zs[:, None] - a[None, :]).min(axis=1), rtol=1e-12)
    check(got, want, np.linalg.norm(A, 2), f"clustered, offdiag={offdiag}")


@pytest.mark.parametrize("scale", [1e-200, 1e200])
def test_extreme_matrix_scales(gpu, scale):
    """Matrices far from unit scale run on an exactly power-of-two-rescaled problem: the squared forms
    (G = M^H M, (M^H M)^-1) overflowed from |A| ~ 1e154 (every sigma came back 0 at 1e200)."""
    from oracle.sigma_oracle import smin_restated
    A = configs.grcar_band(60).todense().real * scale
    zs = core.make_grid(-1, 3, -3.5, 3.5, 7, 7).points().ravel() * scale
    got, _, st = core.smin_many(A, zs, return_info=True)
    assert np.all(st <= 1)
    check(got, smin_restated(A, zs), np.linalg.norm(A, 2), f"scale {scale:g}")


def test_randomised_band_sweep(gpu):
    """A small slice of tools/fuzz_parity.py in the suite: random bands of many shapes (exact-shape and
    runtime-shape kernels), structures (constant diagonals, noisy Toeplitz, general), real/complex,
    scales 1e-3..1e6, with shifts next to eigenvalues, against zgesdd (floored gate)."""
    from oracle.sigma_oracle import smin_restated
    rng = np.random.default_rng(2026)
    for t in range(40):
        n = int(rng.choice([2, 3, 5, 8, 17, 40, 90, 160]))
        kmax = min(16 if t % 7 == 0 else 5, n - 1)
        kl, ku = int(rng.integers(0, kmax + 1)), int(rng.integers(0, kmax + 1))
        cplx = bool(rng.random() < 0.5)
        kind = ("toeplitz", "noisy", "general")[t % 3]
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
        A *= 10.0 ** rng.uniform(-3, 6)
        ev = np.linalg.eigvals(A)
        zs = (rng.uniform(ev.real.min() - 1, ev.real.max() + 1, 12)
              + 1j * rng.uniform(ev.imag.min() - 1, ev.imag.max() + 1, 12))
        zs = np.concatenate([zs, ev[: min(3, n)] * (1 + 1e-9)])
        check(core.smin_many(A, zs), smin_restated(A, zs), np.linalg.norm(A, 2), f"sweep case {t} n={n} ({kl},{ku}) {kind}")


@pytest.mark.parametrize("kl,ku", [(3, 3), (1, 3), (2, 1)])
def test_general_band_rows_every_remainder(gpu, kl, ku):
    """General-band bisection kernels (noisy bands: no diagonal-constant interior): G rows come from the
    staged row table in the form AHA - Re(z) P - Im(z) Q in 8-row blocks, from the band itself for the first
    kl + ku + 1 rows and for the n mod 8 rows after the last block, and rows past n are zero-filled stage
    rows. Every remainder n mod 8 and sizes below one block, bisection forced on every point (shifts well
    outside the spectrum, where the squared form is accurate), against zgesdd."""
    from oracle.sigma_oracle import smin_restated
    rng = np.random.default_rng(7 * kl + ku)
    worst = 0.0
    for n in (7, 9, 15, 16, 17, 64, 66, 67, 68, 69, 70, 71, 133):
        c = (rng.standard_normal(kl + ku + 1) + 1j * rng.standard_normal(kl + ku + 1))
        A = np.zeros((n, n), complex)
        for d in range(-kl, ku + 1):
            m = n - abs(d)
            A += np.diag(np.full(m, c[d + kl]) + 1e-3 * (rng.standard_normal(m) + 1j * rng.standard_normal(m)), d)
        r = np.abs(c).sum()
        ang = rng.uniform(0, 2 * np.pi, 10)
        zs = (1.3 + rng.uniform(0, 1.0, 10)) * r * np.exp(1j * ang)
        got, it, st = core.smin_many(A, zs, opts=_lib.make_opts(force_engine=2), return_info=True)
        assert (st == 1).all(), (n, st)
        worst = max(worst, check(got, smin_restated(A, zs), np.linalg.norm(A, 2), f"general ({kl},{ku}) n={n}"))
        assert np.array_equal(got, core.smin_many(A, zs, opts=_lib.make_opts(force_engine=2)))
    print(f"[general-band rows ({kl},{ku})] worst floored rel err {worst:.2e}")


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_engine_b_variants_bitwise_equal(gpu, tmp_path, name):
    """The wide (NP = 2) and pair (NP = 1, G = 2) bisection variants probe the same shifts with the same
    arithmetic, so the host's per-launch choice between them must not change a bit (PSB_BVARIANT,
    read at handle creation: 1 wide, 2 pair). C1 (short list, pair by default) and C3 (long list)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); from paper_2605_04550_b200 import configs, core; "
            f"c = configs.CONFIGS['{name}']; z = c.grid.points().ravel()[::3]; "
            "np.save(sys.argv[1], core.smin_many(c.matrix(), z))")
    outs = []
    for v in ("1", "2"):
        env = {**os.environ, "PSB_BVARIANT": v}
        path = tmp_path / f"v{v}.npy"
        subprocess.run([sys.executable, "-c", code, str(path)], check=True, env=env,
                       cwd=str(Path(__file__).resolve().parents[1]))
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name,count", [("C2", 24), ("C3", 8)])
def test_singularity_certificate_points_are_below_the_floor(gpu, name, count):
    """Engine L decides a point as singular to working precision (σ = 0, status 2) once it has proven
    σ_min <= 1e-16 max_j ||A e_j|| (the LU prefix ||U^{-H} v1|| and nu = ||M^{-H} v1||
    certificates). At every such point the reference's zgesdd must lie under the parity floor
    1e-5 ||A||_2 * 1e-9 - in fact under 1e-15 ||A||_2 (its own rounding level), checked on a seeded sample
    of the decided points of the full grid."""
    from oracle.sigma_oracle import smin_restated
    cfg = configs.CONFIGS[name]
    A = cfg.matrix()
    Ad = A.todense() if hasattr(A, "todense") else np.asarray(A)
    zs = cfg.grid.points().ravel()
    vals, iters, st = core.smin_many(A, zs, return_info=True)
    dec = np.flatnonzero((st == 2) & (vals == 0.0))
    assert dec.size > 0
    pick = np.random.default_rng(5).choice(dec, min(count, dec.size), replace=False)
    ref = smin_restated(Ad, zs[pick])
    norm2 = np.linalg.norm(Ad, 2)
    check(vals[pick], ref, norm2, f"{name} certified points")
    assert ref.max() <= 1e-15 * norm2, f"{name}: certified point with reference sigma {ref.max():.3e}"
    print(f"{name}: {dec.size} certified points; sample max reference sigma {ref.max() / norm2:.2e} ||A||_2")


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_engine_split_counts_match_the_pipeline(gpu, name):
    """psb_engine_split (the batch scheduler's cost estimate) runs the same classification test as a sweep:
    its counts equal the sweep's engine counts on the same points."""
    cfg = configs.CONFIGS[name]
    A = cfg.matrix(0)
    zs = cfg.grid.points()[::7, ::5].ravel()
    nb, nl = core.engine_split(A, zs)
    core.smin_many(A, zs)
    st = core.last_stats()
    assert (nb, nl) == (st["n_bisect"], st["n_lanczos"]) and nb + nl == zs.size
    assert core.engine_split(A, zs[:0]) == (0, 0)
