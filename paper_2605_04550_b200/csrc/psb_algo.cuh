// psb_algo.cuh — per-point arithmetic of the sigma_min(zI - A) evaluator (K1).
//
// Replaces the per-z dense SVD of the reference
//   pseudospec/core.py:141-168  smin_many   (np.linalg.svd(zI - A)[-1], LAPACK zgesdd)
// by two exact-arithmetic engines that only touch the band of A:
//
//   engine L ("Lanczos"): pivoted band LU of M = zI - A (gbtrf-style, pivots within
//     the band, fill up to kl+ku superdiagonals), then inverse Lanczos on
//     (M^H M)^{-1} = M^{-1} M^{-H} (four banded triangular sweeps per step) with
//     the 3-term recurrence; sigma = 1/sqrt(theta_max). Used where sigma_min is
//     small relative to ||M|| (isolated, fast convergence: 2-12 steps measured).
//
//   engine B ("bisection"): sigma_min^2 is the smallest lambda at which
//     G(lambda) = A^H A - conj(z) A - z A^H + (|z|^2 - lambda) I   (= M^H M - lambda I)
//     stops being positive definite. A pivot-free banded LDL^H (stable on the PD
//     side, where every accepted test lives) decides each bisection step. All
//     z-independent bands are shared, so the state is a b x b register window
//     (b = kl+ku) and the engine is FP64-bound. Used where sigma_min >= tau*S,
//     S = |z| + ||A||_2 bound; there the rounding of G (~eps*S^2) costs at most
//     eps/tau^2 relative accuracy, and Toeplitz-like continua of singular values
//     (which stall Lanczos) do not slow bisection.
//
// Every function here is __host__ __device__, so the same arithmetic also compiles for the host
// (the runtime-shape and static-shape paths share it; only device code calls it in the product).
#pragma once
#include <stdint.h>
#include <math.h>
#ifdef __CUDACC__
#include <cuda_runtime.h>
#define PSB_HD __host__ __device__ __forceinline__
#else
#error "compile with nvcc"
#endif

namespace psb {

// ---------------------------------------------------------------- complex helpers
PSB_HD double2 cmk(double a, double b) { double2 r; r.x = a; r.y = b; return r; }
PSB_HD double2 czero() { return cmk(0.0, 0.0); }
PSB_HD double2 cconj(double2 a) { return cmk(a.x, -a.y); }
PSB_HD double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
PSB_HD double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
PSB_HD double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
PSB_HD double2 cmul(double2 a, double2 b) {
  return cmk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a - b*c   (the chained operand c enters last: depth 2 from c)
PSB_HD double2 cfms(double2 a, double2 b, double2 c) {
  return cmk(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}
// a - conj(b)*c
PSB_HD double2 cfms_cj(double2 a, double2 b, double2 c) {
  return cmk(fma(-b.x, c.x, fma(-b.y, c.y, a.x)), fma(-b.x, c.y, fma(b.y, c.x, a.y)));
}
// a - s*c with real s
PSB_HD double2 cfms_r(double2 a, double s, double2 c) { return cmk(fma(-s, c.x, a.x), fma(-s, c.y, a.y)); }
PSB_HD double cnorm2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
PSB_HD double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
// Re(conj(a) * b)
PSB_HD double cdotr(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }
// 1/d, scaled (Smith) so |d| near the overflow/underflow range stays finite
PSB_HD double2 crcp(double2 d) {
  if (fabs(d.x) >= fabs(d.y)) {
    double r = d.y / d.x, den = fma(d.y, r, d.x);
    double inv = 1.0 / den;
    return cmk(inv, -r * inv);
  } else {
    double r = d.x / d.y, den = fma(d.x, r, d.y);
    double inv = 1.0 / den;
    return cmk(r * inv, -inv);
  }
}

// 1/d = conj(d) / |d|^2 with a MUFU-seeded reciprocal (about 1 ulp) when |d|^2 is safely inside
// the normal range; Smith's scaled division otherwise.
// Reciprocal for the LDL^H pivots: MUFU seed r (relative error e = 1 - x r ~ 2^-23) refined in one
// cubic step, 1/x = r (1 + e + e^2) (1 - e^3)^-1: three dependent FMAs instead of two Newton steps' four,
// ~1 ulp either way (the PD decision only needs the sign of every pivot, and L = s / D is insensitive
// to an ulp in 1/D).
PSB_HD double fast_rcp(double x) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  const double t = fma(e, e, e);
  return fma(r, t, r);
#else
  return 1.0 / x;
#endif
}

PSB_HD double2 crcp_fast(double2 d) {
  const double m = fmax(fabs(d.x), fabs(d.y));
  if (m > 1e-150 && m < 1e150) {
    const double r = fast_rcp(fma(d.x, d.x, d.y * d.y));
    return cmk(d.x * r, -d.y * r);
  }
  return crcp(d);
}

// Lane view of a lane-interleaved array: element i lives at p[i * ld].
struct LV {
  double2* p;
  int ld;
  PSB_HD double2 get(int64_t i) const { return p[i * ld]; }
  PSB_HD void put(int64_t i, double2 v) const { p[i * ld] = v; }
};
struct LVb {
  int* p;
  int ld;
  PSB_HD int get(int64_t i) const { return p[i * ld]; }
  PSB_HD void put(int64_t i, int v) const { p[i * ld] = v; }
};

// Shape of the band problem. Band of A: Ab[(d + kl) * n + i] = A[i, i + d], d in [-kl, ku].
// Factors, stored per row so each triangular sweep streams only what it reads:
//   FU row j (NU = W + 1 complex): [U'(j, j+1..j+W) | rinv_j],  U' = rinv * U (row-scaled)
//   FL row j (NL = kl complex):    [L(j, j+1..j+kl)] (multipliers of elimination step j)
//   piv[j] in 0..kl: row swapped into position j at step j (int32)
// W = kl + ku is the upper bandwidth after partial-pivoting fill.
struct Shape {
  int n, kl, ku, W, NU, NL;
};
PSB_HD Shape make_shape(int n, int kl, int ku) {
  Shape s; s.n = n; s.kl = kl; s.ku = ku; s.W = kl + ku; s.NU = kl + ku + 1; s.NL = kl > 0 ? kl : 1; return s;
}

// ------------------------------------------------------------ engine L: band LU
// Pivoted LU of M = zI - A in a sliding register window of (kl+1) rows x (W+1)
// columns. Pivot rule: first max of |re|+|im| (LAPACK izamax/dcabs1 convention,
// as zgbtrf). Returns false on an exactly zero pivot (M singular in floating point).
struct NoRowHook {
  template <int N>
  PSB_HD bool operator()(int, const double2 (&)[N]) const { return true; }
};

// LU row loop unroll: 1 (measured against 2: C5 -2..4%, C2/C4 unchanged; half the code of the kernel's
// hottest loop, whose warps also walk four sweep loops per pass - ncu put 25% of engine L's stall samples
// on instruction fetch at 2)
#ifndef PSB_LU_UNROLL
#define PSB_LU_UNROLL 1
#endif
constexpr int kLuUnroll = PSB_LU_UNROLL;
// `hook(j, u)` sees each finished U row (u[0..W-1] = U', u[W] = rinv) in forward order, so a
// forward sweep that needs exactly these rows can run fused with the factorization. A hook that
// returns false ends the factorization there (lu_factor returns false, as for an exact zero pivot).
template <int KLM, int KUM, bool DYN, class RowHook = NoRowHook>
PSB_HD bool lu_factor(const Shape& s, const double2* __restrict__ Ab, double2 z, LV FU, LV FL, LVb piv,
                      RowHook hook = RowHook()) {
  constexpr int WM = KLM + KUM;
  const int n = s.n;
  const int kl = DYN ? s.kl : KLM;
  const int ku = DYN ? s.ku : KUM;
  const int W = kl + ku;
  const int NU = W + 1, NL = s.NL;
  double2 win[KLM + 1][WM + 1];
  bool ok = true;
  // initial rows r = 0..kl hold matrix rows r, columns 0..W
#pragma unroll
  for (int r = 0; r <= KLM; r++) {
#pragma unroll
    for (int c = 0; c <= WM; c++) {
      double2 v = czero();
      if (r <= kl && c <= W && r < n && c < n) {
        int d = c - r;
        if (d >= -kl && d <= ku) {
          double2 a = Ab[(int64_t)(d + kl) * n + r];
          v = cmk((d == 0 ? z.x : 0.0) - a.x, (d == 0 ? z.y : 0.0) - a.y);
        }
      }
      win[r][c] = v;
    }
  }
  double2 pre[WM + 1];
#pragma unroll
  for (int c = 0; c <= WM; c++) pre[c] = (c <= W && kl + 1 < n) ? Ab[(int64_t)c * n + kl + 1] : czero();
#pragma unroll kLuUnroll
  for (int j = 0; j < n; j++) {
    // pivot among rows j..j+kl (rows past n are zero and never win a strict '>')
    int p = 0;
    double best = cabs1(win[0][0]);
#pragma unroll
    for (int r = 1; r <= KLM; r++) {
      if (r <= kl) {
        double m = cabs1(win[r][0]);
        if (m > best) { best = m; p = r; }
      }
    }
#pragma unroll
    for (int r = 1; r <= KLM; r++) {
      if (r <= kl && p == r) {
#pragma unroll
        for (int c = 0; c <= WM; c++) {
          double2 t = win[0][c]; win[0][c] = win[r][c]; win[r][c] = t;
        }
      }
    }
    piv.put(j, p);
    double2 d = win[0][0];
    double2 ri;
    if (d.x == 0.0 && d.y == 0.0) { ok = false; ri = czero(); }
    else ri = crcp_fast(d);
    const int64_t rb = (int64_t)j * NU;
    double2 u[WM + 1];
#pragma unroll
    for (int c = 1; c <= WM; c++)
      if (c <= W) {
        u[c - 1] = cmul(win[0][c], ri);
        FU.put(rb + c - 1, u[c - 1]);
      }
    u[DYN ? WM : W] = ri;  // static shapes: u[W] = rinv (the hook is static-shape only)
    FU.put(rb + W, ri);
    if (!hook(j, u)) return false;
#pragma unroll
    for (int r = 1; r <= KLM; r++) {
      if (r <= kl) {
        double2 l = cmul(win[r][0], ri);
        FL.put((int64_t)j * NL + r - 1, l);
#pragma unroll
        for (int c = 1; c <= WM; c++)
          if (c <= W) win[r][c] = cfms(win[r][c], l, win[0][c]);
      }
    }
    // slide the window: row r <- row r+1 shifted one column left
#pragma unroll
    for (int r = 0; r < KLM; r++) {
      if (r < kl) {
#pragma unroll
        for (int c = 0; c < WM; c++)
          if (c < W) win[r][c] = win[r + 1][c + 1];
        win[r][W < WM ? W : WM] = czero();
      }
    }
    // new bottom row: matrix row i = j+1+kl, columns j+1 .. j+1+W (d = c - kl); its band
    // entries were loaded one row earlier (pre), and row i+1's are loaded now
    const int i = j + 1 + kl;
#pragma unroll
    for (int c = 0; c <= WM; c++) {
      if (c <= W) {
        double2 v = czero();
        int col = j + 1 + c;
        if (i < n && col < n) v = cmk((c == kl ? z.x : 0.0) - pre[c].x, (c == kl ? z.y : 0.0) - pre[c].y);
        win[kl][c] = v;
        pre[c] = (i + 1 < n) ? Ab[(int64_t)c * n + i + 1] : czero();
      }
    }
  }
  return ok;
}

// S1: forward sweep, t = U^{-H} r where r is the new Lanczos residual
//   r_k = w_{k-1} - c1 * RA - c2 * RB   (k >= 2), or the start vector v1 (k == 1).
// Writes RA <- r_k, RB <- old RA (fixed roles; no per-lane ping-pong), T <- U^{-H} r_k.
// U^H = U'^H D^H: solve with the unit lower U'^H, then scale by conj(rinv).
// Returns ||r_k||^2 (k >= 2).
template <int KLM, int KUM, bool DYN>
PSB_HD double sweep_s1(const Shape& s, LV F, LV T, LV RA, LV RB, const double2* __restrict__ v1,
                       int k, double c1, double c2) {
  constexpr int WM = KLM + KUM;
  const int n = s.n;
  const int W = DYN ? s.W : WM;
  const int NF = W + 1;  // F = FU
  double2 tw[WM + 1];  // tw[d] = t'_{j-d}
#pragma unroll
  for (int d = 0; d <= WM; d++) tw[d] = czero();
  double bsq = 0.0;
  for (int j = 0; j < n; j++) {
    double2 r;
    if (k == 1) {
      r = v1[j];
      RA.put(j, r);
    } else {
      double2 t = T.get(j), ra = RA.get(j);
      r = cfms_r(t, c1, ra);
      if (k >= 3) r = cfms_r(r, c2, RB.get(j));
      RB.put(j, ra);
      RA.put(j, r);
      bsq += cnorm2(r);
    }
    double2 tp = r;
#pragma unroll
    for (int d = WM; d >= 1; d--) {
      if (d <= W && j - d >= 0) tp = cfms_cj(tp, F.get((int64_t)(j - d) * NF + d - 1), tw[d]);
    }
    double2 ri = F.get((int64_t)j * NF + W);
    T.put(j, cmul(tp, cconj(ri)));
#pragma unroll
    for (int d = WM; d >= 2; d--) tw[d] = tw[d - 1];
    tw[1] = tp;
  }
  return bsq;
}

// S2: backward sweep, apply E^H (row swaps + unit-lower multipliers, transposed).
// Returns ||output||^2.
template <int KLM, int KUM, bool DYN>
PSB_HD double sweep_s2(const Shape& s, LV F, LVb piv, LV T) {  // F = FL
  const int n = s.n;
  const int kl = DYN ? s.kl : KLM;
  const int NL = s.NL;
  double2 yw[KLM + 1];  // yw[r] = y_{j+r}
#pragma unroll
  for (int r = 0; r <= KLM; r++) yw[r] = czero();
  double nrm = 0.0;
  for (int j = n - 1; j >= 0; j--) {
    const int out = j + 1 + kl;
    if (out < n) { T.put(out, yw[kl]); nrm += cnorm2(yw[kl]); }
#pragma unroll
    for (int r = KLM; r >= 1; r--) if (r <= kl) yw[r] = yw[r - 1];
    double2 y = T.get(j);
    const int64_t rb = (int64_t)j * NL - 1;
#pragma unroll
    for (int r = KLM; r >= 1; r--)
      if (r <= kl) y = cfms_cj(y, F.get(rb + r), yw[r]);
    yw[0] = y;
    const int p = piv.get(j);
#pragma unroll
    for (int r = 1; r <= KLM; r++) {
      if (r <= kl && p == r) { double2 t = yw[0]; yw[0] = yw[r]; yw[r] = t; }
    }
  }
#pragma unroll
  for (int r = 0; r <= KLM; r++)
    if (r <= kl && r < n) { T.put(r, yw[r]); nrm += cnorm2(yw[r]); }
  return nrm;
}

// S3: forward sweep, apply E (row swaps + eliminations) to scale * T, in place.
template <int KLM, int KUM, bool DYN>
PSB_HD void sweep_s3(const Shape& s, LV F, LVb piv, LV T, double scale) {  // F = FL
  const int n = s.n;
  const int kl = DYN ? s.kl : KLM;
  const int NL = s.NL;
  double2 bw[KLM + 1];  // bw[r] = b_{j+r}
#pragma unroll
  for (int r = 0; r <= KLM; r++) bw[r] = (r <= kl && r < n) ? cscale(T.get(r), scale) : czero();
  for (int j = 0; j < n; j++) {
    const int p = piv.get(j);
#pragma unroll
    for (int r = 1; r <= KLM; r++) {
      if (r <= kl && p == r) { double2 t = bw[0]; bw[0] = bw[r]; bw[r] = t; }
    }
    const int64_t rb = (int64_t)j * NL - 1;
#pragma unroll
    for (int r = 1; r <= KLM; r++)
      if (r <= kl) bw[r] = cfms(bw[r], F.get(rb + r), bw[0]);
    T.put(j, bw[0]);
#pragma unroll
    for (int r = 0; r < KLM; r++) if (r < kl) bw[r] = bw[r + 1];
    const int in = j + 1 + kl;
    bw[kl] = (in < n) ? cscale(T.get(in), scale) : czero();
  }
}

// S4: backward sweep, x = U^{-1} (scale * T) with U = D U' (x_j = b_j rinv_j - sum U'_{j,c} x_{j+c}),
// in place; returns sum_j Re(conj(RA_j) x_j) (the Lanczos alpha numerator).
template <int KLM, int KUM, bool DYN>
PSB_HD double sweep_s4(const Shape& s, LV F, LV T, LV RA, double scale, double* wn2) {  // F = FU
  constexpr int WM = KLM + KUM;
  const int n = s.n;
  const int W = DYN ? s.W : WM;
  const int NF = W + 1;
  double2 xw[WM + 1];  // xw[c] = x_{j+c}
#pragma unroll
  for (int c = 0; c <= WM; c++) xw[c] = czero();
  double acc = 0.0, nn = 0.0;
  for (int j = n - 1; j >= 0; j--) {
    const int64_t rb = (int64_t)j * NF;
    double2 x = cmul(cscale(T.get(j), scale), F.get(rb + W));
#pragma unroll
    for (int c = WM; c >= 1; c--)
      if (c <= W) x = cfms(x, F.get(rb + c - 1), xw[c]);
    T.put(j, x);
    acc += cdotr(RA.get(j), x);
    nn += cnorm2(x);
#pragma unroll
    for (int c = WM; c >= 2; c--) xw[c] = xw[c - 1];
    xw[1] = x;
  }
  *wn2 = nn;
  return acc;
}

// Largest eigenvalue of the Lanczos tridiagonal T_k (alpha = hist[i].x, beta = hist[i].y).
// Newton on det(T_k - x I) via the LDL^T pivot recurrence d_j(x), started from the interlacing
// bound x0 = top eigenvalue of [[theta_{k-1}, beta_{k-1} s_{k-1}], [., alpha_k]] (s_{k-1}: last
// component of T_{k-1}'s top Ritz vector), which lies between the two largest roots of T_k, so
// Newton converges to the largest one (quadratically once close; a near-double root from a
// ghost only slows it to linear). Guarded by the Weyl upper bound xu. Returns theta;
// *s2 = square of the last component of its eigenvector (= -1 / d_k'(theta)), used for the
// Ritz residual beta_k |s_k|.
PSB_HD double ritz_eval(const double2* hist, int ld, int k, double x, double* dp_out) {
  double d = hist[0].x - x, dp = -1.0;
  double q = 1.0 / d;
  double S = dp * q;
  int j = 1;
  for (; j + 3 < k; j += 4) {  // 4 independent history loads in flight
    const double2 h0 = hist[(int64_t)(j - 1) * ld], h1 = hist[(int64_t)j * ld];
    const double2 h2 = hist[(int64_t)(j + 1) * ld], h3 = hist[(int64_t)(j + 2) * ld];
    const double2 h4 = hist[(int64_t)(j + 3) * ld];
    const double a[4] = {h1.x, h2.x, h3.x, h4.x}, b[4] = {h0.y, h1.y, h2.y, h3.y};
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const double b2 = b[u] * b[u];
      const double dpn = fma(b2 * dp, q * q, -1.0);
      d = a[u] - x - b2 * q;
      q = 1.0 / d;
      dp = dpn;
      S = fma(dp, q, S);
    }
  }
  for (; j < k; j++) {
    const double bj = hist[(int64_t)(j - 1) * ld].y;
    const double b2 = bj * bj;
    const double dpn = fma(b2 * dp, q * q, -1.0);
    d = hist[(int64_t)j * ld].x - x - b2 * q;
    q = 1.0 / d;
    dp = dpn;
    S = fma(dp, q, S);
  }
  *dp_out = dp;
  return 1.0 / S;  // Newton step f/f'
}

PSB_HD double ritz_top(const double2* hist, int ld, int k, double theta_prev, double alpha, double beta,
                       double* s2) {
  // Upper bound: with f(x) = alpha - x + beta^2 sum_i s_i^2 / (x - theta_i) (secular function of
  // T_k over T_{k-1}'s Ritz pairs, sum s_i^2 = 1) and x - theta_i >= x - theta_1, f(x) <=
  // alpha - x + beta^2 / (x - theta_1), whose root is the top eigenvalue of
  // [[theta_1, beta], [beta, alpha]]; Newton from there decreases monotonically to theta_k.
  const double dm = 0.5 * (theta_prev - alpha);
  double x = (0.5 * (theta_prev + alpha) + sqrt(dm * dm + beta * beta)) * (1.0 + 1e-14) + 1e-300;
  double dp = -1.0;
  for (int it = 0; it < 200; it++) {
    const double step = ritz_eval(hist, ld, k, x, &dp);
    if (!(step > 1e-15 * x)) break;
    x -= step;
  }
  ritz_eval(hist, ld, k, x, &dp);
  *s2 = -1.0 / dp;
  return x;
}

// Convergence rule: stop when the Ritz residual r = beta_k |s_k| is below 1e-10 theta,
// or below 1e-8 theta with the Ritz value stationary to 1e-13.
// The stationary branch bounds the Ritz error by r^2 / gap <= 1e-16 theta^2 / gap, i.e. <= 1e-10 theta
// for gaps down to 1e-6 theta. (It was r <= 1e-6 theta with dtheta <= 1e-12 theta: a random diagonal
// band with a 4e-5 relative cluster at sigma_min stopped 8.5e-9 off, found by tools/fuzz_parity.py;
// the tighter rule costs +0.2..1.6% Lanczos steps on C2-C5.) r <= 1e-10 theta alone is not reachable
// everywhere: rounding floors the residual of some ill-conditioned shifts above it.
PSB_HD bool lanczos_converged(double theta, double dtheta, double r, double beta) {
  if (beta == 0.0) return true;
  return (r <= 1e-8 * theta && dtheta <= 1e-13 * theta) || r <= 1e-10 * theta;
}

// --------------------------------------------------------- engine B: PD test
// Is G(lam) = M^H M - lam I, M = zI - A, positive definite? G's band (b = kl + ku) is formed
// row by row from M's entries (g_entry); the diagonal shift is zz = -lam.
// Left-looking banded LDL^H; the previous b rows of L live in a ring of b register
// slots (row j in slot j mod b; the row loop is unrolled by b so every slot index is a
// compile-time constant). Virtual rows before 0 are L = 0, D = 1.
template <int KLM, int KUM>
struct PDRing {
  static constexpr int B = KLM + KUM;
  double2 L[B][B];  // L[slot][d-1] = L(row, row - d)
  double D[B], iD[B];
};

// M = zI - A from the band: M[k, k+e] = (e == 0 ? z : 0) - A[k, k+e], e in [-KL, KU].
PSB_HD double2 m_entry(const double2* __restrict__ Ab, int n, int kl, int k, int e, double2 z) {
  const double2 a = Ab[(int64_t)(kl + e) * n + k];
  return (e == 0) ? csub(z, a) : cmk(-a.x, -a.y);
}

// G[j, j-d] = (M^H M)[j, j-d] = sum_k conj(M[k, j]) M[k, j-d] over k in [j-KU, j-d+KL] (within [0, n)).
// Formed from M's own entries, so its rounding is relative to M's column norms (the scale T(z) of the
// engine split), not to (|z| + ||A||)^2 as the expansion A^H A - conj(z) A - z A^H + |z|^2 I would be.
template <int KLM, int KUM>
PSB_HD double2 g_entry(int n, int j, int d, const double2* __restrict__ Ab, double2 z) {
  double2 v = czero();
#pragma unroll
  for (int t = 0; t <= KLM + KUM - d; t++) {
    const int k = j - KUM + t;
    if (k < 0 || k >= n) continue;
    const double2 m1 = m_entry(Ab, n, KLM, k, KUM - t, z);      // M[k, j]
    const double2 m2 = m_entry(Ab, n, KLM, k, KUM - t - d, z);  // M[k, j-d]
    v = cfms_cj(v, cmk(-m1.x, -m1.y), m2);
  }
  return v;
}

// The same entry from the expansion G = A^H A - conj(z) A - z A^H + |z|^2 I (AHA[d * n + j] =
// (A^H A)[j, j-d], precomputed per matrix; the |z|^2 - lam diagonal term is the caller's zz), with rounding
// relative to (|z| + ||A||)^2: the form of the general-band kernels, whose engine split uses that scale.
// With z = x + iy, a = A[j, j-d], b = A[j-d, j]:  conj(z) a + z conj(b) = x P + y Q,
//   P = a + conj(b),  Q = i (conj(b) - a)   (z-independent; both real on the diagonal, a = b),
// so an entry is AHA_d - x P - y Q: two real-by-complex FMAs (4 DFMA) instead of two complex ones (8).
// g_pq forms (P, Q) exactly as psb_set_matrix packs them into the staged row table (BisRow): one rounding
// per component, the same on the host and the device, so both paths give the same bits.
PSB_HD void g_pq(double2 a, double2 b, double2* P, double2* Q) {
  *P = cmk(a.x + b.x, a.y - b.y);
  *Q = cmk(a.y + b.y, b.x - a.x);
}
PSB_HD double2 g_from_pq(double2 aha, double2 P, double2 Q, double2 z) {
  return cmk(fma(-z.y, Q.x, fma(-z.x, P.x, aha.x)), fma(-z.y, Q.y, fma(-z.x, P.y, aha.y)));
}
template <int KLM, int KUM>
PSB_HD double2 g_entry_aha(int n, int j, int d, const double2* __restrict__ Ab, const double2* __restrict__ AHA,
                           double2 z) {
  const double2 v = AHA[(int64_t)d * n + j];
  if (d > KLM && d > KUM) return v;
  const double2 a = (d <= KLM) ? Ab[(int64_t)(KLM - d) * n + j] : czero();        // A[j, j-d]
  const double2 b = (d <= KUM) ? Ab[(int64_t)(KLM + d) * n + (j - d)] : czero();  // A[j-d, j]
  double2 P, Q;
  g_pq(a, b, &P, &Q);
  return g_from_pq(v, P, Q, z);
}

// One row of the factorization for static shapes, for NP independent shifts lambda_q that share
// the off-diagonal G entries (only the diagonal depends on lambda). U = j mod B (compile-time).
template <int KLM, int KUM, int NP, int U>
PSB_HD void pd_row(PDRing<KLM, KUM> (&R)[NP], int n, int j, const double2* __restrict__ Ab,
                   double2 z, const double (&zz)[NP], bool (&pd)[NP]) {
  constexpr int B = KLM + KUM;
  double2 g[B + 1];
#pragma unroll
  for (int d = 0; d <= B; d++) g[d] = (j - d >= 0) ? g_entry<KLM, KUM>(n, j, d, Ab, z) : czero();
#pragma unroll
  for (int q = 0; q < NP; q++) {
    double2 Lj[B + 1], LD[B + 1];
#pragma unroll
    for (int d = B; d >= 1; d--) {
      const int sc = (U - d + 2 * B) % B;
      double2 sacc = g[d];
#pragma unroll
      for (int dm = B; dm > d; dm--) sacc = cfms_cj(sacc, R[q].L[sc][dm - d - 1], LD[dm]);
      Lj[d] = cscale(sacc, R[q].iD[sc]);
      LD[d] = cscale(Lj[d], R[q].D[sc]);
    }
    double dj = g[0].x + zz[q];
#pragma unroll
    for (int d = 1; d <= B; d++) dj -= cdotr(Lj[d], LD[d]);
#pragma unroll
    for (int d = 1; d <= B; d++) R[q].L[U][d - 1] = Lj[d];
    R[q].D[U] = dj;
    R[q].iD[U] = fast_rcp(dj);
    pd[q] = pd[q] && (dj > 0.0);
  }
}

template <int KLM, int KUM, int NP, int U>
struct PDUnroll {
  PSB_HD static void run(PDRing<KLM, KUM> (&R)[NP], int n, int jb, const double2* Ab, 
                         double2 z, const double (&zz)[NP], bool (&pd)[NP]) {
    if (jb + U < n) {
      pd_row<KLM, KUM, NP, U>(R, n, jb + U, Ab, z, zz, pd);
      PDUnroll<KLM, KUM, NP, U + 1>::run(R, n, jb, Ab, z, zz, pd);
    }
  }
};
template <int KLM, int KUM, int NP>
struct PDUnroll<KLM, KUM, NP, KLM + KUM> {
  PSB_HD static void run(PDRing<KLM, KUM> (&)[NP], int, int, const double2*, double2,
                         const double (&)[NP], bool (&)[NP]) {}
};

// Right-looking (outer-product) banded LDL^H with a sliding lower (b+1)x(b+1) window of the
// partially eliminated Schur complement: W[r][c] = entry (j+r, j+c), c <= r. Step j takes the pivot
// D_j = W[0][0], scales column 0 and updates the trailing window; the next pivot is
// D_{j+1} = W[1][1] - |W[1][0]|^2 / D_j, so the dependency chain per row is one reciprocal plus one
// FMA (the left-looking form chains through all b multipliers of the row). Same arithmetic test.
template <int KLM, int KUM>
struct PDWin {
  static constexpr int B = KLM + KUM;
  double2 W[B + 1][B + 1];
};

template <int KLM, int KUM, int NP, bool AHAF = false>
PSB_HD void pdw_load_row(PDWin<KLM, KUM> (&Wn)[NP], int r, int n, int i, const double2* __restrict__ Ab,
                         double2 z, const double (&zz)[NP], const double2* __restrict__ AHA = nullptr) {
  // row r of the window = matrix row i, columns i-r .. i (G entries G[i, i-d], d = r - c)
  constexpr int B = KLM + KUM;
  double2 g[B + 1];
#pragma unroll
  for (int d = 0; d <= B; d++) {
    g[d] = czero();
    if (d <= r && i < n && i - d >= 0)
      g[d] = AHAF ? g_entry_aha<KLM, KUM>(n, i, d, Ab, AHA, z) : g_entry<KLM, KUM>(n, i, d, Ab, z);
  }
#pragma unroll
  for (int q = 0; q < NP; q++) {
#pragma unroll
    for (int c = 0; c <= B; c++)
      if (c <= r) Wn[q].W[r][c] = g[r - c];
    Wn[q].W[r][r].x += (i < n) ? zz[q] : 1.0;  // rows past n: identity padding (PD-neutral)
    Wn[q].W[r][r].y = 0.0;
  }
}

// log det accumulator: det = mant * 2^expo, renormalised every 16 pivots (pivots of a PD test are
// positive; only PD probes' values are used).
struct LogDet {
  double mant;
  int expo;
  PSB_HD void init() { mant = 1.0; expo = 0; }
  // exponent renormalisation with integer ops only (the FP64 pipe is the engine's bottleneck);
  // a product that left the normal range (only possible for |entries| ~ 1e30+) poisons the value
  PSB_HD void norm() {
#ifdef __CUDA_ARCH__
    const long long b = __double_as_longlong(mant);
    const int e = (int)((b >> 52) & 0x7ff);
    if (e == 0 || e == 0x7ff) { mant = __longlong_as_double(0x7ff8000000000000ll); return; }
    expo += e - 1023;
    mant = __longlong_as_double((b & ~(0x7ffll << 52)) | (1023ll << 52));
#else
    int e;
    mant = frexp(mant, &e);
    expo += e;
#endif
  }
  PSB_HD double value() const { return log(mant) + 0.6931471805599453 * expo; }
  // log |det| (a failed probe's product carries the sign of its negative pivots)
  PSB_HD double absvalue() const { return log(fabs(mant)) + 0.6931471805599453 * expo; }
};

// Same as pdw_load_row with the G row entries given (rows of a diagonal-constant band share them).
template <int KLM, int KUM, int NP>
PSB_HD void pdw_load_row_g(PDWin<KLM, KUM> (&Wn)[NP], int r, const double2 (&g)[KLM + KUM + 1],
                           const double (&zz)[NP]) {
  constexpr int B = KLM + KUM;
#pragma unroll
  for (int q = 0; q < NP; q++) {
#pragma unroll
    for (int c = 0; c <= B; c++)
      if (c <= r) Wn[q].W[r][c] = g[r - c];
    Wn[q].W[r][r].x += zz[q];
    Wn[q].W[r][r].y = 0.0;
  }
}

// pos[q] counts the positive pivots of probe q: after all n rows, n - pos is the number of negative pivots,
// i.e. (Sylvester) the number of sigma_i^2 below the probe - a hint for placing the next probes of a failed
// round (k_bisect), never a decision: the PD answers alone move the bracket.
template <int KLM, int KUM, int NP, bool LD = true>
PSB_HD void pdw_step(PDWin<KLM, KUM> (&Wn)[NP], bool (&pd)[NP], LogDet (&ld)[NP], int (&pos)[NP]) {
  constexpr int B = KLM + KUM;
#pragma unroll
  for (int q = 0; q < NP; q++) {
    auto& W = Wn[q].W;
    const double dj = W[0][0].x;
    const bool positive = dj > 0.0;
    pd[q] = pd[q] && positive;
    pos[q] += positive ? 1 : 0;
    if (LD) ld[q].mant *= dj;
    const double iD = fast_rcp(dj);
    double2 l[B + 1];
#pragma unroll
    for (int r = 1; r <= B; r++) l[r] = cscale(W[r][0], iD);
    // next pivot first (critical path), then the rest of the trailing update
    W[1][1].x = fma(-l[1].x, W[1][0].x, fma(-l[1].y, W[1][0].y, W[1][1].x));
#pragma unroll
    for (int r = 2; r <= B; r++) {
#pragma unroll
      for (int c = 1; c < r; c++) W[r][c] = cfms(W[r][c], l[r], cconj(W[c][0]));
      W[r][r].x = fma(-l[r].x, W[r][0].x, fma(-l[r].y, W[r][0].y, W[r][r].x));
    }
#pragma unroll
    for (int r = 1; r <= B; r++)
#pragma unroll
      for (int c = 1; c <= r; c++) W[r - 1][c - 1] = W[r][c];
  }
}

// Whole PD test (right-looking) for NP shifts; `vote` lets device callers exit early.
template <int KLM, int KUM, int NP>
PSB_HD void pdw_test(int n, const double2* __restrict__ Ab, double2 z,
                     const double (&lam)[NP], bool (&pd)[NP]) {
  constexpr int B = KLM + KUM;
  PDWin<KLM, KUM> Wn[NP];
  double zz[NP];
#pragma unroll
  for (int q = 0; q < NP; q++) { zz[q] = -lam[q]; pd[q] = true; }
  LogDet ld[NP];
#pragma unroll
  for (int q = 0; q < NP; q++) ld[q].init();
#pragma unroll
  for (int r = 0; r <= B; r++) pdw_load_row<KLM, KUM, NP>(Wn, r, n, r, Ab, z, zz);
  int pos[NP];
#pragma unroll
  for (int q = 0; q < NP; q++) pos[q] = 0;
  for (int j = 0; j < n; j++) {
    pdw_step<KLM, KUM, NP>(Wn, pd, ld, pos);
    pdw_load_row<KLM, KUM, NP>(Wn, B, n, j + 1 + B, Ab, z, zz);
    if ((j & 15) == 15)
      for (int q = 0; q < NP; q++) ld[q].norm();
  }
}

template <int KLM, int KUM>
PSB_HD void pd_init(PDRing<KLM, KUM>& R) {
  constexpr int B = KLM + KUM;
#pragma unroll
  for (int s = 0; s < B; s++) {
#pragma unroll
    for (int d = 0; d < B; d++) R.L[s][d] = czero();
    R.D[s] = 1.0;
    R.iD[s] = 1.0;
  }
}

// Host/generic form: whole-test loop (device kernels drive the group loop themselves so
// they can vote on early exit).
template <int KLM, int KUM>
PSB_HD bool pd_test_static(int n, const double2* __restrict__ Ab, double2 z,
                           double lam) {
  constexpr int B = KLM + KUM;
  PDRing<KLM, KUM> R[1];
  pd_init(R[0]);
  const double zz[1] = {-lam};
  bool pd[1] = {true};
  for (int jb = 0; jb < n && pd[0]; jb += B) PDUnroll<KLM, KUM, 1, 0>::run(R, n, jb, Ab, z, zz, pd);
  return pd[0];
}

// Runtime-shape PD test (any kl, ku; ring in a caller-provided scratch of b*b complex + 2b doubles).
// (general-band form: G from the A^H A expansion, see g_entry_aha)
PSB_HD bool pd_test_dyn(int n, int kl, int ku, const double2* __restrict__ Ab, const double2* __restrict__ AHA,
                        double2 z, double lam, LV Lsc, double* Dsc, int dld) {
  const int b = kl + ku;
  const double zz = cnorm2(z) - lam;
  if (b == 0) {  // diagonal A
    for (int j = 0; j < n; j++) {
      double2 v = AHA[j];
      v = cfms_cj(v, z, Ab[j]);
      v = cfms(v, z, cconj(Ab[j]));
      if (!(v.x + zz > 0.0)) return false;
    }
    return true;
  }
  for (int s = 0; s < b; s++) {
    for (int d = 0; d < b; d++) Lsc.put((int64_t)s * b + d, czero());
    Dsc[(int64_t)(2 * s) * dld] = 1.0;
    Dsc[(int64_t)(2 * s + 1) * dld] = 1.0;
  }
  double2 Lj[33], LD[33];
  for (int j = 0; j < n; j++) {
    for (int d = b; d >= 1; d--) {
      const int c = j - d;
      double2 g = czero();
      if (c >= 0) {
        g = AHA[(int64_t)d * n + j];
        if (d <= kl) g = cfms_cj(g, z, Ab[(int64_t)(kl - d) * n + j]);
        if (d <= ku) g = cfms(g, z, cconj(Ab[(int64_t)(kl + d) * n + c]));
      }
      const int sc = ((c % b) + b) % b;
      double2 sacc = g;
      for (int dm = b; dm > d; dm--) sacc = cfms_cj(sacc, Lsc.get((int64_t)sc * b + dm - d - 1), LD[dm]);
      Lj[d] = cscale(sacc, Dsc[(int64_t)(2 * sc + 1) * dld]);
      LD[d] = cscale(Lj[d], Dsc[(int64_t)(2 * sc) * dld]);
    }
    double2 g0 = AHA[j];
    g0 = cfms_cj(g0, z, Ab[(int64_t)kl * n + j]);
    g0 = cfms(g0, z, cconj(Ab[(int64_t)kl * n + j]));
    double dj = g0.x + zz;
    for (int d = 1; d <= b; d++) dj -= cdotr(Lj[d], LD[d]);
    if (!(dj > 0.0)) return false;
    const int s0 = j % b;
    for (int d = 1; d <= b; d++) Lsc.put((int64_t)s0 * b + d - 1, Lj[d]);
    Dsc[(int64_t)(2 * s0) * dld] = dj;
    Dsc[(int64_t)(2 * s0 + 1) * dld] = 1.0 / dj;
  }
  return true;
}

// Multisection state machine of engine B (per point), NP probes per round.
//   phase 1: geometric search upward: probes lo*4^(i+1); the first failing probe closes the bracket
//   phase 2: probes lo + (hi-lo)(i+1)/(NP+1); keep the sub-interval between the last PD probe and
//            the first non-PD probe; stop when (hi - lo) <= rtol * hi; sigma = sqrt((lo + hi)/2)
// (The classification test at (tau S)^2 runs first, in its own pass, as phase 0.)
enum { BIS_CONTINUE = 0, BIS_DONE = 1, BIS_TO_LANCZOS = 2, BIS_FAIL = 3 };
struct MsState {
  double lo, hi;
  int phase, rounds;
};
template <int NP>
PSB_HD void ms_probes(const MsState& st, double (&lam)[NP]) {
#pragma unroll
  for (int i = 0; i < NP; i++) {
    if (st.phase == 1) {
      double f = 4.0;
      for (int t = 0; t < i; t++) f *= 4.0;
      lam[i] = st.lo * f;
    } else {
      lam[i] = st.lo + (st.hi - st.lo) * (double)(i + 1) / (double)(NP + 1);
    }
  }
}
// returns BIS_CONTINUE / BIS_DONE / BIS_FAIL
template <int NP>
PSB_HD int ms_update(MsState& st, const double (&lam)[NP], const bool (&pd)[NP], double rtol, int max_rounds) {
  st.rounds++;
  if (st.phase == 1) {
    int first_fail = -1;
#pragma unroll
    for (int i = NP - 1; i >= 0; i--)
      if (!pd[i]) first_fail = i;
    if (first_fail < 0) {
      st.lo = lam[NP - 1];
      return st.rounds > max_rounds ? BIS_FAIL : BIS_CONTINUE;
    }
    st.hi = lam[first_fail];
    if (first_fail > 0) st.lo = lam[first_fail - 1];
    st.phase = 2;
  } else {
    double lo = st.lo, hi = st.hi;
#pragma unroll
    for (int i = 0; i < NP; i++) {
      if (pd[i]) lo = fmax(lo, lam[i]);
      else hi = fmin(hi, lam[i]);
    }
    if (lo >= hi) {  // non-monotone answers: the decision is at the rounding level here
      const double m = 0.5 * (st.lo + st.hi);
      st.lo = st.hi = m;
      return BIS_DONE;
    }
    st.lo = lo;
    st.hi = hi;
  }
  if (st.hi - st.lo <= rtol * st.hi) return BIS_DONE;
  return st.rounds > max_rounds ? BIS_FAIL : BIS_CONTINUE;
}
PSB_HD double ms_sigma(const MsState& st) { return sqrt(0.5 * (st.lo + st.hi)); }

}  // namespace psb
