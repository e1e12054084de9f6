// psb_engines.cuh — the two persistent K1 kernels (sm_100a).
//
// Both kernels are warp-persistent: each warp owns 32 lanes = 32 independent grid points
// and pulls new points from a global atomic counter (core.py:186-195 sharded row blocks over
// a process pool; here the unit is a point and the balance is dynamic because per-point
// work varies 2..50+ steps). Results are placed by point index, so they are independent of
// scheduling (core.py:181-182).
#pragma once
#include "psb_algo.cuh"

namespace psb {

struct BisArgs {
  int n, kl, ku;
  const double2* __restrict__ Ab;
  const double2* __restrict__ AHA;  // (A^H A)[j, j-d] band: G rows of the general-band kernels
  const double2* __restrict__ zs;
  const int64_t* __restrict__ outidx;  // nullable: output index of point p
  int64_t P;
  double tau, rtol;
  double zscale, sscale;          // exact power-of-two scaling: engines see z * zscale, report sigma * sscale
  const double* __restrict__ offmin;  // min(off-diagonal column, row norm^2) per index j (upper bound)
  double anorm;                   // general-band kernels: split scale S(z) = |z| + sqrt(||A||_1 ||A||_inf)
  double2 dc;                     // TZ kernels: engine-split scale T(z)^2 = (|z - dc| + dr)^2 + offsq >= max_j ||M e_j||^2
  double dr, offsq;               //   (dc, dr: disc holding A's diagonal; offsq: max off-diagonal column norm^2)
  int force, max_tests;
  double* out;
  int32_t* iters;
  int8_t* status;
  int64_t* listA;                 // points handed to the Lanczos engine
  int64_t* listB;                 // points the bisection engine owns (mode 1 input)
  unsigned long long* counters;   // [0] work, [1] nA, [2] pd tests, [3] nB done, [7] nB listed
  int mode;                       // 0: classify (one test, split into listA/listB); 1: bisect listB
  int fallback;                   // 1: listB holds engine-L points that did not converge (forced, [0, lambda_tau]);
  double rmin2;                   //    their result is kept only where sigma^2 >= rmin2 X(z)^2 (squared form accurate)
  int secant;                     // 1: secant-accelerated multisection (G == 1, NP == 2 shapes)
  int counts;                     // 1: count-guided probe placement (negative-pivot counts of failed probes)
  int cnt_min;                    //    least count of the lower failure
  double cnt_slack;               //    probes at the estimate -/+ (hi - estimate) * cnt_slack / count
  double itp_frac0;               //    chord step: first half-width as a fraction of the bracket
  int tz_j0, tz_j1;               // rows [tz_j0, tz_j1] share one G row (diagonal-constant band); j0 > j1: none
  double2* gb;                    // TZ kernels: per-thread G rows formed once per point, lane-interleaved
                                  //   (stride gb_T threads): slots [0, nb) the boundary rows, slot nb the interior row
  int nb;
  int64_t gb_T;
  int64_t tid_base;               // first thread index of this launch (engine B runs as one or two launches)
  double2* dyn_L;                 // DYN only: per-thread b*b ring
  double* dyn_D;                  // DYN only: per-thread 2b
  unsigned long long* rowctr;     // nullable: += LDL^H rows x probes executed for points (roofline accounting)
  const double2* __restrict__ RT; // general-band kernels: z-independent G-row coefficients, row-packed
                                  //   (BisRow<KL,KU>::RW complex per row), staged per warp in shared memory
};

// Row-packed coefficient table of the general-band G rows (psb_set_matrix): row i holds
//   [AHA_d = (A^H A)[i, i-d], d = 0..B | (P_0, Q_0) (both real) | P_d, Q_d, d = 1..D],  D = max(KL, KU),
// with P_d = a + conj(b), Q_d = i (conj(b) - a), a = A[i, i-d], b = A[i-d, i] (g_pq, psb_algo.cuh), so
// G[i, i-d] = AHA_d - Re(z) P_d - Im(z) Q_d (g_entry_aha) reads one contiguous span.
template <int KL, int KU>
struct BisRow {
  static constexpr int B = KL + KU;
  static constexpr int D = KL > KU ? KL : KU;
  static constexpr int RW = B + 2 * D + 2;  // complex per row
  static constexpr int RB = 8;          // rows per stage (one unrolled block of the row loop)
  static constexpr int SE = RB * RW;    // complex per stage
  static constexpr int BYTES = 2 * SE * 16;  // two stages per warp
};

struct LanArgs {
  Shape s;
  const double2* __restrict__ Ab;
  const double2* __restrict__ v1;
  const double2* __restrict__ v1b;  // v1 once (n entries): warp-uniform loads in the fused LU + S1
  const double2* __restrict__ LUT;  // static shapes: the staged LU's row stream (LUS, psb_set_matrix)
  const double2* __restrict__ zs;
  const int64_t* __restrict__ outidx;
  const int64_t* __restrict__ listA;
  unsigned long long* counters;   // [1] nA (read), [4] work, [5] lanczos steps, [6] nL, [8] n not converged,
                                  // [20] LU rows factored (roofline accounting: the LU of a decided point stops early)
  double zscale, sscale;          // exact power-of-two scaling (see BisArgs)
  int64_t* listF;                 // not-converged points (as ~p: forced bisection entries), counters[8] of them
  double* out;
  int32_t* iters;
  int8_t* status;
  double2* scratch;               // per warp: FU n*NU*32 | FL n*NL*32 | T | RA | RB (n*32 each) | hist kmax*32
  int* pivs;                      // per warp: n*32 int32
  int64_t warp_stride, piv_stride;
  int64_t warp_base;              // first warp index of this launch (engine L may run as two launches)
  int kmax, refill;
  int defer;                      // step iterations wait for this many factored lanes while points remain (0: never)
  unsigned long long* prof;       // optional: per-phase clock64 totals [lu, s1, s2, s3, s4, ritz, idle]
  // Certificates of singularity to working precision (psb_set_matrix; INFINITY disables them): the point
  // is decided as sigma = 0 (status 2) once sigma_min <= delta ||A e_j||_max <= delta ||A||_2 is proven,
  // from the fused LU's prefix ||t[0..j]||^2 > tcert (t = U^{-H} v1) or from nu^2 = ||M^{-H} v1||^2 > ncert.
  double tcert, ncert;
};

// ---------------------------------------------------------------- cp.async row ring
// Each lane streams only its own column (its own grid point), so a lane's cp.async groups
// and waits are private: no warp barrier, no cross-lane hazard. Row j of a sweep lives in
// ring slot (sweep step) % D; the copy for step q+D-1 is issued before waiting for step q.
__device__ __forceinline__ void cp16(void* s, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
// zero-filling variant: copies `bytes` (0 or 16) and fills the rest of the 16 with zeros
__device__ __forceinline__ void cp16z(void* s, const void* g, unsigned bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp4(void* s, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int KL, int KU, int D>
struct Ring {
  static constexpr int W = KL + KU, NU = W + 1, NL = (KL > 0 ? KL : 1), SF = W + 4;
  static constexpr int BYTES = D * SF * 32 * 16 + D * 32 * 4;  // per warp
  double2* d;  // this warp's ring
  int* pv;     // pivot ring
  int lane;
  __device__ double2* at(int slot, int f) const { return d + ((slot * SF + f) << 5) + lane; }
  __device__ int* pat(int slot) const { return pv + (slot << 5) + lane; }
};

// S1 (forward): r_k update and t = U^{-H} r_k, right-looking so row j's U' entries are consumed
// at step j (the ring holds current/future rows only). Slot j: FU_j | T_j RA_j RB_j.
// RA holds r_{k-1}, RB r_{k-2}; r_k is written over RB and the caller swaps the two roles.
template <int KL, int KU, int D>
__device__ double pl_s1(int n, const Ring<KL, KU, D>& R, LV FU, LV T, LV RA, LV RB,
                        const double2* __restrict__ v1, int k, double c1, double c2) {
  typedef Ring<KL, KU, D> RG;
  constexpr int W = RG::W, NU = RG::NU;
  // Branch-free in k (lanes of a warp sit at different k): X is v1 (k == 1) or T, and the RA / RB
  // slots are zero-filled where the recurrence does not use them, so r = X - c1 RA - c2 RB with
  // c1 = c2 = 0 at k == 1 and c2 = 0 at k == 2 reproduces the three cases bit for bit.
  const double2* xsrc = (k == 1) ? v1 + R.lane : T.p;  // start vector: lane-replicated copy
  const unsigned za = (k >= 2) ? 16u : 0u, zb = (k >= 3) ? 16u : 0u;
  auto issue = [&](int j, int sl) {  // caller guarantees j < n
#pragma unroll
    for (int f = 0; f < NU; f++) cp16(R.at(sl, f), FU.p + ((int64_t)j * NU + f) * 32);
    cp16(R.at(sl, NU), xsrc + (int64_t)j * 32);
    cp16z(R.at(sl, NU + 1), RA.p + (int64_t)j * 32, za);
    cp16z(R.at(sl, NU + 2), RB.p + (int64_t)j * 32, zb);
    cp_commit();
  };
  double2 acc[W + 1];
#pragma unroll
  for (int d = 0; d <= W; d++) acc[d] = czero();
  double bsq = 0.0;
  auto body = [&](int j, int sl) {
    const double2 r = cfms_r(cfms_r(*R.at(sl, NU), c1, *R.at(sl, NU + 1)), c2, *R.at(sl, NU + 2));
    RB.put(j, r);  // r_k overwrites r_{k-2} (row j already consumed); the caller swaps RA / RB
    bsq += cnorm2(r);  // used for k >= 2 only
    const double2 tp = cadd(r, acc[0]);
    T.put(j, cmul(tp, cconj(*R.at(sl, W))));
#pragma unroll
    for (int d = 1; d <= W; d++) acc[d - 1] = cfms_cj(acc[d], *R.at(sl, d - 1), tp);
    acc[W] = czero();
  };
  // prologue D-1 rows; steady state issues row j+D-1 unconditionally; the last D-1 rows drain
#pragma unroll
  for (int q = 0; q < D - 1; q++)
    if (q < n) issue(q, q);
  // steady state in blocks of D rows, so every ring slot index is a compile-time constant
  int j = 0;
  for (; j + D <= n - (D - 1); j += D) {
#pragma unroll
    for (int u = 0; u < D; u++) {
      issue(j + u + D - 1, (u + D - 1) % D);
      cp_wait<D - 1>();
      body(j + u, u);
    }
  }
  for (; j < n - (D - 1); j++) {
    issue(j + D - 1, (j + D - 1) % D);
    cp_wait<D - 1>();
    body(j, j % D);
  }
  cp_wait<0>();
  for (; j < n; j++) body(j, j % D);
  return bsq;
}

// S2 (backward): E^H. Slot (step q, row j = n-1-q): FL_j | T_j, piv_j. Returns ||out||^2.
template <int KL, int KU, int D>
__device__ double pl_s2(int n, const Ring<KL, KU, D>& R, LV FL, LVb piv, LV T) {
  typedef Ring<KL, KU, D> RG;
  constexpr int NL = RG::NL;
  auto issue = [&](int q, int sl) {  // caller guarantees q < n
    const int j = n - 1 - q;
#pragma unroll
    for (int f = 0; f < KL; f++) cp16(R.at(sl, f), FL.p + ((int64_t)j * NL + f) * 32);
    cp16(R.at(sl, NL), T.p + (int64_t)j * 32);
    cp4(R.pat(sl), piv.p + (int64_t)j * 32);
    cp_commit();
  };
  double2 yw[KL + 1];
#pragma unroll
  for (int r = 0; r <= KL; r++) yw[r] = czero();
  double nrm = 0.0;
  auto body = [&](int q, int sl) {
    const int j = n - 1 - q;
    const int out = j + 1 + KL;
    if (out < n) { T.put(out, yw[KL]); nrm += cnorm2(yw[KL]); }
#pragma unroll
    for (int r = KL; r >= 1; r--) yw[r] = yw[r - 1];
    double2 y = *R.at(sl, NL);
#pragma unroll
    for (int r = KL; r >= 1; r--) y = cfms_cj(y, *R.at(sl, r - 1), yw[r]);
    yw[0] = y;
    const int p = *R.pat(sl);
#pragma unroll
    for (int r = 1; r <= KL; r++)
      if (p == r) { const double2 t = yw[0]; yw[0] = yw[r]; yw[r] = t; }
  };
#pragma unroll
  for (int q = 0; q < D - 1; q++)
    if (q < n) issue(q, q);
  // steady state in blocks of D rows, so every ring slot index is a compile-time constant
  int q = 0;
  for (; q + D <= n - (D - 1); q += D) {
#pragma unroll
    for (int u = 0; u < D; u++) {
      issue(q + u + D - 1, (u + D - 1) % D);
      cp_wait<D - 1>();
      body(q + u, u);
    }
  }
  for (; q < n - (D - 1); q++) {
    issue(q + D - 1, (q + D - 1) % D);
    cp_wait<D - 1>();
    body(q, q % D);
  }
  cp_wait<0>();
  for (; q < n; q++) body(q, q % D);
#pragma unroll
  for (int r = 0; r <= KL; r++)
    if (r < n) { T.put(r, yw[r]); nrm += cnorm2(yw[r]); }
  return nrm;
}

// S3 (forward): E applied to scale*T in place. Slot j: FL_j | T_{j+1+KL}, piv_j.
template <int KL, int KU, int D>
__device__ void pl_s3(int n, const Ring<KL, KU, D>& R, LV FL, LVb piv, LV T, double scale) {
  typedef Ring<KL, KU, D> RG;
  constexpr int NL = RG::NL;
  auto issue = [&](int j, int sl) {  // caller guarantees j < n; T row j+1+KL exists except for the last KL+1
#pragma unroll
    for (int f = 0; f < KL; f++) cp16(R.at(sl, f), FL.p + ((int64_t)j * NL + f) * 32);
    const bool t_in = j + 1 + KL < n;
    cp16z(R.at(sl, NL), T.p + (int64_t)(t_in ? j + 1 + KL : j) * 32, t_in ? 16u : 0u);
    cp4(R.pat(sl), piv.p + (int64_t)j * 32);
    cp_commit();
  };
  double2 bw[KL + 1];
#pragma unroll
  for (int r = 0; r <= KL; r++) bw[r] = (r < n) ? cscale(T.get(r), scale) : czero();
  auto body = [&](int j, int sl) {
    const int p = *R.pat(sl);
#pragma unroll
    for (int r = 1; r <= KL; r++)
      if (p == r) { const double2 t = bw[0]; bw[0] = bw[r]; bw[r] = t; }
#pragma unroll
    for (int r = 1; r <= KL; r++) bw[r] = cfms(bw[r], *R.at(sl, r - 1), bw[0]);
    T.put(j, bw[0]);
#pragma unroll
    for (int r = 0; r < KL; r++) bw[r] = bw[r + 1];
    bw[KL] = cscale(*R.at(sl, NL), scale);  // zero-filled past the end
  };
#pragma unroll
  for (int q = 0; q < D - 1; q++)
    if (q < n) issue(q, q);
  // steady state in blocks of D rows, so every ring slot index is a compile-time constant
  int j = 0;
  for (; j + D <= n - (D - 1); j += D) {
#pragma unroll
    for (int u = 0; u < D; u++) {
      issue(j + u + D - 1, (u + D - 1) % D);
      cp_wait<D - 1>();
      body(j + u, u);
    }
  }
  for (; j < n - (D - 1); j++) {
    issue(j + D - 1, (j + D - 1) % D);
    cp_wait<D - 1>();
    body(j, j % D);
  }
  cp_wait<0>();
  for (; j < n; j++) body(j, j % D);
}

// S4 (backward): x = U^{-1}(scale*T) in place; returns sum Re(conj(RA_j) x_j).
// Slot (step q, row j = n-1-q): FU_j | T_j RA_j.
template <int KL, int KU, int D>
__device__ double pl_s4(int n, const Ring<KL, KU, D>& R, LV FU, LV T, LV RA, double scale, double* wn2) {
  typedef Ring<KL, KU, D> RG;
  constexpr int W = RG::W, NU = RG::NU;
  auto issue = [&](int q, int sl) {  // caller guarantees q < n
    const int j = n - 1 - q;
#pragma unroll
    for (int f = 0; f < NU; f++) cp16(R.at(sl, f), FU.p + ((int64_t)j * NU + f) * 32);
    cp16(R.at(sl, NU), T.p + (int64_t)j * 32);
    cp16(R.at(sl, NU + 1), RA.p + (int64_t)j * 32);
    cp_commit();
  };
  double2 xw[W + 1];
#pragma unroll
  for (int c = 0; c <= W; c++) xw[c] = czero();
  double acc = 0.0, nn = 0.0;
  auto body = [&](int q, int sl) {
    const int j = n - 1 - q;
    double2 x = cmul(cscale(*R.at(sl, NU), scale), *R.at(sl, W));
#pragma unroll
    for (int c = W; c >= 1; c--) x = cfms(x, *R.at(sl, c - 1), xw[c]);
    T.put(j, x);
    acc += cdotr(*R.at(sl, NU + 1), x);
    nn += cnorm2(x);
#pragma unroll
    for (int c = W; c >= 2; c--) xw[c] = xw[c - 1];
    xw[1] = x;
  };
#pragma unroll
  for (int q = 0; q < D - 1; q++)
    if (q < n) issue(q, q);
  // steady state in blocks of D rows, so every ring slot index is a compile-time constant
  int q = 0;
  for (; q + D <= n - (D - 1); q += D) {
#pragma unroll
    for (int u = 0; u < D; u++) {
      issue(q + u + D - 1, (u + D - 1) % D);
      cp_wait<D - 1>();
      body(q + u, u);
    }
  }
  for (; q < n - (D - 1); q++) {
    issue(q + D - 1, (q + D - 1) % D);
    cp_wait<D - 1>();
    body(q, q % D);
  }
  cp_wait<0>();
  for (; q < n; q++) body(q, q % D);
  *wn2 = nn;
  return acc;
}

// cp.async ring depth (rows in flight + 1): 16 for tridiagonal bands, 8 otherwise, 4 for (3,3). Measured on
// B200: C4 (1,1) 425 -> 400 ms at 16 (end of round 2, where shallower rings would fit two blocks per SM:
// 81.6 ms at 16, 84.8 / 89.7 / 103.8 ms at 8 / 6 / 4 - the kernel is HBM-bound, more warps do not help); C2 (1,3) 3.26 -> 3.45 ms at 13, so wider bands keep 8 (at 4: C2
// 2.3 -> 2.4, C3 14.9 -> 15.1 ms). (3,3) (C5, whose engine-L points are mostly LU-bound) at 4: the
// per-warp ring drops from 42 to 21 KB, so two engine-L blocks fit an SM: C5 matrices 0/1/17/63
// 813/326/709/452 -> 747/302/615/411 ms (depth 3: within 1%).
#ifndef PSB_D33
#define PSB_D33 4
#endif
#ifndef PSB_DW
#define PSB_DW 8
#endif
#ifndef PSB_D11
#define PSB_D11 16
#endif
template <int KL, int KU>
struct RingDepth {
  static constexpr int D = (KL + KU <= 2) ? PSB_D11 : (KL == 3 && KU == 3 ? PSB_D33 : PSB_DW);
};

__device__ __forceinline__ int64_t out_index(const int64_t* outidx, int64_t p) { return outidx ? outidx[p] : p; }

// ----------------------------------------------------------------- engine B kernel
// mode 0 (NP = G = 1): classification — one LDL^H test per point at lambda = (tau X(z))^2; PD points
//   go to listB (sigma >= tau X), the rest to listA (Lanczos engine).
// mode 1: multisection of the listB points. A group of G lanes owns one point and every lane runs NP
//   independent LDL^H chains (sharing the G-row formation), so a round tests K = G*NP shifts: search
//   rounds probe upward (or geometrically inside [lo, U^2]), then the bracket [lo, hi] is cut at
//   lo + (hi-lo)(i+1)/(K+1) or at the secant probes (K = 2). The group keeps [max PD probe, min non-PD
//   probe] (shuffle reductions). Probe i = gl*NP + q is the same shift for (NP, G) = (2, 1) and (1, 2),
//   so those two variants return the same bits and the host may launch either; every sigma is a pure
//   function of (A, z).
// TZ: the band has a diagonal-constant interior (a.tz_j0 <= a.tz_j1) whose G rows are formed once per
// point; the general-band row loop is a separate instantiation so each gets its own register budget.
template <int KL, int KU, bool DYN, int NP, int G, bool TZ>
__global__ void __launch_bounds__(128) k_bisect(BisArgs a) {
  constexpr int B = KL + KU;
  constexpr int K = NP * G;
  constexpr bool SEC = (NP * G == 2);  // secant acceleration: two probes per round (one lane x 2, or 2 lanes x 1)
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;               // lane within the group
  const int leader = lane - gl;          // group leader lane
  const int64_t tid = a.tid_base + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t p = -1;
  double2 z = czero();
  double lo = 0.0, hi = 0.0;
  int phase = 1, rounds = 0;
  double x2 = 0.0;  // X(z)^2 of the lane's point
  // secant acceleration state (G == 1): log det at lo and at the previous PD point lp
  double Llo = 0.0, lp = 0.0, Lp = 0.0;
  bool have_lo = false, have_p = false, use_sec = false;
  // the two lowest failed probes that carry a negative-pivot count (fa < fb; counts ca <= cb)
  double fa = INFINITY, fb = INFINITY;
  int ca = 0, cb = 0;
  bool use_cnt = true;
  // log |det| at hi when exactly one sigma_i^2 lies below it (the root is isolated: det changes sign once)
  double Lhi = 0.0, ifrac = a.itp_frac0;
  bool have_hi = false, use_itp = true;
  bool exhausted = false;
  const int64_t total = (a.mode == 0) ? a.P : (int64_t)a.counters[7];
  while (true) {
    const unsigned idle = __ballot_sync(FULL, p < 0 && gl == 0);  // idle groups (leader bits)
    if (idle && !exhausted) {
      const int cnt = __popc(idle);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)cnt);
      base = __shfl_sync(FULL, base, 0);
      const int rank = __popc(idle & ((1u << leader) - 1u));
      const bool grp_idle = (idle >> leader) & 1u;
      if (grp_idle) {
        const int64_t q = (int64_t)base + rank;
        if (q < total) {
          const int64_t entry = (a.mode == 0) ? q : a.listB[q];
          const bool forced = entry < 0;          // forced bisection of a point that failed classification
          const int64_t pt = forced ? ~entry : entry;
          z = cscale(a.zs[pt], a.zscale);
          // split at sigma = tau T(z): engine B's squared-form error is c eps T^2 / (2 sigma^2) relative
          // (c <= 0.6 measured), so sigma >= tau T keeps it below ~1e-10
          double lam_tau;
          if constexpr (TZ && !DYN) {  // (x2 = X(z)^2 = lam_tau / tau^2, kept for the fallback check)  // G formed from M's entries: rounding relative to T(z)^2
            const double dz = hypot(z.x - a.dc.x, z.y - a.dc.y) + a.dr;
            lam_tau = a.tau * a.tau * (dz * dz + a.offsq);
          } else {  // G from the A^H A expansion: rounding relative to S(z)^2 = (|z| + ||A||)^2
            const double sz = hypot(z.x, z.y) + a.anorm;
            lam_tau = a.tau * a.tau * sz * sz;
          }
          if (a.mode == 0 && a.force == 1) {  // Lanczos-only mode: hand over immediately
            if (gl == 0) {
              unsigned long long slot = atomicAdd(&a.counters[1], 1ull);
              a.listA[slot] = pt;
            }
          } else {
            p = pt;
            rounds = 0;
            x2 = lam_tau / (a.tau * a.tau);
            if constexpr (TZ && !DYN) {
              // G rows of this point that are not the shared interior row: rows [0, tz_j0) and
              // (tz_j1, n), then the interior row itself. They depend on z only, so every test of the
              // point reads them instead of re-forming them (keeps the row loops' registers low).
              constexpr int B = KL + KU;
              for (int sl = 0; sl <= a.nb; sl++) {
                const int i = (sl == a.nb) ? a.tz_j0 : (sl < a.tz_j0 ? sl : a.tz_j1 + 1 + (sl - a.tz_j0));
#pragma unroll
                for (int d = 0; d <= B; d++)
                  a.gb[((int64_t)sl * (B + 1) + d) * a.gb_T + tid] = (i - d >= 0) ? g_entry<KL, KU>(a.n, i, d, a.Ab, z) : czero();
              }
            }
            lo = lam_tau; hi = INFINITY; phase = 1;
            if (a.mode == 1 && !forced) {
              // upper bound sigma_min^2 <= min_j min(||M e_j||^2, ||e_j^T M||^2): the search then
              // closes the bracket geometrically from both ends (far points no longer climb from lo)
              double u2 = INFINITY;
              for (int j = 0; j < a.n; j++) {
                const double2 m = csub(z, a.Ab[(int64_t)a.kl * a.n + j]);
                u2 = fmin(u2, cnorm2(m) + a.offmin[j]);
              }
              u2 *= 1.0 + 1e-12;
              if (u2 > lo) hi = u2;
            }
            have_lo = have_p = use_sec = false;
            fa = fb = INFINITY; ca = cb = 0; use_cnt = true;
            have_hi = false; use_itp = true; ifrac = a.itp_frac0;
            if (a.mode == 1 && forced) { lo = 0.0; hi = lam_tau; phase = 2; }
          }
        }
      }
      if ((int64_t)base + cnt >= total) exhausted = true;
    }
    const unsigned act = __ballot_sync(FULL, p >= 0);
    if (!act) {
      if (exhausted) break;
      continue;
    }
    const bool me = p >= 0;
    double lam[NP];
#pragma unroll
    for (int q = 0; q < NP; q++) {
      const int i = gl * NP + q;
      if (a.mode == 0) lam[q] = lo;
      else if (phase == 1) lam[q] = (hi == INFINITY) ? lo * exp2(2.0 * (i + 1))
                                                      : lo * exp2(log2(hi / lo) * (double)(i + 1) / (double)(K + 1));
      else lam[q] = lo + (hi - lo) * (double)(i + 1) / (double)(K + 1);
      if (!me) lam[q] = 1.0;
    }
    // Secant step (G == 1, NP == 2): det G(lambda) = prod (sigma_i^2 - lambda) is positive, decreasing
    // and convex below sigma_min^2, so the secant through two PD points (lp, lo) has its root ls below
    // sigma_min^2 (a valid lower bound). Probe ls and ls + (ls - lo)/10; the PD tests alone decide
    // the bracket, so a poor secant costs time, never correctness.
#ifdef PSB_ROUND_STATS
    int rtype = (phase == 1) ? 0 : 1;  // 0 search, 1 section, 2 secant, 3 count, 4 chord
#endif
    if constexpr (SEC) {
      if (a.mode == 1 && me && phase == 2 && use_sec && have_lo && have_p && a.secant) {
        const double dL = Lp - Llo;  // log(f(lp) / f(lo)) > 0 (NaN if a product overflowed)
        if (dL > 1e-300 && dL < 700.0) {
          const double ls = lo + (lo - lp) / expm1(dL);
          if (ls > lo && ls < hi) {
            double p1 = ls + 0.1 * (ls - lo);
            if (!(p1 < hi)) p1 = 0.5 * (ls + hi);
#pragma unroll
            for (int q = 0; q < NP; q++) lam[q] = (gl * NP + q == 0) ? ls : p1;  // probe 0: ls, probe 1: p1
#ifdef PSB_ROUND_STATS
            rtype = 2;
#endif
          }
        }
      }
    }
    // Count-guided step: a failed probe's LDL^H has as many negative pivots as there are sigma_i^2 below it.
    // Near the bottom edge of a banded spectrum the count grows like N(lambda)^2 ~ (lambda - sigma_1^2) / kappa
    // (sigma_k^2 ~ sigma_1^2 + kappa (k^2 - 1)), so the two lowest counted failures (fa, ca), (fb, cb) give
    // the estimate s = (fa - r fb) / (1 - r), r = ((ca + 1/2)^2 - 1) / ((cb + 1/2)^2 - 1). While the bracket
    // still holds several singular values (ca >= cnt_min = 2) a three-section round buys 1.58 bits, the
    // estimate several; the round probes s -/+ the estimate's slack (hi - s) cnt_slack / ca. Measured (B200,
    // tests per bisection point / kernel ms): C5 matrix 0 41.3 / 425 without, 35.6 / 381 with (cnt_min 2,
    // slack 2; cnt_min 3: 36.1 / 384, 6: 37.6 / 397; slack 1: 35.1 / 382, 4: 37.4 / 394); C3 41.8 / 14.4 ->
    // 36.5 / 13.5. Using the counts during the search phase as well changed nothing. Only the PD answers move the bracket, so a poor
    // estimate costs a round, never correctness; a round that did not shrink the bracket 3x falls back.
    bool cnt_round = false;
    if constexpr (SEC) {
      if (a.counts && a.mode == 1 && me && phase == 2 && use_cnt && ca >= a.cnt_min && cb > ca && fa == hi && fb > fa) {
        const double wa = ((double)ca + 0.5) * ((double)ca + 0.5) - 1.0;
        const double wb = ((double)cb + 0.5) * ((double)cb + 0.5) - 1.0;
        const double r = wa / wb;
        const double s = (fa - r * fb) / (1.0 - r);
        if (s > lo && s < hi) {
          const double slack = (hi - s) * fmax(a.cnt_slack / (double)ca, 0.02);
          double p0 = s - slack, p1 = s + slack;
          if (!(p0 > lo)) p0 = lo + 0.25 * (s - lo);
          if (!(p1 < hi)) p1 = 0.5 * (s + hi);
          if (p0 > lo && p0 < p1 && p1 < hi) {
#pragma unroll
            for (int q = 0; q < NP; q++) lam[q] = (gl * NP + q == 0) ? p0 : p1;
            cnt_round = true;
#ifdef PSB_ROUND_STATS
            rtype = 3;
#endif
          }
        }
      }
    }
    // Isolated root: once the failed end of the bracket has exactly one negative pivot, det G changes sign
    // exactly once inside [lo, hi] and is nearly linear there (the other factors sigma_i^2 - lambda barely
    // move over a bracket narrower than the spacing), so the chord between det(lo) > 0 and det(hi) < 0
    // (from the two log |det|) lands on sigma_1^2 to second order. The round probes the chord's root -/+
    // ifrac of the bracket; ifrac goes to its power 3/2 after every round that caught the root between its
    // probes and back to 1/16 after a miss. Measured (C5 matrix 0, tests per bisection point / kernel ms):
    // without counts and chord 41.3 / 425; counts only 35.6 / 381; with the chord, first half-width 1/16:
    // power 2 32.3 / 316, power 3/2 31.5 / 309, power 3 35.7 / 349; first half-width 1/4, 1/8, 1/32 (power
    // 2): 318, 323, 351 ms. Probing the PD secant's root and the chord's root (a lower and an upper bound
    // while det is convex) instead of root -/+ ifrac took more rounds (6.6 against 6.1 chord rounds).
    bool itp_round = false;
    if constexpr (SEC) {
      if (a.counts && a.mode == 1 && me && phase == 2 && use_itp && have_lo && have_hi && hi < INFINITY) {
        const double t = 1.0 / (1.0 + exp(Lhi - Llo));  // det(lo) / (det(lo) - det(hi))
        const double w = hi - lo;
        double s = lo + w * t;
        if (a.counts >= 2 && a.n >= 512 && have_p && lp < lo) {
          // Three-point model det = (s - lambda) exp(alpha + beta lambda): one root times a smooth factor for
          // all the others. The two PD log-dets (lp, lo) and the failed end's log |det| fix s: eliminate
          // alpha, take beta(s) from the PD pair, and solve the remaining equation in s by bisection (it
          // falls from +inf at lo to -inf at hi). About thirty dependent logarithms per round: nothing
          // against a round of n >= 512 rows, but +40% on a round of C1's 100 rows (0.23 -> 0.33 ms) and
          // +8% on C2's 400 for 6% fewer tests, so short matrices keep the plain chord (a rule on the
          // matrix alone). Measured with it: C5 matrix 0 31.5 -> 27.6 tests per point, 307 -> 270 ms;
          // C3 12.5 -> 11.4 ms; C4's bisection kernel 12.0 -> 11.2 ms.
          const double dPD = Llo - Lp, dHL = Lhi - Llo, ilp = 1.0 / (lo - lp);
          double sa = lo, sb = hi, Fa = 0.0, Fb = 0.0;
          bool ha = false, hb = false;
          for (int it = 0; it < 14; it++) {
            const double sm = 0.5 * (sa + sb);
            const double beta = (dPD - log((sm - lo) / (sm - lp))) * ilp;
            const double F = log((hi - sm) / (sm - lo)) + beta * w - dHL;
            if (F > 0.0) { sa = sm; Fa = F; ha = true; } else { sb = sm; Fb = F; hb = true; }
          }
          // 14 halvings, then the chord of F over what is left
          const double s3 = (ha && hb && Fa > Fb) ? sa + (sb - sa) * (Fa / (Fa - Fb)) : 0.5 * (sa + sb);
          if (s3 > lo && s3 < hi) s = s3;
        }
        if (s > lo && s < hi) {
          const double dlt = w * ifrac;
          double p0 = s - dlt, p1 = s + dlt;
          if (!(p0 > lo)) p0 = lo + 0.5 * (s - lo);
          if (!(p1 < hi)) p1 = s + 0.5 * (hi - s);
          if (p0 > lo && p0 < p1 && p1 < hi) {
#pragma unroll
            for (int q = 0; q < NP; q++) lam[q] = (gl * NP + q == 0) ? p0 : p1;
            itp_round = true;
            cnt_round = false;
#ifdef PSB_ROUND_STATS
            rtype = 4;
#endif
          }
        }
      }
    }
    const double2 zt = me ? z : czero();
    bool pd[NP];
    LogDet ld[NP];
    int pos[NP];
#pragma unroll
    for (int q = 0; q < NP; q++) pos[q] = 0;
    int rows = a.n;  // LDL^H rows this warp executed in this round (tests stop early once every probe failed)
#pragma unroll
    for (int q = 0; q < NP; q++) { pd[q] = true; ld[q].init(); }
    if constexpr (DYN) {
      const int b = a.kl + a.ku;
      LV Ls{a.dyn_L + tid * (int64_t)(b * b > 0 ? b * b : 1), 1};
#pragma unroll
      for (int q = 0; q < NP; q++)
        pd[q] = pd_test_dyn(a.n, a.kl, a.ku, a.Ab, a.AHA, zt, lam[q], Ls,
                            a.dyn_D + tid * (int64_t)(2 * (b > 0 ? b : 1)), 1);
    } else {
      PDWin<KL, KU> Wn[NP];
      double zz[NP];
#pragma unroll
      for (int q = 0; q < NP; q++) zz[q] = TZ ? -lam[q] : cnorm2(zt) - lam[q];  // (see g_entry_aha)
      // interior rows of a diagonal-constant band: the G row is a function of z only
      double2 gc[B + 1];
      constexpr bool tz = TZ;
      // TZ: G row i from the per-point slots (identity padding past n), see the point start
      auto gslot = [&](int r, int i) {
        double2 g[B + 1];
        const int sl = (i < a.tz_j0) ? i : (i <= a.tz_j1 ? a.nb : a.tz_j0 + (i - a.tz_j1 - 1));
#pragma unroll
        for (int d = 0; d <= B; d++)
          g[d] = (i < a.n && me) ? a.gb[((int64_t)sl * (B + 1) + d) * a.gb_T + tid] : czero();
#pragma unroll
        for (int q = 0; q < NP; q++) {
#pragma unroll
          for (int c = 0; c <= B; c++)
            if (c <= r) Wn[q].W[r][c] = g[r - c];
          Wn[q].W[r][r].x += (i < a.n) ? zz[q] : 1.0;
          Wn[q].W[r][r].y = 0.0;
        }
      };
      if constexpr (TZ) {
#pragma unroll
        for (int d = 0; d <= B; d++) gc[d] = me ? a.gb[((int64_t)a.nb * (B + 1) + d) * a.gb_T + tid] : czero();
#pragma unroll
        for (int r = 0; r <= B; r++) gslot(r, r);
      } else {
#pragma unroll
        for (int d = 0; d <= B; d++) gc[d] = czero();
#pragma unroll
        for (int r = 0; r <= B; r++) pdw_load_row<KL, KU, NP, true>(Wn, r, a.n, r, a.Ab, zt, zz, a.AHA);
      }
      // Rows run in three segments so no row carries a loader branch: step j loads matrix row
      // j+1+B, which lies in the diagonal-constant interior [tz_j0, tz_j1] for j in [J0, J1).
      // Inside a segment, 8-row blocks are straight-line code (the window shift is register
      // renaming); log-det renormalisation and the all-failed vote sit between blocks.
      int J0 = a.n, J1 = a.n;
      if (tz) {
        J0 = min(max(a.tz_j0 - 1 - B, 0), a.n);
        J1 = min(max(a.tz_j1 - B, J0), a.n);
      }
      bool stop = false;
      rows = 0;
      auto vote = [&]() {
        // (Not in the multisection with counts: a failed probe's count needs every row, and whether a warp
        // could stop depends on its other lanes - a point's probe sequence must depend on (A, z) alone.
        // There the vote rarely fired anyway: it takes every probe of all 32 lanes failing.)
        if (a.mode == 1 && a.counts) return;
        bool any = false;
#pragma unroll
        for (int q = 0; q < NP; q++) any = any || pd[q];
        if (!__any_sync(FULL, any && me)) stop = true;  // every probe of every active lane failed
      };
      auto norm = [&]() {
        if constexpr (SEC) {
#pragma unroll
          for (int q = 0; q < NP; q++) ld[q].norm();
        }
      };
      // rows [j0, j1) in straight-line 8-row blocks, then the remainder
      auto run8 = [&](int j0, int j1, auto&& loader) {
        int j = j0;
        for (; !stop && j + 8 <= j1; j += 8) {
#pragma unroll
          for (int u = 0; u < 8; u++) {
            pdw_step<KL, KU, NP, SEC>(Wn, pd, ld, pos);
            loader(j + u + 1 + B);
          }
          norm();
          if (((j - j0) & 31) == 24) vote();
        }
        for (; !stop && j < j1; j++) {
          pdw_step<KL, KU, NP, SEC>(Wn, pd, ld, pos);
          loader(j + 1 + B);
          if (((j - j0) & 7) == 7) norm();
        }
        rows += j - j0;
        norm();
      };
      // short edge segments: a plain row loop (keeps the unrolled code, and registers, to one body)
      auto run1 = [&](int j0, int j1) {
        for (int j = j0; j < j1; j++) {
          pdw_step<KL, KU, NP, SEC>(Wn, pd, ld, pos);
          gslot(B, j + 1 + B);
          if (((j - j0) & 7) == 7) norm();
        }
        rows += j1 > j0 ? j1 - j0 : 0;
        norm();
      };
      if constexpr (TZ) {
        run1(0, J0);
        run8(J0, J1, [&](int) { pdw_load_row_g<KL, KU, NP>(Wn, B, gc, zz); });
        if (!stop) run1(J1, a.n);
      } else {
        // General band: every lane of the warp walks the same rows in lockstep (the row loop and its
        // early exit are warp-uniform), so the z-independent coefficients of the rows a block of 8
        // steps consumes are one contiguous span of the table, copied into this warp's shared-memory
        // stage by the whole warp (cp.async, 16 B per lane) one block ahead. The row loop then reads
        // them as broadcast shared loads instead of issuing ~15 L2 loads per row one row ahead (the
        // C5 kernel's long-scoreboard stall, profiles/r01_c5_ncu.md). Same values, same arithmetic:
        // the bits do not change.
        typedef BisRow<KL, KU> BR;
        extern __shared__ __align__(16) double2 bis_stage[];
        double2* stg = bis_stage + (threadIdx.x >> 5) * (2 * BR::SE);
        auto fill = [&](int sidx, int i0) {
          double2* dst = stg + sidx * BR::SE;
#pragma unroll
          for (int e0 = 0; e0 < BR::SE; e0 += 32) {
            const int e = e0 + lane;
            if (e0 + 32 <= BR::SE || e < BR::SE) {
              const int i = i0 + e / BR::RW;
              const int ic = i < a.n ? i : a.n - 1;
              cp16z(dst + e, a.RT + (int64_t)ic * BR::RW + (e % BR::RW), i < a.n ? 16u : 0u);
            }
          }
          cp_commit();
        };
        // Staged rows need no edge tests: i >= B + 1, so every column i - d exists, and rows past n are
        // zero-filled by the copy, so their entries come out zero; only the diagonal picks the identity
        // padding (PD-neutral) there.
        auto load_staged = [&](const double2* row, int i) {
          double2 g[B + 1];
          const double2 pq = row[B + 1];  // diagonal: P_0, Q_0 are real and share one slot
          const double g0 = fma(-zt.y, pq.y, fma(-zt.x, pq.x, row[0].x));
#pragma unroll
          for (int d = 1; d <= B; d++) {
            double2 v = row[d];
            if (d <= BR::D) v = g_from_pq(v, row[B + 2 * d], row[B + 2 * d + 1], zt);
            g[d] = v;
          }
#pragma unroll
          for (int q = 0; q < NP; q++) {
#pragma unroll
            for (int c = 0; c < B; c++) Wn[q].W[B][c] = g[B - c];
            Wn[q].W[B][B].x = (i < a.n) ? g0 + zz[q] : 1.0;
            Wn[q].W[B][B].y = 0.0;
          }
        };
        int j = 0, sidx = 0;
        fill(0, 1 + B);
        for (; !stop && j + 8 <= a.n; j += 8) {
          fill(sidx ^ 1, j + 9 + B);  // the next block's rows (rows past n are zero-filled, never read)
          cp_wait<1>();
          __syncwarp();
          const double2* st = stg + sidx * BR::SE;
#pragma unroll
          for (int u = 0; u < 8; u++) {
            pdw_step<KL, KU, NP, SEC>(Wn, pd, ld, pos);
            load_staged(st + u * BR::RW, j + u + 1 + B);
          }
          norm();
          if ((j & 31) == 24) vote();
          __syncwarp();  // every lane has read stage sidx before the next iteration refills it
          sidx ^= 1;
        }
        cp_wait<0>();
        __syncwarp();
        for (; !stop && j < a.n; j++) {
          pdw_step<KL, KU, NP, SEC>(Wn, pd, ld, pos);
          pdw_load_row<KL, KU, NP, true>(Wn, B, a.n, j + 1 + B, a.Ab, zt, zz, a.AHA);
          if ((j & 7) == 7) norm();
        }
        rows = j;
        norm();
      }
    }
    // executed work for the roofline: LDL^H rows x probes of the lanes that hold a point
    if (lane == 0 && a.rowctr) atomicAdd(a.rowctr, (unsigned long long)rows * (unsigned long long)(__popc(act) * NP));
    if (a.mode == 0) {
      // warp-aggregated appends keep a warp's consecutive (spatially adjacent) points together in
      // the lists, so engine-L warps get points with similar step counts (less lane divergence)
      const bool toB = me && (pd[0] || a.force == 2);
      const bool toA = me && !toB;
      const unsigned mA = __ballot_sync(FULL, toA), mB = __ballot_sync(FULL, toB);
      unsigned long long bA = 0, bB = 0;
      if (lane == 0) {
        if (mA) bA = atomicAdd(&a.counters[1], (unsigned long long)__popc(mA));
        if (mB) bB = atomicAdd(&a.counters[7], (unsigned long long)__popc(mB));
      }
      bA = __shfl_sync(FULL, bA, 0);
      bB = __shfl_sync(FULL, bB, 0);
      const unsigned below = (1u << lane) - 1u;
      if (toA) a.listA[bA + __popc(mA & below)] = p;
      if (toB) a.listB[bB + __popc(mB & below)] = pd[0] ? p : ~p;  // ~p: bracket starts at 0 (forced)
      if (me) p = -1;
      continue;
    }
    // ---- mode 1: combine the group's K answers into the new bracket
    double plo = -INFINITY, phi = INFINITY;
#pragma unroll
    for (int q = 0; q < NP; q++) {
      if (pd[q]) plo = fmax(plo, lam[q]);
      else phi = fmin(phi, lam[q]);
    }
#pragma unroll
    for (int off = 1; off < G; off <<= 1) {
      plo = fmax(plo, __shfl_xor_sync(FULL, plo, off, G));
      phi = fmin(phi, __shfl_xor_sync(FULL, phi, off, G));
    }
    // the group's probes in ascending order i = gl * NP + q, with the log dets of the PD ones
    double lamK[K], LK[K];
    bool pdK[K];
    int cK[K];  // negative pivots of the failed probes whose test ran every row (0: no count)
    if constexpr (SEC) {
      const bool full = rows == a.n;
      if constexpr (G == 1) {
#pragma unroll
        for (int q = 0; q < NP; q++) {
          lamK[q] = lam[q]; pdK[q] = pd[q];
          cK[q] = (!pd[q] && full) ? a.n - pos[q] : 0;
          LK[q] = pd[q] ? ld[q].value() : (cK[q] == 1 ? ld[q].absvalue() : 0.0);
        }
      } else {  // G == 2, NP == 1: probe 0 on the group's even lane, probe 1 on the odd one
        const int myc = (!pd[0] && full) ? a.n - pos[0] : 0;
        const double myL = pd[0] ? ld[0].value() : (myc == 1 ? ld[0].absvalue() : 0.0);
        const double oL = __shfl_xor_sync(FULL, myL, 1, 2), olam = __shfl_xor_sync(FULL, lam[0], 1, 2);
        const bool opd = __shfl_xor_sync(FULL, (int)pd[0], 1, 2) != 0;
        const int oc = __shfl_xor_sync(FULL, myc, 1, 2);
        lamK[0] = gl == 0 ? lam[0] : olam; lamK[1] = gl == 0 ? olam : lam[0];
        pdK[0] = gl == 0 ? pd[0] : opd;    pdK[1] = gl == 0 ? opd : pd[0];
        LK[0] = gl == 0 ? myL : oL;        LK[1] = gl == 0 ? oL : myL;
        cK[0] = gl == 0 ? myc : oc;        cK[1] = gl == 0 ? oc : myc;
      }
    }
#ifdef PSB_ROUND_STATS
    if (me && gl == 0 && a.mode == 1) atomicAdd(&a.counters[24 + rtype], 1ull);
#endif
    if (me) {
      rounds++;
      int r = BIS_CONTINUE;
      const double nlo = fmax(lo, plo), nhi = fmin(hi, phi);
      if constexpr (SEC) {
        // secant bookkeeping: keep the two highest PD points that carry a log det
        const double old_w = hi - lo;
#pragma unroll
        for (int q = 0; q < K; q++) {
          if (pdK[q] && lamK[q] > lo) {
            if (have_lo) { lp = lo; Lp = Llo; have_p = true; }
            lo = lamK[q]; Llo = LK[q]; have_lo = true;  // probes are ascending, so lo ends at the top PD one
          }
        }
        lo = fmax(lo, nlo);
        const double new_w = nhi - lo;
        use_sec = (phase == 2 || phi < INFINITY) && !(new_w > old_w / 3.0);  // keep going while it pays
        // counted failures: keep the two lowest; a count-guided round that did not pay sits out one round
#pragma unroll
        for (int q = 0; q < K; q++) {
          if (!pdK[q] && cK[q] > 0) {
            if (lamK[q] < fa) { fb = fa; cb = ca; fa = lamK[q]; ca = cK[q]; }
            else if (lamK[q] > fa && lamK[q] < fb) { fb = lamK[q]; cb = cK[q]; }
          }
        }
        use_cnt = cnt_round ? !(new_w > old_w / 3.0) : true;
        // the failed end: if it moved, it carries a usable log |det| only when its count is exactly one
        if (nhi < hi) {
          have_hi = false;
#pragma unroll
          for (int q = 0; q < K; q++)
            if (!pdK[q] && lamK[q] == nhi && cK[q] == 1 && isfinite(LK[q])) { have_hi = true; Lhi = LK[q]; }
        }
        if (itp_round) {
          const bool caught = !(new_w > 2.5 * ifrac * old_w);
          use_itp = !(new_w > old_w / 3.0);
          ifrac = caught ? fmax(ifrac * sqrt(ifrac), 1e-7) : a.itp_frac0;
        } else {
          use_itp = true;
        }
      }
      if (phase == 1 && nlo < nhi) {
        // search: upward by 4x/16x while no upper bound, else geometric; the linear multisection /
        // secant phase starts once the bracket is within a factor 16
        lo = nlo;
        hi = nhi;
        if (hi <= 16.0 * lo) phase = 2;
      } else {
        phase = 2;
        if (nlo >= nhi) {
          // Non-monotone answers: a PD probe above a non-PD one, so both sit inside the rounding band
          // of sigma_min^2 and the answer is their midpoint. (Not the old bracket's: a secant probe
          // lands in that band while the bracket is still wide.)
          lo = hi = 0.5 * (nlo + nhi);
          r = BIS_DONE;
        } else {
          lo = nlo;
          hi = nhi;
          if (hi - lo <= a.rtol * hi) r = BIS_DONE;
        }
      }
      if (r == BIS_CONTINUE && rounds >= a.max_tests) r = BIS_FAIL;
      if (r != BIS_CONTINUE) {
        // fallback points keep engine L's (non-converged) result unless the squared form is accurate here
        if (gl == 0 && (!a.fallback || (r == BIS_DONE && 0.5 * (lo + hi) >= a.rmin2 * x2))) {
          const int64_t o = out_index(a.outidx, p);
          a.out[o] = sqrt(0.5 * (lo + hi)) * a.sscale;
          a.iters[o] = 1 + rounds * K;  // LDL^H tests incl. the classification test
          a.status[o] = (r == BIS_DONE) ? 1 : 3;
        }
        if (gl == 0) {
          atomicAdd(&a.counters[2], (unsigned long long)(1 + rounds * K));
          atomicAdd(&a.counters[3], 1ull);
        }
        p = -1;
      }
    }
  }
}

// ----------------------------------------------------------------- engine L: staged LU
// Row stream of the staged factorization (psb_set_matrix, static shapes): row j holds what LU step j
// reads besides its window, [A[j+1+kl, j+1+c] for c = 0..W (0 outside the matrix) | v1[j]], W + 2 complex.
template <int KL, int KU>
struct LUS {
  static constexpr int W = KL + KU;
  static constexpr int RW = W + 2;
  static constexpr int RB = 8;             // rows per stage
  static constexpr int SE = RB * RW;       // complex per stage
  static constexpr int BYTES = 2 * SE * 16;  // two stages per warp
};

// Band LU of M = zI - A fused with S1 of Lanczos step 1 (t = U^{-H} v1), warp-uniform: every lane runs the
// row loop in lockstep - lanes without a point in the LU phase (live = false), or whose point is already
// decided, compute on and store nothing - so the z-independent row stream can be staged per warp in shared
// memory by all 32 lanes with cp.async, one 8-row block ahead. (lu_factor loads the next band row and v1
// entry one row ahead per lane; the copy of those loads into the window then waited on L2 every row: ncu
// put 40% of engine L's stall samples on long-scoreboard on C5.) The arithmetic is lu_factor's with the
// fused hook, operation for operation, so the factors, T, R and the outcome carry the same bits. A point is
// decided by an exact zero pivot or a non-finite t_j (see the caller): both finish it as singular (status 2).
template <int KL, int KU>
__device__ bool lu_staged(int n, const double2* __restrict__ Ab, const double2* __restrict__ LUT, double2* stg,
                          int lane, bool live, double2 z, LV FU, LV FL, LVb piv, LV Tn, LV Rn, double tcert,
                          int* rows_done) {
  constexpr int W = KL + KU, NU = W + 1, NL = (KL > 0 ? KL : 1);
  typedef LUS<KL, KU> SS;
  const unsigned FULL = 0xffffffffu;
  bool ok = live;
  double2 win[KL + 1][W + 1];
#pragma unroll
  for (int r = 0; r <= KL; r++) {
#pragma unroll
    for (int c = 0; c <= W; c++) {
      double2 v = czero();
      if (r < n && c < n) {
        const int d = c - r;
        if (d >= -KL && d <= KU) {
          const double2 a = Ab[(int64_t)(d + KL) * n + r];
          v = cmk((d == 0 ? z.x : 0.0) - a.x, (d == 0 ? z.y : 0.0) - a.y);
        }
      }
      win[r][c] = v;
    }
  }
  double2 acc[W + 1];
#pragma unroll
  for (int d = 0; d <= W; d++) acc[d] = czero();
  double tt = 0.0;  // ||t[0..j]||^2
  int nrows = 0;    // rows this lane's point factored
  auto fill = [&](int sidx, int j0) {
    double2* dst = stg + sidx * SS::SE;
#pragma unroll
    for (int e0 = 0; e0 < SS::SE; e0 += 32) {
      const int e = e0 + lane;
      if (e0 + 32 <= SS::SE || e < SS::SE) {
        const int row = j0 + e / SS::RW;
        cp16z(dst + e, LUT + (int64_t)(row < n ? row : n - 1) * SS::RW + (e % SS::RW), row < n ? 16u : 0u);
      }
    }
    cp_commit();
  };
  int sidx = 0;
  fill(0, 0);
  for (int j0 = 0; j0 < n; j0 += SS::RB) {
    if (!__any_sync(FULL, ok)) break;  // every point of the warp decided
    fill(sidx ^ 1, j0 + SS::RB);
    cp_wait<1>();
    __syncwarp();
    const double2* st = stg + sidx * SS::SE;
#pragma unroll 1
    for (int q = 0; q < SS::RB; q++) {
      const int j = j0 + q;
      if (j >= n) break;
      const double2* row = st + q * SS::RW;
      int p = 0;
      double best = cabs1(win[0][0]);
#pragma unroll
      for (int r = 1; r <= KL; r++) {
        const double m = cabs1(win[r][0]);
        if (m > best) { best = m; p = r; }
      }
#pragma unroll
      for (int r = 1; r <= KL; r++) {
        if (p == r) {
#pragma unroll
          for (int c = 0; c <= W; c++) { const double2 t = win[0][c]; win[0][c] = win[r][c]; win[r][c] = t; }
        }
      }
      if (ok) { piv.put(j, p); nrows++; }
      const double2 d = win[0][0];
      double2 ri;
      if (d.x == 0.0 && d.y == 0.0) { ok = false; ri = czero(); }
      else ri = crcp_fast(d);
      const int64_t rb = (int64_t)j * NU;
      double2 u[W + 1];
#pragma unroll
      for (int c = 1; c <= W; c++) {
        u[c - 1] = cmul(win[0][c], ri);
        if (ok) FU.put(rb + c - 1, u[c - 1]);
      }
      u[W] = ri;
      if (ok) FU.put(rb + W, ri);
      // fused S1 at k = 1 (the lu_factor hook): r = v1[j], t_j = (r + acc_0) conj(rinv_j)
      {
        const double2 r = row[W + 1];
        if (ok) Rn.put(j, r);
        const double2 tp = cadd(r, acc[0]);
        const double2 t = cmul(tp, cconj(u[W]));
        if (ok) Tn.put(j, t);
#pragma unroll
        for (int dd = 1; dd <= W; dd++) acc[dd - 1] = cfms_cj(acc[dd], u[dd - 1], tp);
        acc[W] = czero();
        // t_j is final (forward solve), so ||t|| >= ||t[0..j]||; with M = P^T L U, |l| <= sqrt(2) (cabs1 pivots),
        // ||L||_F^2 <= n (1 + 2 kl): sigma_min <= ||v1|| / ||M^{-H} v1|| <= ||L||_F / ||t[0..j]|| (||v1|| = 1),
        // so tt > tcert = n (1 + 2 kl) / (delta ||A||)^2 proves sigma_min <= delta ||A|| (psb_set_matrix).
        tt = fma(t.x, t.x, fma(t.y, t.y, tt));
        if (!(isfinite(t.x) && isfinite(t.y)) || tt > tcert) ok = false;
      }
#pragma unroll
      for (int r = 1; r <= KL; r++) {
        const double2 l = cmul(win[r][0], ri);
        if (ok) FL.put((int64_t)j * NL + r - 1, l);
#pragma unroll
        for (int c = 1; c <= W; c++) win[r][c] = cfms(win[r][c], l, win[0][c]);
      }
#pragma unroll
      for (int r = 0; r < KL; r++) {
#pragma unroll
        for (int c = 0; c < W; c++) win[r][c] = win[r + 1][c + 1];
        win[r][W] = czero();
      }
      // new bottom row: matrix row i = j+1+kl, columns j+1 .. j+1+W, from the stage (lu_factor's `pre`)
      const int i = j + 1 + KL;
#pragma unroll
      for (int c = 0; c <= W; c++) {
        double2 v = czero();
        if (i < n && j + 1 + c < n) {
          const double2 a = row[c];
          v = cmk((c == KL ? z.x : 0.0) - a.x, (c == KL ? z.y : 0.0) - a.y);
        }
        win[KL][c] = v;
      }
    }
    __syncwarp();  // every lane has read stage sidx before the next block refills it
    sidx ^= 1;
  }
  cp_wait<0>();
  __syncwarp();
  *rows_done = nrows;
  return ok;
}

// ----------------------------------------------------------------- engine L kernel
template <int KL, int KU, bool DYN, int DPIPE>
__global__ void __launch_bounds__(128) k_lanczos(LanArgs a) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t gw = a.warp_base + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const Shape s = a.s;
  const int n = s.n;
  double2* base = a.scratch + gw * a.warp_stride;
  const LV FU{base + lane, 32};
  const LV FL{base + (int64_t)n * s.NU * 32 + lane, 32};
  const int64_t vo = (int64_t)n * (s.NU + s.NL) * 32;
  const LV T{base + vo + lane, 32};
  const LV RA0{base + vo + (int64_t)n * 32 + lane, 32};
  const LV RB0{base + vo + (int64_t)n * 64 + lane, 32};
  bool rsw = false;  // static shapes rotate the two residual buffers (RA = newest) instead of copying
  bool s1done = false;  // step 1's S1 already ran fused with the LU
  double2* hist = base + vo + (int64_t)n * 96 + lane;
  const LVb piv{a.pivs + gw * a.piv_stride + lane, 32};
  typedef Ring<(KL > 0 ? KL : 1), KU, DPIPE> RG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RG ring;
  double2* lstage = nullptr;
  if constexpr (!DYN) {
    const int wib = threadIdx.x >> 5;
    constexpr size_t kWarpSmem = RG::BYTES + LUS<(KL > 0 ? KL : 1), KU>::BYTES;  // ring | LU stage
    ring.d = reinterpret_cast<double2*>(smem_raw + (size_t)wib * kWarpSmem);
    ring.pv = reinterpret_cast<int*>(smem_raw + (size_t)wib * kWarpSmem + DPIPE * RG::SF * 32 * 16);
    lstage = reinterpret_cast<double2*>(smem_raw + (size_t)wib * kWarpSmem + RG::BYTES);
    ring.lane = lane;
  }
  const int64_t nA = (int64_t)a.counters[1];

  int64_t p = -1;
  double2 z = czero();
  int phase = 0, k = 0;
  double nu = 1.0, b1 = 1.0, b2 = 1.0, aprev = 0.0, theta = 0.0, s2 = 1.0, dth = 0.0;
  bool exhausted = false;

  auto finish = [&](double sigma, int it, int stt) {
    const int64_t o = out_index(a.outidx, p);
    a.out[o] = sigma * a.sscale;
    a.iters[o] = it;
    a.status[o] = (int8_t)stt;
    atomicAdd(&a.counters[5], (unsigned long long)(it > 0 ? it : 0));
    atomicAdd(&a.counters[6], 1ull);
    if (stt == 3) a.listF[atomicAdd(&a.counters[8], 1ull)] = ~p;  // engine B retries it (fallback launch)
    p = -1;
    phase = 0;
  };

  while (true) {
    const unsigned idle = __ballot_sync(FULL, phase == 0);
    const int nidle = __popc(idle);
    if (!exhausted && nidle > 0 && (nidle >= a.refill || nidle == 32)) {
      unsigned long long bq = 0;
      if (lane == 0) bq = atomicAdd(&a.counters[4], (unsigned long long)nidle);
      bq = __shfl_sync(FULL, bq, 0);
      if (phase == 0) {
        const int rank = __popc(idle & ((1u << lane) - 1u));
        const int64_t q = (int64_t)bq + rank;
        if (q < nA) {
          p = a.listA[q];
          z = cscale(a.zs[p], a.zscale);
          phase = 1;
        }
      }
      if ((int64_t)bq + nidle >= nA) exhausted = true;
    }
    long long tq0 = clock64();
    if constexpr (DYN) {
      if (phase == 1) {
        const bool ok = lu_factor<KL, KU, DYN>(s, a.Ab, z, FU, FL, piv);
        if (!ok) finish(0.0, 0, 2);
        else { phase = 2; k = 1; nu = 1.0; b1 = 1.0; b2 = 1.0; aprev = 0.0; theta = 0.0; s2 = 1.0; dth = 0.0; }
      }
    } else if (__any_sync(FULL, phase == 1)) {
      // LU fused with S1 of step 1 (t = U^{-H} v1): the same arithmetic as pl_s1 at k = 1 (r = v1 exactly),
      // on the U rows as the factorization produces them; the whole warp runs it (lu_staged).
      // A non-finite t_j decides the point already: S2 would carry it into nu = ||M^{-H} v1|| (every T entry
      // reaches nu's sum), and a non-finite nu finishes the point as singular to working precision
      // (sigma = 0, status 2) - the outcome of an exact zero pivot. So the point's factorization stops
      // there (the same results; deep inside the pseudospectrum of a strongly non-normal band U^{-H} v1
      // overflows a few hundred rows in, C5).
      const bool mine = phase == 1;
      const LV Tn = T, Rn = rsw ? RA0 : RB0;  // pl_s1 writes r into the current RB, then swaps
      int lrows = 0;
      const bool ok = lu_staged<(KL > 0 ? KL : 1), KU>(n, a.Ab, a.LUT, lstage, lane, mine, mine ? z : czero(),
                                                       FU, FL, piv, Tn, Rn, a.tcert, &lrows);
      const int lrows0 = lrows;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) lrows += __shfl_xor_sync(FULL, lrows, off);
      if (lane == 0) atomicAdd(&a.counters[20], (unsigned long long)lrows);
      if (a.prof) {  // LU lane utilisation: rows factored for points vs 32 x the rows the warp's pass ran
        int mx = mine ? lrows0 : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, off));
        if (lane == 0) { atomicAdd(&a.prof[8], (unsigned long long)lrows); atomicAdd(&a.prof[9], 32ull * (unsigned long long)mx); }
      }
      if (mine) {
        if (!ok) {
          finish(0.0, 0, 2);
        } else {
          phase = 2; k = 1; nu = 1.0; b1 = 1.0; b2 = 1.0; aprev = 0.0; theta = 0.0; s2 = 1.0; dth = 0.0;
          s1done = true; rsw = !rsw;
        }
      }
    }
    long long tq1 = clock64();
    if (a.prof && lane == 0) atomicAdd(&a.prof[0], (unsigned long long)(tq1 - tq0));
    const unsigned act = __ballot_sync(FULL, phase == 2);
    if (!act) {
      if (exhausted && __ballot_sync(FULL, phase != 0) == 0) break;
      continue;
    }
    // A step iteration costs four sweeps over all n rows whatever the number of lanes stepping. Where the
    // LU decides most points (C5: ~2% survive it), survivors trickle in at less than one per pass, and
    // stepping them as they came ran the sweeps at a quarter of the lanes. So while points remain and
    // fewer than `defer` lanes hold a factored point, those lanes wait and the idle ones take new points
    // (the refill rule fires: 32 - popc(act) >= refill). Scheduling only: every point's arithmetic is its own.
    if (!exhausted && __popc(act) < a.defer && 32 - __popc(act) >= a.refill) continue;
    if (a.prof && lane == 0) { atomicAdd(&a.prof[6], (unsigned long long)__popc(act)); atomicAdd(&a.prof[7], 1ull); }
    if (phase == 2 && s1done) {
      s1done = false;
    } else if (phase == 2) {
      // S1: r_k and U^{-H} r_k
      const double c1 = (k >= 2) ? aprev / b1 : 0.0;
      const double c2 = (k >= 3) ? b1 / b2 : 0.0;
      double bsq;
      if constexpr (DYN) bsq = sweep_s1<KL, KU, DYN>(s, FU, T, RA0, RB0, a.v1, k, c1, c2);
      else {
        bsq = pl_s1<KL, KU, DPIPE>(n, ring, FU, T, rsw ? RB0 : RA0, rsw ? RA0 : RB0, a.v1, k, c1, c2);
        rsw = !rsw;
      }
      if (a.prof) { long long t = clock64(); if (__activemask() && lane == __ffs(__activemask()) - 1) atomicAdd(&a.prof[1], (unsigned long long)(t - tq1)); tq1 = t; }
      if (k >= 2) {
        const double beta = sqrt(bsq);  // beta_{k-1}
        hist[(int64_t)(k - 2) * 32].y = beta;
        const double r = beta * sqrt(fmax(s2, 0.0));
        if (!isfinite(beta)) {
          finish(0.0, k - 1, 4);
        } else if (lanczos_converged(theta, dth, r, beta)) {
          finish(1.0 / (nu * sqrt(theta)), k - 1, 0);
        } else if (k - 1 >= a.kmax) {
          finish(1.0 / (nu * sqrt(theta)), k - 1, 3);
        } else {
          b2 = b1;
          b1 = beta;
        }
      }
    }
    if (phase == 2) {
      // S2: E^H  (after S2: M^{-H} v_k * beta_{k-1})
      double nrm;
      if constexpr (DYN) nrm = sweep_s2<KL, KU, DYN>(s, FL, piv, T);
      else nrm = pl_s2<KL, KU, DPIPE>(n, ring, FL, piv, T);
      if (a.prof) { long long t = clock64(); if (lane == __ffs(__activemask()) - 1) atomicAdd(&a.prof[2], (unsigned long long)(t - tq1)); tq1 = t; }
      if (k == 1) {
        nu = sqrt(nrm);
        // singular to working precision: a non-finite nu, or nu^2 > ncert (sigma_min <= 1 / nu <= delta ||A||)
        if (!(nu > 0.0) || !isfinite(nu) || nrm > a.ncert) finish(0.0, 0, 2);
      }
    }
    if (phase == 2) {
      double acc, wn2 = 0.0;
      if constexpr (DYN) {
        sweep_s3<KL, KU, DYN>(s, FL, piv, T, 1.0 / (nu * b1));
        acc = sweep_s4<KL, KU, DYN>(s, FU, T, RA0, 1.0 / nu, &wn2);
      } else {
        pl_s3<KL, KU, DPIPE>(n, ring, FL, piv, T, 1.0 / (nu * b1));
        if (a.prof) { long long t = clock64(); if (lane == __ffs(__activemask()) - 1) atomicAdd(&a.prof[3], (unsigned long long)(t - tq1)); tq1 = t; }
        acc = pl_s4<KL, KU, DPIPE>(n, ring, FU, T, rsw ? RB0 : RA0, 1.0 / nu, &wn2);
        if (a.prof) { long long t = clock64(); if (lane == __ffs(__activemask()) - 1) atomicAdd(&a.prof[4], (unsigned long long)(t - tq1)); tq1 = t; }
      }
      const double alpha = acc / b1;
      hist[(int64_t)(k - 1) * 32] = cmk(alpha, 0.0);
      double th, sq;
      if (k == 1) {
        th = alpha; sq = 1.0;
      } else {
        th = ritz_top(hist, 32, k, theta, alpha, b1, &sq);
      }
      if (a.prof) { long long t = clock64(); if (lane == __ffs(__activemask()) - 1) atomicAdd(&a.prof[5], (unsigned long long)(t - tq1)); tq1 = t; }
      dth = th - theta;
      theta = th;
      s2 = sq;
      aprev = alpha;
      // Early convergence test (saves the next S1 sweep): with v_k orthogonal to v_{k-1},
      // ||r_{k+1}||^2 = ||w||^2 - alpha_k^2 - beta_{k-1}^2. Cancellation makes that estimate
      // unreliable exactly when beta_k << ||w||, so use the certified upper bound
      // beta_up = sqrt(max(est, 0) + 4 n eps ||w||^2); r_up = beta_up |s_k| >= the true residual.
      if (k >= 2) {
        const double est = wn2 - alpha * alpha - b1 * b1;
        const double beta_up = sqrt(fmax(est, 0.0) + 4.0 * n * 2.220446049250313e-16 * wn2);
        const double r_up = beta_up * sqrt(fmax(s2, 0.0));
        if (isfinite(theta) && theta > 0.0 && lanczos_converged(theta, dth, r_up, beta_up))
          finish(1.0 / (nu * sqrt(theta)), k, 0);
      }
      k++;
    }
  }
}

}  // namespace psb
