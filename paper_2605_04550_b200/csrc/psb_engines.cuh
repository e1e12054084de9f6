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
  const double2* __restrict__ AHA;
  const double2* __restrict__ zs;
  const int64_t* __restrict__ outidx;  // nullable: output index of point p
  int64_t P;
  double anorm, tau, rtol;
  int force, max_tests;
  double* out;
  int32_t* iters;
  int8_t* status;
  int64_t* listA;                 // points handed to the Lanczos engine
  unsigned long long* counters;   // [0] work, [1] nA, [2] pd tests, [3] nB
  double2* dyn_L;                 // DYN only: per-thread b*b ring
  double* dyn_D;                  // DYN only: per-thread 2b
};

struct LanArgs {
  Shape s;
  const double2* __restrict__ Ab;
  const double2* __restrict__ v1;
  const double2* __restrict__ zs;
  const int64_t* __restrict__ outidx;
  const int64_t* __restrict__ listA;
  unsigned long long* counters;   // [1] nA (read), [4] work, [5] lanczos steps, [6] nL
  double* out;
  int32_t* iters;
  int8_t* status;
  double2* scratch;               // per warp: F n*NF*32 | T n*32 | RA n*32 | RB n*32 | hist kmax*32
  uint8_t* pivs;                  // per warp: n*32
  int64_t warp_stride, piv_stride;
  int kmax, refill;
};

__device__ __forceinline__ int64_t out_index(const int64_t* outidx, int64_t p) { return outidx ? outidx[p] : p; }

// ----------------------------------------------------------------- engine B kernel
template <int KL, int KU, bool DYN>
__global__ void __launch_bounds__(128) k_bisect(BisArgs a) {
  constexpr int B = KL + KU;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t p = -1;
  double2 z = czero();
  BisState st;
  st.lam = 1.0; st.tests = 0; st.phase = 0; st.lo = st.hi = 0.0;
  bool exhausted = false;
  while (true) {
    unsigned idle = __ballot_sync(FULL, p < 0);
    if (idle && !exhausted) {
      const int cnt = __popc(idle);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)cnt);
      base = __shfl_sync(FULL, base, 0);
      if (p < 0) {
        const int rank = __popc(idle & ((1u << lane) - 1u));
        const int64_t q = (int64_t)base + rank;
        if (q < a.P) {
          z = a.zs[q];
          if (a.force == 1) {  // Lanczos-only mode: hand over immediately
            unsigned long long slot = atomicAdd(&a.counters[1], 1ull);
            a.listA[slot] = q;
          } else {
            p = q;
            bis_start(st, hypot(z.x, z.y), a.anorm, a.tau);
          }
        }
      }
      if ((int64_t)base + cnt >= a.P) exhausted = true;
    }
    const unsigned act = __ballot_sync(FULL, p >= 0);
    if (!act) {
      if (exhausted) break;
      continue;
    }
    const bool me = p >= 0;
    const double lam = me ? st.lam : 1.0;
    const double2 zt = me ? z : czero();
    bool pd = true;
    if constexpr (DYN) {
      const int b = a.kl + a.ku;
      LV Ls{a.dyn_L + tid * (int64_t)(b * b > 0 ? b * b : 1), 1};
      pd = pd_test_dyn(a.n, a.kl, a.ku, a.Ab, a.AHA, zt, lam, Ls, a.dyn_D + tid * (int64_t)(2 * (b > 0 ? b : 1)), 1);
    } else {
      PDRing<KL, KU> R;
      pd_init(R);
      const double zz = cnorm2(zt) - lam;
      int grp = 0;
      for (int jb = 0; jb < a.n; jb += B) {
        PDUnroll<KL, KU, 0>::run(R, a.n, jb, a.Ab, a.AHA, zt, zz, pd);
        if ((++grp & 7) == 0 && !__any_sync(FULL, pd && me)) break;  // every active lane failed
      }
    }
    if (me) {
      const int r = bis_update(st, pd, a.rtol, a.force == 2, a.max_tests);
      if (r == BIS_DONE || r == BIS_FAIL) {
        const int64_t o = out_index(a.outidx, p);
        a.out[o] = bis_sigma(st);
        a.iters[o] = st.tests;
        a.status[o] = (r == BIS_DONE) ? 1 : 3;
        atomicAdd(&a.counters[2], (unsigned long long)st.tests);
        atomicAdd(&a.counters[3], 1ull);
        p = -1;
      } else if (r == BIS_TO_LANCZOS) {
        unsigned long long slot = atomicAdd(&a.counters[1], 1ull);
        a.listA[slot] = p;
        atomicAdd(&a.counters[2], (unsigned long long)st.tests);
        p = -1;
      }
    }
  }
}

// ----------------------------------------------------------------- engine L kernel
template <int KL, int KU, bool DYN>
__global__ void __launch_bounds__(128) k_lanczos(LanArgs a) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const Shape s = a.s;
  const int n = s.n;
  double2* base = a.scratch + gw * a.warp_stride;
  const LV F{base + lane, 32};
  const LV T{base + (int64_t)n * s.NF * 32 + lane, 32};
  const LV RA{base + (int64_t)n * (s.NF + 1) * 32 + lane, 32};
  const LV RB{base + (int64_t)n * (s.NF + 2) * 32 + lane, 32};
  double2* hist = base + (int64_t)n * (s.NF + 3) * 32 + lane;
  const LVb piv{a.pivs + gw * a.piv_stride + lane, 32};
  const int64_t nA = (int64_t)a.counters[1];

  int64_t p = -1;
  double2 z = czero();
  int phase = 0, k = 0;
  double nu = 1.0, b1 = 1.0, b2 = 1.0, aprev = 0.0, theta = 0.0, s2 = 1.0, dth = 0.0;
  bool exhausted = false;

  auto finish = [&](double sigma, int it, int stt) {
    const int64_t o = out_index(a.outidx, p);
    a.out[o] = sigma;
    a.iters[o] = it;
    a.status[o] = (int8_t)stt;
    atomicAdd(&a.counters[5], (unsigned long long)(it > 0 ? it : 0));
    atomicAdd(&a.counters[6], 1ull);
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
          z = a.zs[p];
          phase = 1;
        }
      }
      if ((int64_t)bq + nidle >= nA) exhausted = true;
    }
    if (phase == 1) {
      const bool ok = lu_factor<KL, KU, DYN>(s, a.Ab, z, F, piv);
      if (!ok) {
        finish(0.0, 0, 2);
      } else {
        phase = 2; k = 1; nu = 1.0; b1 = 1.0; b2 = 1.0; aprev = 0.0; theta = 0.0; s2 = 1.0; dth = 0.0;
      }
    }
    const unsigned act = __ballot_sync(FULL, phase == 2);
    if (!act) {
      if (exhausted && __ballot_sync(FULL, phase != 0) == 0) break;
      continue;
    }
    if (phase == 2) {
      // S1: r_k and U^{-H} r_k
      const double c1 = (k >= 2) ? aprev / b1 : 0.0;
      const double c2 = (k >= 3) ? b1 / b2 : 0.0;
      const double bsq = sweep_s1<KL, KU, DYN>(s, F, T, RA, RB, a.v1, k, c1, c2);
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
      const double nrm = sweep_s2<KL, KU, DYN>(s, F, piv, T);
      if (k == 1) {
        nu = sqrt(nrm);
        if (!(nu > 0.0) || !isfinite(nu)) finish(0.0, 0, 2);  // singular to working precision
      }
    }
    if (phase == 2) {
      sweep_s3<KL, KU, DYN>(s, F, piv, T, 1.0 / (nu * b1));
      const double acc = sweep_s4<KL, KU, DYN>(s, F, T, RA, 1.0 / nu);
      const double alpha = acc / b1;
      hist[(int64_t)(k - 1) * 32] = cmk(alpha, 0.0);
      double th, sq;
      if (k == 1) {
        th = alpha; sq = 1.0;
      } else {
        const double x0 = (fmax(theta, alpha) + b1) * (1.0 + 1e-14) + 1e-300;
        th = ritz_top(hist, 32, k, x0, &sq);
      }
      dth = th - theta;
      theta = th;
      s2 = sq;
      aprev = alpha;
      k++;
    }
  }
}

}  // namespace psb
