// psb_capi.cu — C ABI (include/psb200.h) over the K1 engines and the K2 predictor.
//
// Host side of the drop-in boundary: validates like the reference (ParameterError ->
// PSB_ERR_PARAM, NumericalError -> PSB_ERR_NUMERICAL), owns device memory through an opaque
// handle, and runs the device pipeline
//   [bisection engine: classify + bisect]  ->  [Lanczos engine: LU + inverse Lanczos]
// on one stream. There is no host fallback: every sigma comes from these kernels.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/psb200.h"
#include "psb_dispatch.cuh"
#include "psb_predict.cuh"

using namespace psb;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr; cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Pinned host staging: copies between pageable caller buffers and the device go through it, so
// every cudaMemcpyAsync is a direct DMA (a memcpy on each side of the call is far cheaper than
// the driver's pageable staging).
struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr; cap = 0;
    size_t want = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() { if (p) cudaFreeHost(p); p = nullptr; cap = 0; }
  template <class T> T* at(size_t byte_off) const { return reinterpret_cast<T*>((char*)p + byte_off); }
};

}  // namespace

struct psb_handle {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr, stream2 = nullptr;
  cudaEvent_t ev[14] = {};  // per-launch timing events (run_pipeline)
  std::string err;
  std::mutex mu;
  // matrix
  int n = 0, kl = 0, ku = 0;
  double2 dc{0.0, 0.0};  // engine-split scale (BisArgs): disc of A's diagonal, max off-diagonal column norm^2
  double dr = 0.0, offsq = 0.0;
  double sscale = 1.0, zscale = 1.0;  // exact power-of-two problem scaling (psb_set_matrix)
  double anorm = 0.0;    // general-band kernels' split scale: sqrt(||A||_1 ||A||_inf) >= ||A||_2
  double cert = INFINITY;  // engine L's singularity certificate base 1 / (delta max_j ||A e_j||)^2 (LanArgs)
  int tz_j0 = 1, tz_j1 = 0;  // interior rows sharing one G row (diagonal-constant band), empty by default
  // development knobs, read once at psb_create (A/B switches; defaults are the product path):
  //   PSB_TAU=x default engine split, PSB_BVARIANT=1/2 force the wide / pair bisection variant, PSB_NOBEXP=1 no second engine-B launch, PSB_BTPB=n engine-B block size, PSB_NOSEC=1 plain multisection, PSB_NOTZ=1 per-row G formation, PSB_LWARPS=N cap on
  //   Lanczos warps, PSB_PROF=1 per-phase clock64 counters of the Lanczos kernel (stderr)
  bool k_secant = true, k_toeplitz = true, k_prof = false;
  long long k_lwarps = 0;
  int k_refill = 16;
  int k_btpb = 128;
  double k_tau = 0.0;
  double k_cert_delta = 1e-16;  // PSB_CERT_DELTA=x (0: certificates off, the round-2 overflow rule alone)
  bool k_bexpand = true, k_fallback = true, k_seq = false;
  int k_bvariant = 0;
  double k_lfrac = 0.0;  // 0: by the rule
  int k_defer = 16;
  int k_counts = 2;
  int k_lgmin = 256, k_lgratio = 20;
  int k_bfull = 1;
  struct FitEntry { const void* f; int lkey, btpb, tpb, occ, occFull; int64_t threads; int wregs; };
  std::vector<FitEntry> fit_cache;  // engine-B launch shapes per (kernel, engine-L share)
  struct LanEntry { const void* f; int lsmem, occ, regs; };
  std::vector<LanEntry> lan_cache;  // engine-L occupancy and registers per kernel
  bool have_matrix = false;
  DevBuf Ab, AHA, RT, LUT, v1, offmin, gbuf, listF;
  // per call
  DevBuf zs, outidx, out, iters, status, listA, listB, counters, scratch, pivs, dynL, dynD;
  DevBuf xs, ys, prof;
  PinBuf pin;
  // predictor
  DevBuf params, feat, eig, prob, region, idx, selblk, g13;
  // current device selection (psb_region_select / the region path): h->outidx[0, sel_P) of an sel_N grid
  bool sel_valid = false;
  int64_t sel_N = 0, sel_P = 0;
  int32_t sel_nx = 0;
  psb_stats stats{};
};

// Every entry point runs on the handle's device and gives the caller's current device back on
// return (a torch.distributed rank bound to cuda:r must not find itself on cuda:0 afterwards).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

static int fail(psb_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(h, PSB_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                       " at " #call);                                     \
  } while (0)

static bool fallback_off(const psb_handle* h) { return !h->k_fallback; }

namespace psb {
// Grid shifts on the device: point t is grid index g = idx[t] (or t), z = xs[g % nx] + i ys[g / nx].
// xs / ys are the host's linspace values, so z carries exactly the reference's bits (core.py:70-78).
__global__ void k_grid_points(const double* __restrict__ xs, int nx, const double* __restrict__ ys,
                              const int64_t* __restrict__ idx, int64_t P, double2* __restrict__ zs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int64_t g = idx ? idx[t] : t;
  zs[t] = make_double2(xs[g % nx], ys[g / nx]);
}

}  // namespace psb

// ----------------------------------------------------------------------------- dispatch
// Exact-shape kernel sets (the BASELINE configs and the reference's random banded ensemble
// beta in 1..4, generate.py:42-69) register themselves from their own translation units
// (psb_shape.cu); every other band up to 16/16 runs the runtime-shape (DYN) set.
static std::vector<KPair>& shape_registry() {
  static std::vector<KPair> r;
  return r;
}
void psb::register_shape(const KPair& k) { shape_registry().push_back(k); }

static bool pick(int kl, int ku, KPair* out) {
  const KPair* dyn = nullptr;
  for (const KPair& k : shape_registry()) {
    if (k.kl == kl && k.ku == ku) { *out = k; return true; }
    if (k.kl < 0) dyn = &k;
  }
  if (!dyn) return false;
  *out = *dyn;
  return true;
}

static bool fallback_off(const psb_handle* h);
static constexpr int kClassifyOnly = 3;  // internal force_engine value of psb_engine_split
static int default_kmax(int n) { return std::min(3000, std::max(64, 4 * n)); }

extern "C" {

int psb_version(void) { return 1; }

int psb_create(int device, psb_handle** out) {
  if (!out) return PSB_ERR_PARAM;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return PSB_ERR_CUDA;
  if (device < 0 || device >= count) return PSB_ERR_PARAM;
  DeviceGuard dg(device);
  psb_handle* h = new psb_handle();
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return PSB_ERR_CUDA; }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  h->k_secant = getenv("PSB_NOSEC") == nullptr;
  h->k_toeplitz = getenv("PSB_NOTZ") == nullptr;
  h->k_prof = getenv("PSB_PROF") != nullptr;
  h->k_bexpand = getenv("PSB_NOBEXP") == nullptr;
  h->k_fallback = getenv("PSB_NOFALLBACK") == nullptr;
  h->k_bvariant = getenv("PSB_BVARIANT") ? atoi(getenv("PSB_BVARIANT")) : 0;
  h->k_seq = getenv("PSB_SEQ") != nullptr;  // dev: engine B after engine L (full occupancy) instead of beside it
  h->k_tau = getenv("PSB_TAU") ? atof(getenv("PSB_TAU")) : 0.0;  // dev: default engine split
  h->k_btpb = getenv("PSB_BTPB") ? atoi(getenv("PSB_BTPB")) : 0;  // 0: pick per launch
  h->k_lwarps = getenv("PSB_LWARPS") ? atoll(getenv("PSB_LWARPS")) : 0;
  h->k_lgmin = getenv("PSB_LGMIN") ? atoi(getenv("PSB_LGMIN")) : 256;   // dev: long-general rule, min bisection points per SM
  h->k_lgratio = getenv("PSB_LGRATIO") ? atoi(getenv("PSB_LGRATIO")) : 20;  // dev: ... and nA <= ratio * nB
  h->k_counts = getenv("PSB_COUNTS") ? atoi(getenv("PSB_COUNTS")) : 2;  // dev: 0 count-guided probe placement off, 1 without the three-point chord
  h->k_defer = getenv("PSB_DEFER") ? atoi(getenv("PSB_DEFER")) : 16;      // dev: engine-L step deferral (0: off)
  h->k_lfrac = getenv("PSB_LFRAC") ? atof(getenv("PSB_LFRAC")) : 0.0;   // dev: SM share hosting an engine-L block (long general lists)
  h->k_bfull = getenv("PSB_BFULL") ? atoi(getenv("PSB_BFULL")) : 1;     // dev: 0 restores the two-launch engine B on long general lists
  h->k_refill = getenv("PSB_REFILL") ? atoi(getenv("PSB_REFILL")) : 16;  // dev: engine-L refill threshold
  h->k_cert_delta = getenv("PSB_CERT_DELTA") ? atof(getenv("PSB_CERT_DELTA")) : 1e-16;
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking) != cudaSuccess) { delete h; return PSB_ERR_CUDA; }
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  *out = h;
  return PSB_OK;
}

void psb_destroy(psb_handle* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  DevBuf* bufs[] = {&h->Ab, &h->AHA, &h->RT, &h->LUT, &h->v1, &h->offmin, &h->gbuf, &h->listF, &h->zs, &h->outidx, &h->out, &h->iters, &h->status, &h->listA, &h->listB,
                    &h->counters, &h->scratch, &h->pivs, &h->dynL, &h->dynD, &h->xs, &h->ys, &h->params,
                    &h->feat, &h->eig, &h->prob, &h->region, &h->idx, &h->selblk, &h->g13};
  for (DevBuf* b : bufs) b->release();
  h->pin.release();
  for (auto& ev : h->ev) if (ev) cudaEventDestroy(ev);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->stream2) cudaStreamDestroy(h->stream2);
  delete h;
}

const char* psb_last_error(const psb_handle* h) { return h ? h->err.c_str() : "null handle"; }

int psb_get_stats(const psb_handle* h, psb_stats* out) {
  if (!h || !out) return PSB_ERR_PARAM;
  *out = h->stats;
  return PSB_OK;
}

int psb_set_matrix(psb_handle* h, const double* band, int32_t n, int32_t kl, int32_t ku) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  // no matrix until every upload below succeeded (a failed call must not leave a mixed state)
  h->have_matrix = false;
  if (!band) return fail(h, PSB_ERR_PARAM, "band is NULL");
  if (n < 2) return fail(h, PSB_ERR_PARAM, "expected a square matrix with n >= 2, got n=" + std::to_string(n));
  if (kl < 0 || ku < 0 || kl >= n || ku >= n)
    return fail(h, PSB_ERR_PARAM, "bandwidths must satisfy 0 <= kl, ku < n");
  if (kl > 16 || ku > 16)
    return fail(h, PSB_ERR_PARAM, "band evaluator supports kl, ku <= 16, got kl=" + std::to_string(kl) +
                                      " ku=" + std::to_string(ku));
  const int nd = kl + ku + 1;
  typedef std::complex<double> cd;
  const cd* Ain = reinterpret_cast<const cd*>(band);
  double amax = 0.0;
  for (int64_t t = 0; t < (int64_t)nd * n; t++) {
    if (!std::isfinite(Ain[t].real()) || !std::isfinite(Ain[t].imag()))
      return fail(h, PSB_ERR_PARAM, "matrix entries must be finite");
    amax = std::max(amax, std::max(std::fabs(Ain[t].real()), std::fabs(Ain[t].imag())));
  }
  // Exact power-of-two scaling for matrices far from unit scale: the engines then run on A / 2^e and
  // z / 2^e (|entries| <= 1) and sigma is multiplied back by 2^e, so the squared forms (G = M^H M,
  // Lanczos on (M^H M)^-1) stay in range for |A| up to 1e+-300 (they overflowed from ~1e154). Inside
  // [2^-64, 2^64] nothing is scaled: those matrices keep their validated bits (the scaled problem
  // rounds the log-determinants of the secant differently, and moves the overflow edge of sigma).
  const int ea = (amax > 0.0) ? std::ilogb(amax) : 0;
  const int e2 = (ea > 64 || ea < -64) ? ea + 1 : 0;
  h->sscale = std::ldexp(1.0, e2);
  h->zscale = std::ldexp(1.0, -e2);
  std::vector<cd> Asc((size_t)nd * n);
  for (int64_t t = 0; t < (int64_t)nd * n; t++)
    Asc[t] = cd(std::ldexp(Ain[t].real(), -e2), std::ldexp(Ain[t].imag(), -e2));
  const cd* A = Asc.data();
  const int b = kl + ku;
  CK(cudaSetDevice(h->device));
  // Engine-split scale T(z)^2 = (|z - dc| + dr)^2 + offsq bounds every column norm^2 of M = zI - A:
  // |M[j,j]| = |z - a_jj| <= |z - dc| + dr, and the off-diagonal part of column j is z-independent.
  {
    double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (int i = 0; i < n; i++) {
      const cd a = A[(int64_t)kl * n + i];
      xmin = std::min(xmin, a.real()); xmax = std::max(xmax, a.real());
      ymin = std::min(ymin, a.imag()); ymax = std::max(ymax, a.imag());
    }
    const cd c(0.5 * (xmin + xmax), 0.5 * (ymin + ymax));
    double r = 0.0;
    for (int i = 0; i < n; i++) r = std::max(r, std::abs(A[(int64_t)kl * n + i] - c));
    std::vector<double> off(n, 0.0), offr(n, 0.0);
    for (int d = -kl; d <= ku; d++) {
      if (d == 0) continue;
      for (int i = 0; i < n; i++)
        if (i + d >= 0 && i + d < n) {
          off[i + d] += std::norm(A[(int64_t)(d + kl) * n + i]);
          offr[i] += std::norm(A[(int64_t)(d + kl) * n + i]);
        }
    }
    std::vector<double> om(n);
    for (int i = 0; i < n; i++) om[i] = std::min(off[i], offr[i]);
    CK(h->offmin.ensure(sizeof(double) * n));
    CK(cudaMemcpy(h->offmin.p, om.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    // Engine L's singularity certificates (LanArgs::tcert/ncert) prove sigma_min <= delta max_j ||A e_j||,
    // and max_j ||A e_j|| <= ||A||_2: a point decided there is singular to working precision against the
    // parity gate's floor 1e-14 ||A||_2. Computed on the scaled matrix the engines see.
    double colmax2 = 0.0;
    for (int i = 0; i < n; i++) colmax2 = std::max(colmax2, off[i] + std::norm(A[(int64_t)kl * n + i]));
    const double dl = h->k_cert_delta;
    h->cert = (dl > 0.0 && colmax2 > 0.0) ? 1.0 / (dl * dl * colmax2) : INFINITY;
    h->dc = make_double2(c.real(), c.imag());
    h->dr = r * (1.0 + 1e-15);
    h->offsq = *std::max_element(off.begin(), off.end()) * (1.0 + 1e-15);
  }
  // General-band kernels: A^H A band AHA[d*n + j] = (A^H A)[j, j-d] = sum_k conj(A[k, j]) A[k, j-d], and
  // ||A||_2 <= sqrt(||A||_1 ||A||_inf) for their split scale
  {
    auto Aat = [&](int i, int c) -> cd {
      const int d = c - i;
      if (d < -kl || d > ku || i < 0 || c < 0 || i >= n || c >= n) return cd(0, 0);
      return A[(int64_t)(d + kl) * n + i];
    };
    std::vector<cd> aha((size_t)(b + 1) * n, cd(0, 0));
    for (int j = 0; j < n; j++)
      for (int d = 0; d <= b && j - d >= 0; d++) {
        const int c = j - d;
        cd acc(0, 0);
        for (int k = std::max(0, j - ku); k <= std::min(n - 1, c + kl); k++) acc += std::conj(Aat(k, j)) * Aat(k, c);
        aha[(size_t)d * n + j] = acc;
      }
    std::vector<double> colsum(n, 0.0), rowsum(n, 0.0);
    for (int d = -kl; d <= ku; d++)
      for (int i = 0; i < n; i++) {
        if (i + d < 0 || i + d >= n) continue;
        const double m = std::abs(A[(int64_t)(d + kl) * n + i]);
        rowsum[i] += m;
        colsum[i + d] += m;
      }
    h->anorm = std::sqrt(*std::max_element(colsum.begin(), colsum.end()) * *std::max_element(rowsum.begin(), rowsum.end()));
    CK(h->AHA.ensure(sizeof(cd) * (b + 1) * n));
    CK(cudaMemcpy(h->AHA.p, aha.data(), sizeof(cd) * (b + 1) * n, cudaMemcpyHostToDevice));
    // the same coefficients row-packed for the general-band bisection kernels (BisRow, psb_engines.cuh):
    // row i = [AHA_d (d = 0..b) | (P_0, Q_0) | P_d, Q_d (d = 1..D)], D = max(kl, ku), with
    // P = a + conj(b), Q = i (conj(b) - a), a = A[i, i-d], b = A[i-d, i] (g_pq: plain sums, one rounding each)
    const int Dm = std::max(kl, ku);
    const int RW = b + 2 * Dm + 2;
    std::vector<cd> rt((size_t)RW * n, cd(0, 0));
    for (int i = 0; i < n; i++) {
      cd* row = rt.data() + (size_t)i * RW;
      for (int d = 0; d <= b; d++) row[d] = aha[(size_t)d * n + i];
      for (int d = 0; d <= Dm; d++) {
        const cd av = (d <= kl) ? A[(int64_t)(kl - d) * n + i] : cd(0, 0);
        const cd bv = (d <= ku && i - d >= 0) ? A[(int64_t)(kl + d) * n + (i - d)] : cd(0, 0);
        const cd P(av.real() + bv.real(), av.imag() - bv.imag());
        const cd Q(av.imag() + bv.imag(), bv.real() - av.real());
        if (d == 0) row[b + 1] = cd(P.real(), Q.real());
        else { row[b + 2 * d] = P; row[b + 2 * d + 1] = Q; }
      }
    }
    CK(h->RT.ensure(sizeof(cd) * rt.size()));
    CK(cudaMemcpy(h->RT.p, rt.data(), sizeof(cd) * rt.size(), cudaMemcpyHostToDevice));
  }
  // Lanczos start vector: fixed, identical for every z (determinism)
  std::vector<cd> v1(n);
  double nrm = 0.0;
  for (int i = 0; i < n; i++) {
    v1[i] = cd(std::cos(0.7071 * i + 0.3), std::sin(1.3 * i + 0.1));
    nrm += std::norm(v1[i]);
  }
  nrm = std::sqrt(nrm);
  for (auto& v : v1) v /= nrm;
  CK(cudaSetDevice(h->device));
  CK(h->Ab.ensure(sizeof(cd) * nd * n));
  CK(h->v1.ensure(sizeof(cd) * n * 33));
  CK(cudaMemcpyAsync(h->Ab.p, A, sizeof(cd) * nd * n, cudaMemcpyHostToDevice, h->stream));
  // [0, n): v1; [n, 33n): v1 replicated per lane (v1rep[j*32 + lane]) for coalesced cp.async
  std::vector<cd> v1x((size_t)n * 33);
  for (int i = 0; i < n; i++) {
    v1x[i] = v1[i];
    for (int l = 0; l < 32; l++) v1x[(size_t)n + (size_t)i * 32 + l] = v1[i];
  }
  CK(cudaMemcpyAsync(h->v1.p, v1x.data(), sizeof(cd) * n * 33, cudaMemcpyHostToDevice, h->stream));
  // the staged LU's row stream (LUS, psb_engines.cuh): row j = [A[j+1+kl, j+1+c] for c = 0..b (0 outside the
  // matrix) | v1[j]]
  std::vector<cd> lut((size_t)(b + 2) * n, cd(0, 0));
  for (int j = 0; j < n; j++) {
    cd* row = lut.data() + (size_t)j * (b + 2);
    const int i = j + 1 + kl;
    for (int c = 0; c <= b; c++)
      if (i < n && j + 1 + c < n) row[c] = A[(int64_t)c * n + i];
    row[b + 1] = v1[j];
  }
  CK(h->LUT.ensure(sizeof(cd) * lut.size()));
  CK(cudaMemcpyAsync(h->LUT.p, lut.data(), sizeof(cd) * lut.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->n = n; h->kl = kl; h->ku = ku;
  // Rows whose G(lambda) row entries are bitwise identical: G row j is formed from A's rows
  // [j - ku, j + kl] (g_entry), so rows j whose whole window matches row m's window entry for entry
  // share one G row; the bisection engine forms it once per test. The values are the same numbers
  // the per-row path would form, so results do not change.
  {
    auto same_arow = [&](int i, int m) {
      for (int e = -kl; e <= ku; e++)
        if (A[(int64_t)(e + kl) * n + i] != A[(int64_t)(e + kl) * n + m]) return false;
      return true;
    };
    auto same_row = [&](int i, int m) {
      for (int o = -ku; o <= kl; o++)
        if (!same_arow(i + o, m + o)) return false;
      return true;
    };
    const int m = n / 2;
    h->tz_j0 = 1; h->tz_j1 = 0;
    if (m >= b && m + kl < n) {
      int j0 = m, j1 = m;
      while (j0 - 1 >= b && same_row(j0 - 1, m)) j0--;
      while (j1 + 1 + kl < n && same_row(j1 + 1, m)) j1++;
      // the TZ kernels keep a point's boundary G rows in per-thread slots: only for short boundaries
      if (j1 - j0 >= 16 && j0 + (n - 1 - j1) <= 32) { h->tz_j0 = j0; h->tz_j1 = j1; }
    }
  }
  h->have_matrix = true;
  return PSB_OK;
}

}  // extern "C"

// Flop / byte models, counting only the arithmetic the kernels must do.
// One right-looking LDL^H row per probe: b column scalings (2 flops), b(b-1)/2 off-diagonal complex
// updates (8), b diagonal updates (4), one reciprocal (1) -> 4b^2 + 2b + 1.
static double flops_ldl_row(int kl, int ku) { const double b = kl + ku; return 4.0 * b * b + 2.0 * b + 1.0; }
// Forming one G row from M = zI - A: entry d is a sum of b - d + 1 products conj(M[k,j]) M[k,j-d]
// (8 flops each) -> 4 (b+1)(b+2) + 2 (the two diagonals of M); shared by the probes of a round, and
// formed once per round for the interior rows of a diagonal-constant band.
static double flops_g_row(int kl, int ku) { const double b = kl + ku; return 4.0 * (b + 1) * (b + 2) + 2.0; }
// Forming one G row from the A^H A expansion (g_entry_aha): entry d = 1..max(kl, ku) is AHA_d - Re(z) P_d
// - Im(z) Q_d (two real-by-complex FMAs, 8 flops), the diagonal the same with real P_0, Q_0 (4 flops), plus
// |z|^2 - lambda on the diagonal.
static double flops_g_row_aha(int kl, int ku) { return 8.0 * std::max(kl, ku) + 4.0 + 2.0; }
static double flops_lu_row(int kl, int ku) { const int W = kl + ku; return 6.0 * W + 6.0 + kl * (6.0 + 8.0 * W); }
static double flops_it_row(int kl, int ku) {
  const int W = kl + ku;
  // S1: r update 4 + norm 3 + W cFMA + cmul; S2: kl cFMA; S3: kl cFMA + scale; S4: W cFMA + 2 cmul + dot
  return (4 + 3 + 8.0 * W + 6) + (8.0 * kl) + (8.0 * kl + 2) + (8.0 * W + 6 + 2 + 2);
}
static double bytes_it_row(int kl, int ku) {
  const int W = kl + ku;
  // factors read twice per step (S1,S4: U' + rinv; S2,S3: L) + int32 pivots twice;
  // vectors (steady state, k >= 3): S1 r3 w2 (the residual buffers rotate), S2 r1 w1, S3 r1 w1, S4 r2 w1
  return 16.0 * (2.0 * (W + 1) + 2.0 * kl) + 8.0 + 16.0 * (5 + 2 + 2 + 3);
}

// Core pipeline on device buffers. zs/outidx/out/iters/status are device pointers.
static int run_pipeline(psb_handle* h, const double2* d_zs, const int64_t* d_outidx, int64_t P, double* d_out,
                        int32_t* d_iters, int8_t* d_status, const psb_opts* o, cudaStream_t st,
                        int force_override = -1) {
  psb_opts opt{};
  // Engine split: 1.5e-3 below n = 1000, 1e-3 from there (model error <= 7e-11 / 1.7e-10).
  // A function of the matrix only, so every sigma stays a function of (A, z). Measured per config:
  // n >= 1000 (C3-C5) is faster at 1e-3 (C4 102 -> 85 ms); at n = 400 (C2) 1e-3 leaves the
  // bisection engine a few more points than it has threads next to engine L (2.2 -> 2.46 ms).
  opt.tau = h->k_tau > 0 ? h->k_tau : (h->n >= 1000 ? 1e-3 : 1.5e-3); opt.bis_rtol = 2e-12; opt.kmax = 0; opt.force_engine = 0; opt.refill = h->k_refill;
  if (o) {
    if (o->tau > 0) opt.tau = o->tau;
    if (o->bis_rtol > 0) opt.bis_rtol = o->bis_rtol;
    if (o->kmax > 0) opt.kmax = o->kmax;
    opt.force_engine = (o->force_engine >= 0 && o->force_engine <= 2) ? o->force_engine : 0;
    if (o->refill > 0) opt.refill = o->refill;
  }
  if (force_override >= 0) opt.force_engine = force_override;  // internal modes (kClassifyOnly)
  const int n = h->n, kl = h->kl, ku = h->ku;
  const int kmax = opt.kmax > 0 ? opt.kmax : default_kmax(n);
  KPair kp;
  if (!pick(kl, ku, &kp)) return fail(h, PSB_ERR_CUDA, "library built without a kernel set for this band shape");
  const bool dyn = kp.kl < 0;
  if (!dyn && h->tz_j0 <= h->tz_j1 && h->k_toeplitz) { kp.b = kp.bt; kp.bm = kp.bmt; kp.bm2 = kp.bmt2; }  // diagonal-constant row loop
  h->stats = psb_stats{};
  h->stats.n_points = P;
  if (P == 0) return PSB_OK;

  CK(h->counters.ensure(sizeof(unsigned long long) * 48));  // [16..19]: row counters (classify, B, fallback, B2), [20] LU rows
  CK(h->listA.ensure(sizeof(int64_t) * P));
  CK(h->listB.ensure(sizeof(int64_t) * P));
  CK(h->listF.ensure(sizeof(int64_t) * P));
  unsigned long long* cnt = h->counters.as<unsigned long long>();
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 48, st));

  // ---- classification: one LDL^H test per point at lambda = (tau S)^2 splits the points
  // general-band static kernels stage their G-row coefficients per warp in dynamic shared memory
  const int bsw = (!dyn && !(h->tz_j0 <= h->tz_j1 && h->k_toeplitz)) ? kp.bsmem : 0;
  auto bsm = [&](int tpb) { return (size_t)(tpb / 32) * (size_t)bsw; };
  int occB = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, kp.b, 128, bsm(128)));
  occB = std::max(occB, 1);
  BisArgs ba;
  ba.n = n; ba.kl = kl; ba.ku = ku;
  ba.Ab = h->Ab.as<double2>(); ba.AHA = h->AHA.as<double2>(); ba.offmin = h->offmin.as<double>();
  ba.zs = d_zs; ba.outidx = d_outidx; ba.P = P;
  ba.zscale = h->zscale; ba.sscale = h->sscale;
  ba.anorm = h->anorm; ba.dc = h->dc; ba.dr = h->dr; ba.offsq = h->offsq; ba.tau = opt.tau; ba.rtol = opt.bis_rtol;
  ba.force = opt.force_engine; ba.max_tests = 400;
  ba.out = d_out; ba.iters = d_iters; ba.status = d_status;
  ba.listA = h->listA.as<int64_t>(); ba.listB = h->listB.as<int64_t>(); ba.counters = cnt;
  ba.dyn_L = nullptr; ba.dyn_D = nullptr;
  ba.RT = h->RT.as<double2>();
  ba.rowctr = cnt + 16;  // classification rows x probes
  ba.mode = 0; ba.fallback = 0; ba.rmin2 = 0.0;
  ba.secant = h->k_secant ? 1 : 0;
  ba.counts = h->k_counts;
  ba.cnt_min = 2;
  ba.cnt_slack = 2.0;
  ba.itp_frac0 = 0.0625;
  ba.tz_j0 = h->k_toeplitz ? h->tz_j0 : 1;
  ba.tz_j1 = h->k_toeplitz ? h->tz_j1 : 0;
  const int64_t gridC = std::max<int64_t>(1, std::min<int64_t>((int64_t)occB * h->num_sms, (P + 127) / 128));
  int64_t gridB = (int64_t)occB * h->num_sms, gridB2 = 0;
  cudaStream_t sB = st;  // engine B's stream (stream2 behind engine L in the sequential mode)
  bool b2pair = false;  // the expansion launch runs the pair variant (one probe per lane)
  if (dyn) {
    const int b = std::max(kl + ku, 1);
    const int64_t threads = std::max(gridB, gridC) * 128;
    CK(h->dynL.ensure(sizeof(double2) * threads * b * b));
    CK(h->dynD.ensure(sizeof(double) * threads * 2 * b));
    ba.dyn_L = h->dynL.as<double2>(); ba.dyn_D = h->dynD.as<double>();
  }
  ba.gb = nullptr; ba.nb = 0; ba.gb_T = 0; ba.tid_base = 0;
  const bool tzk = !dyn && h->tz_j0 <= h->tz_j1 && h->k_toeplitz;
  if (tzk) {
    // per-thread G-row slots of the TZ kernels (boundary rows + the interior row), sized per launch
    ba.nb = h->tz_j0 + (n - 1 - h->tz_j1);
    CK(h->gbuf.ensure(sizeof(double2) * (size_t)(ba.nb + 1) * (kl + ku + 1) * (size_t)(gridC * 128)));
    ba.gb = h->gbuf.as<double2>();
  }
  ba.gb_T = gridC * 128;
  CK(cudaEventRecord(h->ev[0], st));
  kp.b<<<(unsigned)gridC, 128, bsm(128), st>>>(ba);
  CK(cudaGetLastError());
  CK(cudaEventRecord(h->ev[1], st));
  // One host round trip reads the list lengths: it sizes both grids and, more importantly, makes the
  // Lanczos blocks (large shared-memory ring) land on every SM before the bisection blocks are
  // submitted. (Launching both straight after classification let the bisection engine take two
  // blocks per SM first and left the Lanczos engine short of SMs: C2 3.3 -> 4.6 ms, measured.)
  unsigned long long hc0[8];
  CK(cudaMemcpyAsync(hc0, cnt, sizeof(hc0), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t nA = (int64_t)hc0[1], nB = (int64_t)hc0[7];
  if (opt.force_engine == kClassifyOnly) {  // psb_engine_split: the split's counts, no sigma
    h->stats.n_bisect = nB; h->stats.n_lanczos = nA;
    float msC0 = 0.f;
    cudaEventElapsedTime(&msC0, h->ev[0], h->ev[1]);
    h->stats.ms_classify = msC0; h->stats.ms_total = msC0;
    h->stats.launches = 1;
    return PSB_OK;
  }
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));  // reset the work counter

  // ---- engine L (band LU + inverse Lanczos) on stream2, concurrently with engine B
  const Shape s = make_shape(n, kl, ku);
  const int64_t warp_stride = ((int64_t)n * (s.NU + s.NL + 3) + kmax) * 32;  // double2 units
  const int64_t piv_stride = ((int64_t)n * 32 + 63) / 64 * 64;                 // int32 units
  // Engine L runs 4-warp blocks (one block per SM with the 8-deep ring). One-warp blocks spread its
  // warps over every SM: faster alone (C2 3.0 -> 2.6 ms) but the concurrent step got slower (3.3 ->
  // 4.3 ms) because every SM then hosts more engine-L warps next to the FP64-bound bisection warps.
  constexpr int kLWarpsPerBlock = 4;
  const int lsmem = kp.lsmem * kLWarpsPerBlock;
  // General-band lists with bisection work (C5): engine B is usually the long pole (FP64-bound, ~1.3 us per
  // point against 0.06-0.3 us for engine L's, most of which a certificate decides early), and two engine-L
  // blocks leave an SM no room for a bisection warp. Engine L then starts with one block on a third of the
  // SMs, engine B is one launch of its full-occupancy grid (its blocks fill the SMs engine L left free at
  // once and the rest as engine L's blocks retire), and the rest of engine L's grid is queued behind engine
  // B: if engine L turns out the longer one, it gets the whole GPU when engine B ends. Launch shape only:
  // the same bits. Rule: nB >= 256 per SM and nA <= 20 nB (engine L's cost per point is not known before it
  // runs: 0.06 us (matrix 1) ... 0.31 us (matrix 0) on C5).
  // Measured, C5 matrices 0/4/12/42/10, before engine L's step deferral: two-launch engine B beside engine
  // L on every SM 483/522/548/918/645 ms; one engine-L block on every SM 471/521/549/920/648; on half
  // 449/496/527/903/629; on a third 442/484/524/900/625. With the deferral (engine L ~25% shorter): half
  // 434/469/516/897/615, a third 428/462/509/891/614. Widening the rule from (1024 per SM, nA <= 3 nB) to
  // (256, 20) with the queued remainder: 20 of the 64 matrices 3..18% faster (matrix 1 147 -> 120 ms), one
  // slower (matrix 45, engine L as long as engine B: 162 -> 196 ms); C5 pass 13.77 -> 13.29 s.
  // After the count-guided probe policy (engine B ~18% shorter) engine L outlasted engine B on 25 matrices,
  // all with nA > 3 nB: two thirds of the SMs there (matrices 45/28/23/63/53/1: 192/237/276/123/156/114 ->
  // 160/188/241/102/129/100 ms), a third where nA <= 3 nB (matrices 0/42 lose 3%/1% on two thirds).
  const bool long_general = bsw > 0 && nA > 0 && h->k_bfull && !h->k_seq &&
                            nB >= (int64_t)h->k_lgmin * h->num_sms && (int64_t)h->k_lgratio * nB >= nA;
  int64_t gridL = 0, gridL2 = 0;  // gridL2: engine L's second launch (long general lists), queued behind engine B
  LanArgs la{};
  int occL = 0;
  if (nA > 0) {
    // memoised per kernel: attribute set-up and the occupancy query once per handle
    auto it = std::find_if(h->lan_cache.begin(), h->lan_cache.end(),
                           [&](const psb_handle::LanEntry& c) { return c.f == (const void*)kp.l && c.lsmem == lsmem; });
    if (it != h->lan_cache.end()) {
      occL = it->occ;
    } else {
      if (lsmem > 48 * 1024) CK(cudaFuncSetAttribute(kp.l, cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occL, kp.l, 32 * kLWarpsPerBlock, lsmem));
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, kp.l));
      h->lan_cache.push_back({(const void*)kp.l, lsmem, occL, fa.numRegs});
    }
    occL = std::max(occL, 1);
    const double budget = 24.0 * (1ull << 30);  // scratch budget (HBM is 180 GB)
    const double per_warp = warp_stride * 16.0 + piv_stride * 4.0;
    int64_t warps = std::min<int64_t>((int64_t)occL * h->num_sms * kLWarpsPerBlock, (nA + 31) / 32);
    warps = std::min<int64_t>(warps, (int64_t)(budget / per_warp));
    if (h->k_lwarps > 0) warps = std::min<int64_t>(warps, h->k_lwarps);
    warps = std::max<int64_t>(kLWarpsPerBlock, (warps + kLWarpsPerBlock - 1) / kLWarpsPerBlock * kLWarpsPerBlock);
    const int64_t warps_all = warps;  // every warp engine L may run (scratch is per warp)
    if (long_general) {
      // a third of the SMs where engine B is clearly the longer engine (nA <= 3 nB), two thirds otherwise
      const double share = h->k_lfrac > 0 ? h->k_lfrac : (3 * nB >= nA ? 1.0 / 3.0 : 2.0 / 3.0);
      warps = std::min<int64_t>(warps, std::max<int64_t>(1, (int64_t)(share * h->num_sms + 0.5)) * kLWarpsPerBlock);
      gridL2 = (warps_all - warps) / kLWarpsPerBlock;
    }
    gridL = warps / kLWarpsPerBlock;
    CK(h->scratch.ensure((size_t)(warps_all * warp_stride * sizeof(double2))));
    CK(h->pivs.ensure((size_t)(warps_all * piv_stride * 4)));
    la.warp_base = 0;
    la.s = s; la.Ab = h->Ab.as<double2>();
    la.v1 = dyn ? h->v1.as<double2>() : h->v1.as<double2>() + n;  // pipelined sweeps read the replicated copy
    la.v1b = h->v1.as<double2>();
    la.LUT = h->LUT.as<double2>();
    la.zs = d_zs; la.outidx = d_outidx; la.listA = h->listA.as<int64_t>(); la.counters = cnt; la.listF = h->listF.as<int64_t>();
    la.zscale = h->zscale; la.sscale = h->sscale;
    la.out = d_out; la.iters = d_iters; la.status = d_status;
    la.scratch = h->scratch.as<double2>(); la.pivs = h->pivs.as<int>();
    la.warp_stride = warp_stride; la.piv_stride = piv_stride;
    la.kmax = kmax; la.refill = std::min(32, std::max(1, opt.refill));
    la.defer = h->k_defer;
    la.ncert = h->cert;
    la.tcert = std::isfinite(h->cert) ? h->cert * (double)n * (1.0 + 2.0 * kl) : INFINITY;
    la.prof = nullptr;
    if (h->k_prof) {
      CK(h->prof.ensure(128));
      CK(cudaMemsetAsync(h->prof.p, 0, 128, st));
      la.prof = h->prof.as<unsigned long long>();
    }
    CK(cudaEventRecord(h->ev[5], st));
    CK(cudaStreamWaitEvent(h->stream2, h->ev[5], 0));
    CK(cudaEventRecord(h->ev[7], h->stream2));
    kp.l<<<(unsigned)gridL, 32 * kLWarpsPerBlock, lsmem, h->stream2>>>(la);
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev[3], h->stream2));
  }
  // ---- engine B (bisection) on the caller's stream, sharing the SMs with engine L
  if (nB > 0) {
    // Engine B fills what engine L leaves of each SM's register file (L: one 4-warp block per SM).
    // The block size is the one that fits the most threads there (points rarely outnumber threads by
    // much, so a second pass over a few leftover points would double the kernel). Launch shape never
    // changes a result: every sigma is a function of (A, z) only.
    cudaFuncAttributes fl{};
    if (nA > 0) {
      for (const auto& c : h->lan_cache)
        if (c.f == (const void*)kp.l) fl.numRegs = c.regs;
    }
    auto warp_regs = [](int r) { return (r * 32 + 255) / 256 * 256; };
    // best block size for a variant: the most threads in what engine L leaves of each SM
    struct Fit { int tpb, occ, occFull; int64_t threads; int wregs; };
    const int regsLkey = (nA > 0) ? warp_regs(fl.numRegs) * (int)(gridL > 0 ? kLWarpsPerBlock : 0) : -1;
    auto fit = [&](bis_fn f, Fit* out) -> cudaError_t {
      // memoised per (kernel, engine-L register share): the attribute and occupancy queries cost
      // microseconds per call, a visible share of a small grid's step
      for (const auto& c : h->fit_cache)
        if (c.f == (const void*)f && c.lkey == regsLkey && c.btpb == h->k_btpb) {
          *out = Fit{c.tpb, c.occ, c.occFull, c.threads, c.wregs};
          return cudaSuccess;
        }
      cudaFuncAttributes fb;
      cudaError_t e = cudaFuncGetAttributes(&fb, f);
      if (e != cudaSuccess) return e;
      *out = Fit{128, 1, 1, -1, warp_regs(fb.numRegs)};
      for (int cand : {128, 64, 32}) {
        if (h->k_btpb > 0 && cand != h->k_btpb) continue;
        int occM = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occM, f, cand, bsm(cand));
        if (e != cudaSuccess) return e;
        occM = std::max(occM, 1);
        int occ = occM;
        if (nA > 0) {
          const int regsL = warp_regs(fl.numRegs) * (int)(gridL > 0 ? kLWarpsPerBlock : 0);
          const int regsB = warp_regs(fb.numRegs) * (cand / 32);
          occ = std::max(1, std::min(occM, (65536 - regsL) / regsB));
        }
        const int64_t thr = (int64_t)occ * cand * h->num_sms;
        if (thr > out->threads) *out = Fit{cand, occ, occM, thr, warp_regs(fb.numRegs)};
      }
      h->fit_cache.push_back({(const void*)f, regsLkey, h->k_btpb, out->tpb, out->occ, out->occFull, out->threads,
                              out->wregs});
      return cudaSuccess;
    };
    // Wide variant (NP probes per lane) or the pair (two lanes per point, same bits): the pair when
    // every point gets its two lanes in one pass (short lists: twice the threads on the same latency
    // chain), the wide variant otherwise (long lists: one G-row formation serves both probes).
    Fit fw, fp;
    CK(fit(kp.bm, &fw));
    CK(fit(kp.bm2, &fp));
    // General bands (staged kernels, C5): engine L takes whole SMs first, so engine B runs mostly at full
    // occupancy behind it, and a list of up to ~5 full-occupancy pair passes finishes sooner on the pair (its
    // late points take half the latency): C5 matrices 1 / 63 (69 k / 60 k points) 301 -> 278, 391 -> 376 ms;
    // matrices 0 / 17 (307 k / 228 k, 13 / 10 passes) lose on it (732 -> 782, 594 -> 632 ms) and keep the wide one.
    const double pair_pass = (double)fp.occFull * h->num_sms * fp.tpb / 2.0;  // points per full pair pass
    const bool short_general = bsw > 0 && (double)nB <= 5.0 * pair_pass;
    const bool pair = kp.bm2 != kp.bm &&
                      (h->k_bvariant == 2 || (h->k_bvariant == 0 && (2 * nB <= fp.threads || short_general)));
    // ((4,4) and the runtime shapes have one variant; PSB_BVARIANT=1/2 forces wide/pair for tests)
    if (pair) { kp.bm = kp.bm2; kp.np = 1; kp.g = 2; }
    const Fit& fc = pair ? fp : fw;
    const int tpbB = fc.tpb, occShare = fc.occ, occFull = fc.occFull;
    const int64_t wantB = (nB * kp.g + tpbB - 1) / tpbB;
    gridB = std::max<int64_t>(1, std::min<int64_t>((int64_t)occShare * h->num_sms, wantB));
    const bool seq = h->k_seq && nA > 0 && gridL > 0;
    if (seq || long_general) gridB = std::max<int64_t>(1, std::min<int64_t>((int64_t)occFull * h->num_sms, wantB));
    // A second launch, queued behind engine L on its stream, takes the SM share engine L releases when
    // it finishes (both launches pull from the same work counter), so a long bisection tail runs at
    // full occupancy instead of the share it had next to engine L.
    // Only for long lists (>= 4 points per thread after the expansion): with ~1-2 points per thread the
    // late starters' last points stretch the tail by a point's latency (C3: +4%; C5: -15%).
    bis_fn fB2 = kp.bm;
    int tpb2 = tpbB, g2 = kp.g;
    if (nA > 0 && gridL > 0 && h->k_bexpand && !seq && !long_general) {
      const int64_t extra = std::max<int64_t>(0, std::min<int64_t>((int64_t)occFull * h->num_sms, wantB) - gridB);
      if (nB * kp.g >= 4 * (gridB + extra) * tpbB) {
        gridB2 = extra;  // long list: the same (wide) variant at full occupancy (C5 1157 -> 975 ms)
      } else if (!pair && kp.bm2 != kp.bm && nB * kp.g >= 2 * gridB * tpbB) {
        // 2-4 points per thread: the pair variant, whose late points finish in about half the latency
        // (C3 15.1 -> 14.8 ms; on C5's long list it lost to the wide expansion, 975 -> 1064 ms)
        const int wB1 = (int)((gridB + h->num_sms - 1) / h->num_sms) * (tpbB / 32);  // B1 warps per SM
        const int used = ((wB1 + 3) / 4) * fw.wregs;                                  // per 16K slice
        const int per_slice = std::max(0, (16384 - used) / fp.wregs);
        const int64_t ex2 = std::min<int64_t>((int64_t)4 * per_slice * h->num_sms, (2 * nB + 31) / 32);
        if (ex2 > 0) { gridB2 = ex2; fB2 = kp.bm2; tpb2 = 32; g2 = 2; b2pair = true; }
      }
    }
    (void)g2;
    ba.mode = 1;
    ba.max_tests = 200;
    ba.rowctr = cnt + 17;  // engine-B rows x probes (the expansion launch counts into cnt[19])
    ba.gb_T = gridB * tpbB + gridB2 * tpb2;
    ba.tid_base = 0;
    if (tzk) {  // after the host round trip the classification kernel is done: resizing is safe
      CK(h->gbuf.ensure(sizeof(double2) * (size_t)(ba.nb + 1) * (kl + ku + 1) * (size_t)ba.gb_T));
      ba.gb = h->gbuf.as<double2>();
    }
    if (dyn) {
      CK(h->dynL.ensure(sizeof(double2) * (size_t)ba.gb_T * std::max(kl + ku, 1) * std::max(kl + ku, 1)));
      CK(h->dynD.ensure(sizeof(double) * (size_t)ba.gb_T * 2 * std::max(kl + ku, 1)));
      ba.dyn_L = h->dynL.as<double2>(); ba.dyn_D = h->dynD.as<double>();
    }
    sB = seq ? h->stream2 : st;
    CK(cudaEventRecord(h->ev[8], sB));
    kp.bm<<<(unsigned)gridB, tpbB, bsm(tpbB), sB>>>(ba);
    CK(cudaGetLastError());
    if (gridB2 > 0) {
      BisArgs b2 = ba;
      b2.tid_base = gridB * tpbB;
      b2.rowctr = cnt + 19;
      fB2<<<(unsigned)gridB2, tpb2, bsm(tpb2), h->stream2>>>(b2);
      CK(cudaGetLastError());
      CK(cudaEventRecord(h->ev[6], h->stream2));
    }
  } else {
    gridB = 0;
  }
  CK(cudaEventRecord(h->ev[2], sB));
  if (gridL2 > 0 && nB > 0) {
    // Engine L's remaining blocks, queued behind engine B on its stream: if engine L (on its share of the
    // SMs) is still running when engine B ends, they take the whole GPU and pull from the same work counter;
    // if it has finished, they find the list exhausted and exit at once. So a list whose engine L turns out
    // longer than estimated costs little (both launches own separate scratch: warp_base).
    LanArgs l2 = la;
    l2.warp_base = gridL * kLWarpsPerBlock;
    CK(cudaEventRecord(h->ev[12], sB));
    kp.l<<<(unsigned)gridL2, 32 * kLWarpsPerBlock, lsmem, sB>>>(l2);
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev[11], sB));
  } else {
    gridL2 = 0;
  }
  if (sB != st) CK(cudaStreamWaitEvent(st, h->ev[2], 0));
  if (nA > 0) CK(cudaStreamWaitEvent(st, h->ev[3], 0));
  if (gridB2 > 0) CK(cudaStreamWaitEvent(st, h->ev[6], 0));
  CK(cudaEventRecord(h->ev[4], st));
  unsigned long long hc[32];
  CK(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  bool ran_fallback = false;
  if (hc[8] > 0 && opt.force_engine == 0 && !fallback_off(h)) {
    // Engine L points that hit kmax (a tight cluster at sigma_min; tools/fuzz_parity.py) get one more
    // chance on engine B from the bracket [0, lambda_tau]; its answer replaces engine L's only where the
    // squared form is accurate (sigma >= 4e-4 X: model error <= 5e-10). The rest stay status 3 and
    // surface as NumericalError like the reference's LinAlgError path (core.py:157-166).
    unsigned long long* cF = cnt + 9;  // engine-B counters of this launch: [0] work, [2] tests, [3] done, [7] listed
    BisArgs bf = ba;
    bf.mode = 1; bf.fallback = 1; bf.rmin2 = 16e-8; bf.max_tests = 200;
    bf.listB = h->listF.as<int64_t>();
    bf.counters = cF;
    bf.rowctr = cnt + 18;
    CK(cudaMemsetAsync(cF, 0, sizeof(unsigned long long) * 7, st));
    CK(cudaMemcpyAsync(cF + 7, cnt + 8, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
    const int tpbF = 128;
    const int64_t gridF = std::min<int64_t>((int64_t)h->num_sms, ((int64_t)hc[8] * kp.g + tpbF - 1) / tpbF);
    bf.gb_T = gridF * tpbF; bf.tid_base = 0;
    if (tzk) {
      CK(h->gbuf.ensure(sizeof(double2) * (size_t)(bf.nb + 1) * (kl + ku + 1) * (size_t)bf.gb_T));
      bf.gb = h->gbuf.as<double2>();
    }
    if (dyn) {
      CK(h->dynL.ensure(sizeof(double2) * (size_t)bf.gb_T * std::max(kl + ku, 1) * std::max(kl + ku, 1)));
      CK(h->dynD.ensure(sizeof(double) * (size_t)bf.gb_T * 2 * std::max(kl + ku, 1)));
      bf.dyn_L = h->dynL.as<double2>(); bf.dyn_D = h->dynD.as<double>();
    }
    CK(cudaEventRecord(h->ev[9], st));
    kp.bm<<<(unsigned)gridF, tpbF, bsm(tpbF), st>>>(bf);
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev[10], st));
    CK(cudaStreamSynchronize(st));
    ran_fallback = true;
  }
  const int64_t nA_run = (int64_t)hc[1], nB_run = (int64_t)hc[7];
  if (getenv("PSB_ROUND_STATS") && hc[3] > 0)
    fprintf(stderr, "[psb rounds] per bisection point: search %.2f section %.2f secant %.2f count %.2f chord %.2f\n",
            (double)hc[24] / hc[3], (double)hc[25] / hc[3], (double)hc[26] / hc[3], (double)hc[27] / hc[3], (double)hc[28] / hc[3]);
  // Per-launch windows from events recorded on each kernel's own stream right before and after it, with
  // no host round trip inside any window (roofline denominators, bench.py):
  //   classification ev0 -> ev1; engine L ev7 -> ev3 (stream2); engine B ev8 -> the later of its own end
  //   (ev2) and the expansion launch's end (ev6, queued behind engine L on stream2); fallback ev9 -> ev10.
  float msC = 0, msB = 0, msL = 0, msT = 0, msF = 0;
  cudaEventElapsedTime(&msC, h->ev[0], h->ev[1]);
  if (nB > 0) {
    cudaEventElapsedTime(&msB, h->ev[8], h->ev[2]);
    if (gridB2 > 0) { float m2 = 0; cudaEventElapsedTime(&m2, h->ev[8], h->ev[6]); msB = std::max(msB, m2); }
  }
  if (nA > 0) {
    cudaEventElapsedTime(&msL, h->ev[7], h->ev[3]);
    if (gridL2 > 0) {  // engine L's window: the union of its two launches' windows (the second may find nothing left)
      float s2 = 0, e2 = 0;
      cudaEventElapsedTime(&s2, h->ev[7], h->ev[12]);
      cudaEventElapsedTime(&e2, h->ev[7], h->ev[11]);
      msL = (s2 >= msL) ? msL + (e2 - s2) : std::max(msL, e2);
    }
  }
  if (ran_fallback) cudaEventElapsedTime(&msF, h->ev[9], h->ev[10]);
  cudaEventElapsedTime(&msT, h->ev[0], ran_fallback ? h->ev[10] : h->ev[4]);
  if (h->k_prof && nA_run > 0) {
    unsigned long long pr[16];
    cudaMemcpy(pr, h->prof.p, 128, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[psb prof] LU lane utilisation %.3f (%llu point-rows of %llu lane-rows the warps' passes ran)\n",
            pr[9] ? (double)pr[8] / (double)pr[9] : 0.0, pr[8], pr[9]);
    fprintf(stderr, "[psb prof] warp-cycles: lu %.3g s1 %.3g s2 %.3g s3 %.3g s4 %.3g ritz %.3g (gridL %lld) "
            "lane-occupancy of step iterations %.3f over %llu warp-steps\n",
            (double)pr[0], (double)pr[1], (double)pr[2], (double)pr[3], (double)pr[4], (double)pr[5], (long long)gridL,
            pr[7] ? (double)pr[6] / (32.0 * (double)pr[7]) : 0.0, pr[7]);
  }
  psb_stats& S = h->stats;
  S.n_bisect = (int64_t)hc[3];
  S.n_lanczos = (int64_t)hc[6];
  S.pd_tests = (int64_t)hc[2] + nA_run;  // bisected points count their classification test; + Lanczos points' one
  S.lanczos_iters = (int64_t)hc[5];
  {
    // Executed FP64 flops, from the kernels' own row counters (a test stops early
    // once every probe of the warp failed, so rows, not tests x n, measure the work). Per LDL^H row and
    // probe: 4b^2 + 2b + 1. G rows:
    //  - diagonal-constant (TZ) kernels form a point's boundary rows and its interior row once per point
    //    from M's entries (4(b+1)(b+2) + 2 each) and read them in every test;
    //  - general-band kernels form every row of every test from the A^H A expansion
    //    (8(kl+1) + 8(ku+1) + 2, g_entry_aha), once per lane for the lane's NP probes.
    const double nb1 = tzk ? (double)(h->tz_j0 + (n - 1 - h->tz_j1) + 1) : 0.0;
    const double rc = (double)hc[16], r1 = (double)hc[17], r2 = (double)hc[19];
    const double np1 = (double)kp.np, np2 = b2pair ? 1.0 : (double)kp.np;
    const double ldl = flops_ldl_row(kl, ku);
    const double pts_c = (double)(nA_run + nB_run), pts_b = (double)(int64_t)hc[3];
    S.flops_classify = rc * ldl + (tzk ? pts_c * nb1 * flops_g_row(kl, ku) : rc * flops_g_row_aha(kl, ku));
    S.flops_bisect = (r1 + r2) * ldl + (tzk ? pts_b * nb1 * flops_g_row(kl, ku)
                                            : (r1 / np1 + r2 / np2) * flops_g_row_aha(kl, ku));
  }
  // LU rows as counted by engine L (a decided point's factorization stops early), sweeps n rows per step
  S.flops_lanczos = (double)hc[20] * flops_lu_row(kl, ku) + (double)hc[5] * n * flops_it_row(kl, ku);
  S.bytes_lanczos = (double)hc[20] * (16.0 * (s.NU + kl) + 4.0) + (double)hc[5] * n * bytes_it_row(kl, ku);
  S.ms_bisect = msB; S.ms_lanczos = msL; S.ms_total = msT; S.ms_classify = msC; S.ms_fallback = msF;
  S.launches = 1 + (gridL > 0 ? 1 : 0) + (gridL2 > 0 ? 1 : 0) + (nB > 0 ? 1 : 0) + (gridB2 > 0 ? 1 : 0) + (ran_fallback ? 1 : 0);
  S.grid_bisect = (int32_t)(gridB + gridB2); S.grid_lanczos = (int32_t)gridL;
  if ((int64_t)(hc[3] + hc[6]) != P)
    return fail(h, PSB_ERR_CUDA, "internal: points finished " + std::to_string(hc[3] + hc[6]) + " != " +
                                     std::to_string(P));
  return PSB_OK;
}

// First point with status >= 3 (not converged / non-finite) -> NumericalError.
static int check_status(psb_handle* h, const int8_t* status, const int64_t* map, int64_t P, int64_t* fail_index) {
  for (int64_t i = 0; i < P; i++) {
    const int64_t o = map ? map[i] : i;
    if (status[o] >= 3) {
      if (fail_index) *fail_index = i;
      return fail(h, PSB_ERR_NUMERICAL, status[o] == 3 ? "band Lanczos did not converge" : "non-finite value");
    }
  }
  return PSB_OK;
}

extern "C" {

int psb_smin_points_device(psb_handle* h, const double* d_zs, int64_t P, const psb_opts* opts, double* d_sigma,
                           int32_t* d_iters, int8_t* d_status, void* stream) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->have_matrix) return fail(h, PSB_ERR_PARAM, "no matrix set");
  if (P < 0 || (P > 0 && (!d_zs || !d_sigma))) return fail(h, PSB_ERR_PARAM, "bad point arguments");
  DeviceGuard dg(h->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  if (!d_iters) { CK(h->iters.ensure(sizeof(int32_t) * std::max<int64_t>(P, 1))); d_iters = h->iters.as<int32_t>(); }
  if (!d_status) { CK(h->status.ensure(sizeof(int8_t) * std::max<int64_t>(P, 1))); d_status = h->status.as<int8_t>(); }
  return run_pipeline(h, reinterpret_cast<const double2*>(d_zs), nullptr, P, d_sigma, d_iters, d_status, opts, st);
}

int psb_smin_points(psb_handle* h, const double* zs, int64_t P, const psb_opts* opts, double* sigma, int32_t* iters,
                    int8_t* status, int64_t* fail_index) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (fail_index) *fail_index = -1;
  if (!h->have_matrix) return fail(h, PSB_ERR_PARAM, "no matrix set");
  if (P < 0 || (P > 0 && (!zs || !sigma))) return fail(h, PSB_ERR_PARAM, "bad point arguments");
  if (P == 0) { h->stats = psb_stats{}; return PSB_OK; }
  // a non-finite shift is the reference's LinAlgError path: NumericalError with the index (core.py:157-166)
  for (int64_t i = 0; i < 2 * P; i++)
    if (!std::isfinite(zs[i])) {
      if (fail_index) *fail_index = i / 2;
      return fail(h, PSB_ERR_NUMERICAL, "non-finite shift point");
    }
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  CK(h->zs.ensure(sizeof(double2) * P));
  CK(h->out.ensure(sizeof(double) * P));
  CK(h->iters.ensure(sizeof(int32_t) * P));
  CK(h->status.ensure(sizeof(int8_t) * P));
  // pinned staging: [zs | sigma | iters | status]
  const size_t oz = 0, os = oz + 16 * (size_t)P, oi = os + 8 * (size_t)P, ot = oi + 4 * (size_t)P;
  CK(h->pin.ensure(ot + (size_t)P));
  std::memcpy(h->pin.at<char>(oz), zs, 16 * (size_t)P);
  CK(cudaMemcpyAsync(h->zs.p, h->pin.at<char>(oz), sizeof(double2) * P, cudaMemcpyHostToDevice, st));
  int rc = run_pipeline(h, h->zs.as<double2>(), nullptr, P, h->out.as<double>(), h->iters.as<int32_t>(),
                        h->status.as<int8_t>(), opts, st);
  if (rc != PSB_OK) return rc;
  CK(cudaMemcpyAsync(h->pin.at<char>(os), h->out.p, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
  if (iters) CK(cudaMemcpyAsync(h->pin.at<char>(oi), h->iters.p, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->pin.at<char>(ot), h->status.p, sizeof(int8_t) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(sigma, h->pin.at<char>(os), 8 * (size_t)P);
  if (iters) std::memcpy(iters, h->pin.at<char>(oi), 4 * (size_t)P);
  if (status) std::memcpy(status, h->pin.at<char>(ot), (size_t)P);
  const int8_t* stat_h = h->pin.at<int8_t>(ot);
  return check_status(h, stat_h, nullptr, P, fail_index);
}

int psb_engine_split(psb_handle* h, const double* zs, int64_t P, int64_t* n_bisect, int64_t* n_lanczos) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->have_matrix) return fail(h, PSB_ERR_PARAM, "no matrix set");
  if (P < 0 || (P > 0 && !zs) || !n_bisect || !n_lanczos) return fail(h, PSB_ERR_PARAM, "bad point arguments");
  for (int64_t i = 0; i < 2 * P; i++)
    if (!std::isfinite(zs[i])) return fail(h, PSB_ERR_PARAM, "non-finite shift point");
  *n_bisect = 0; *n_lanczos = 0;
  if (P == 0) { h->stats = psb_stats{}; return PSB_OK; }
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  CK(h->zs.ensure(sizeof(double2) * P));
  CK(h->out.ensure(sizeof(double) * P));
  CK(h->iters.ensure(sizeof(int32_t) * P));
  CK(h->status.ensure(sizeof(int8_t) * P));
  CK(cudaMemcpyAsync(h->zs.p, zs, sizeof(double2) * P, cudaMemcpyHostToDevice, st));
  const int rc = run_pipeline(h, h->zs.as<double2>(), nullptr, P, h->out.as<double>(), h->iters.as<int32_t>(),
                              h->status.as<int8_t>(), nullptr, st, kClassifyOnly);
  if (rc != PSB_OK) return rc;
  *n_bisect = h->stats.n_bisect;
  *n_lanczos = h->stats.n_lanczos;
  return PSB_OK;
}

}  // extern "C"

// Ordered compaction of a device mask into h->outidx (np.flatnonzero order, core.py:204): three kernels
// and one 8-byte read-back of the count (the pipeline sizes its launches on the host).
static int select_device(psb_handle* h, const uint8_t* d_mask, int64_t N, cudaStream_t st, int64_t* P) {
  const int64_t nblk = (N + SEL_TPB - 1) / SEL_TPB;
  CK(h->outidx.ensure(sizeof(int64_t) * std::max<int64_t>(N, 1)));
  CK(h->selblk.ensure(sizeof(unsigned long long) * (nblk + 1)));
  unsigned long long* blk = h->selblk.as<unsigned long long>();
  int64_t* d_count = reinterpret_cast<int64_t*>(blk + nblk);
  k_sel_count<<<(unsigned)nblk, SEL_TPB, 0, st>>>(d_mask, N, blk);
  k_sel_scan<<<1, SEL_TPB, 0, st>>>(blk, nblk, d_count);
  k_sel_scatter<<<(unsigned)nblk, SEL_TPB, 0, st>>>(d_mask, N, blk, h->outidx.as<int64_t>());
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h->pin.at<char>(0), d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *P = *h->pin.at<int64_t>(0);
  h->sel_N = N;
  h->sel_P = *P;
  return PSB_OK;
}

// Shared body of psb_smin_grid (mode 0: full grid, mode 1: host region uploaded and compacted on the
// device) and psb_smin_selection (mode 2: the handle's current selection from psb_region_select).
static int grid_eval(psb_handle* h, const double* xs, int32_t nx, const double* ys, int32_t ny, int mode,
                     const uint8_t* region, const psb_opts* opts, double* sigma, int32_t* iters, int8_t* status,
                     int64_t* fail_index) {
  if (fail_index) *fail_index = -1;
  if (!h->have_matrix) return fail(h, PSB_ERR_PARAM, "no matrix set");
  if (!xs || !ys || !sigma || nx < 1 || ny < 1) return fail(h, PSB_ERR_PARAM, "bad grid arguments");
  const int64_t N = (int64_t)nx * ny;
  if (mode == 2 && (!h->sel_valid || h->sel_N != N || h->sel_nx != nx))
    return fail(h, PSB_ERR_PARAM, "no device selection for this grid (call psb_region_select first)");
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  // pinned staging: [count | xs | ys | sigma | iters | status]
  const size_t ox = 64, oy = ox + 8 * (size_t)nx, os = oy + 8 * (size_t)ny, oi = os + 8 * (size_t)N,
               ot = oi + 4 * (size_t)N;
  CK(h->pin.ensure(ot + (size_t)N));
  std::memcpy(h->pin.at<char>(ox), xs, 8 * (size_t)nx);
  std::memcpy(h->pin.at<char>(oy), ys, 8 * (size_t)ny);
  CK(h->out.ensure(sizeof(double) * N));
  CK(h->iters.ensure(sizeof(int32_t) * N));
  CK(h->status.ensure(sizeof(int8_t) * N));
  CK(h->xs.ensure(8 * (size_t)nx));
  CK(h->ys.ensure(8 * (size_t)ny));
  CK(cudaMemcpyAsync(h->xs.p, h->pin.at<char>(ox), 8 * (size_t)nx, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->ys.p, h->pin.at<char>(oy), 8 * (size_t)ny, cudaMemcpyHostToDevice, st));
  int64_t P = N;
  const int64_t* d_idx = nullptr;
  int extra = 0;  // kernels launched here besides the pipeline
  if (mode == 1) {
    h->sel_valid = false;  // the region path reuses the selection buffers
    CK(h->region.ensure(N));
    CK(cudaMemcpyAsync(h->region.p, region, N, cudaMemcpyHostToDevice, st));
    int rc = select_device(h, h->region.as<uint8_t>(), N, st, &P);
    if (rc != PSB_OK) return rc;
    extra += 3;
  } else if (mode == 2) {
    P = h->sel_P;
  }
  if (mode != 0) {
    d_idx = h->outidx.as<int64_t>();
    // NaN marks unevaluated points (core.py:203); the full grid overwrites every entry
    k_fill_nan<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(h->out.as<double>(), N);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(h->iters.p, 0, sizeof(int32_t) * N, st));
    CK(cudaMemsetAsync(h->status.p, 0, sizeof(int8_t) * N, st));
    extra += 1;
  }
  CK(h->zs.ensure(sizeof(double2) * std::max<int64_t>(P, 1)));
  if (P > 0) {
    // shifts from the grid axes on the device: z = xs[g % nx] + i ys[g / nx] (the host's linspace bits)
    k_grid_points<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(h->xs.as<double>(), nx, h->ys.as<double>(), d_idx, P,
                                                              h->zs.as<double2>());
    CK(cudaGetLastError());
    int rc = run_pipeline(h, h->zs.as<double2>(), d_idx, P, h->out.as<double>(), h->iters.as<int32_t>(),
                          h->status.as<int8_t>(), opts, st);
    if (rc != PSB_OK) return rc;
    extra += 1;  // k_grid_points
  } else {
    h->stats = psb_stats{};
  }
  h->stats.launches += extra;
  CK(cudaMemcpyAsync(h->pin.at<char>(os), h->out.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
  if (iters) CK(cudaMemcpyAsync(h->pin.at<char>(oi), h->iters.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h->pin.at<char>(ot), h->status.p, sizeof(int8_t) * N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(sigma, h->pin.at<char>(os), 8 * (size_t)N);
  if (iters) std::memcpy(iters, h->pin.at<char>(oi), 4 * (size_t)N);
  if (status) std::memcpy(status, h->pin.at<char>(ot), (size_t)N);
  const int8_t* stat_h = h->pin.at<int8_t>(ot);
  if (mode == 0) return check_status(h, stat_h, nullptr, P, fail_index);
  // restricted: off-region status is 0, so any failure is a selected point; only then is the point's rank
  // in the selection (the index NumericalError names, core.py:163-165) looked up, from the device list
  bool bad = false;
  for (int64_t g = 0; g < N && !bad; g++) bad = stat_h[g] >= 3;
  if (!bad) return PSB_OK;
  std::vector<int64_t> idx((size_t)P);
  CK(cudaMemcpy(idx.data(), d_idx, sizeof(int64_t) * P, cudaMemcpyDeviceToHost));
  return check_status(h, stat_h, idx.data(), P, fail_index);
}

extern "C" {

int psb_smin_grid(psb_handle* h, const double* xs, int32_t nx, const double* ys, int32_t ny, const uint8_t* region,
                  const psb_opts* opts, double* sigma, int32_t* iters, int8_t* status, int64_t* fail_index) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  return grid_eval(h, xs, nx, ys, ny, region ? 1 : 0, region, opts, sigma, iters, status, fail_index);
}

int psb_smin_selection(psb_handle* h, const double* xs, int32_t nx, const double* ys, int32_t ny,
                       const psb_opts* opts, double* sigma, int32_t* iters, int8_t* status, int64_t* fail_index) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  return grid_eval(h, xs, nx, ys, ny, 2, nullptr, opts, sigma, iters, status, fail_index);
}

}  // extern "C"

// FP64 roofline denominator: independent DFMA chains, 8 per thread (no memory traffic).
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
#pragma unroll
      for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

extern "C" {

int psb_fp64_peak(psb_handle* h, double* tflops) {
  if (!h || !tflops) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  CK(h->prob.ensure(64));
  const int iters = 4096, blocks = h->num_sms * 8, threads = 256;
  k_dfma_peak<<<blocks, threads, 0, st>>>(h->prob.as<double>(), 64, 0.9999999, 1e-7);  // warm-up
  CK(cudaGetLastError());
  CK(cudaEventRecord(h->ev[0], st));
  k_dfma_peak<<<blocks, threads, 0, st>>>(h->prob.as<double>(), iters, 0.9999999, 1e-7);
  CK(cudaEventRecord(h->ev[1], st));
  CK(cudaEventSynchronize(h->ev[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  const double flops = 2.0 * 8.0 * 8.0 * iters * (double)blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return PSB_OK;
}

int psb_predict_points(psb_handle* h, const double* params, const double* mean33, const double* std33,
                       const double* f30, const double* eig, int32_t n_eig, const double* eig_mean,
                       const double* zs, int64_t P, double* prob) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!params || !mean33 || !std33 || !f30 || !eig || !eig_mean || n_eig < 1 || P < 0 || (P > 0 && (!zs || !prob)))
    return fail(h, PSB_ERR_PARAM, "bad predictor arguments");
  if (P == 0) return PSB_OK;
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  const size_t npar = MlpOff::total;
  CK(h->params.ensure(sizeof(double) * npar));
  CK(h->feat.ensure(sizeof(double) * 96));
  CK(h->eig.ensure(sizeof(double2) * n_eig));
  CK(h->zs.ensure(sizeof(double2) * P));
  CK(h->prob.ensure(sizeof(double) * P));
  CK(cudaMemcpyAsync(h->params.p, params, sizeof(double) * npar, cudaMemcpyHostToDevice, st));
  double feat[96];
  std::memcpy(feat, mean33, 33 * sizeof(double));
  std::memcpy(feat + 33, std33, 33 * sizeof(double));
  std::memcpy(feat + 66, f30, 30 * sizeof(double));
  CK(cudaMemcpyAsync(h->feat.p, feat, sizeof(feat), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->eig.p, eig, sizeof(double2) * n_eig, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->zs.p, zs, sizeof(double2) * P, cudaMemcpyHostToDevice, st));
  PredictArgs a;
  a.params = h->params.as<double>();
  a.mean33 = h->feat.as<double>();
  a.std33 = h->feat.as<double>() + 33;
  a.f30 = h->feat.as<double>() + 66;
  a.eig = h->eig.as<double2>();
  a.eig_mean = cmk(eig_mean[0], eig_mean[1]);
  a.n_eig = n_eig;
  a.zs = h->zs.as<double2>();
  a.P = P;
  a.prob = h->prob.as<double>();
  CK(h->g13.ensure(sizeof(double) * 2 * P));
  a.g13 = h->g13.as<double>();
  k_point_features<<<(unsigned)((P + 127) / 128), 128, 0, st>>>(a);
  CK(cudaGetLastError());
  const size_t smem = MLP_SMEM;
  CK(cudaFuncSetAttribute(k_predict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = (P + MLP_PB - 1) / MLP_PB;
  k_predict<<<(unsigned)grid, MLP_TPB, smem, st>>>(a);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(prob, h->prob.p, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PSB_OK;
}

int psb_region_select(psb_handle* h, const double* prob, int32_t ny, int32_t nx, double tau, int32_t k,
                      uint8_t* region, int64_t* idx, int64_t* count) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!prob || !region || ny < 1 || nx < 1 || k < 1 || (k % 2) == 0)
    return fail(h, PSB_ERR_PARAM, "bad region arguments");
  const int64_t N = (int64_t)ny * nx;
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  h->sel_valid = false;
  CK(h->prob.ensure(sizeof(double) * N));
  CK(h->region.ensure(N));
  CK(h->pin.ensure(64));
  CK(cudaMemcpyAsync(h->prob.p, prob, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  k_region<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(h->prob.as<double>(), ny, nx, tau, k, h->region.as<uint8_t>());
  CK(cudaGetLastError());
  // the selected points' row-major index list stays on the device for psb_smin_selection
  int64_t P = 0;
  int rc = select_device(h, h->region.as<uint8_t>(), N, st, &P);
  if (rc != PSB_OK) return rc;
  CK(cudaMemcpyAsync(region, h->region.p, N, cudaMemcpyDeviceToHost, st));
  if (idx && P > 0) CK(cudaMemcpyAsync(idx, h->outidx.p, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (count) *count = P;
  h->sel_valid = true;
  h->sel_nx = nx;
  return PSB_OK;
}

int psb_recall_sweep(psb_handle* h, const double* prob, const uint8_t* truth, int32_t ny, int32_t nx, int32_t k,
                     const double* taus, int32_t n_tau, double* recall) {
  if (!h) return PSB_ERR_PARAM;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!prob || !truth || !taus || !recall || ny < 1 || nx < 1 || k < 1 || (k % 2) == 0 || n_tau < 1 ||
      n_tau > 4096)
    return fail(h, PSB_ERR_PARAM, "bad recall-sweep arguments");
  const int64_t N = (int64_t)ny * nx;
  int64_t denom = 0;
  for (int64_t g = 0; g < N; g++) denom += truth[g] ? 1 : 0;
  if (denom == 0) {  // _recall: an empty truth zone has recall 1.0 (pipeline.py:235-237)
    for (int t = 0; t < n_tau; t++) recall[t] = 1.0;
    return PSB_OK;
  }
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  CK(h->prob.ensure(sizeof(double) * N));
  CK(h->region.ensure(N));
  CK(h->xs.ensure(sizeof(double) * n_tau + sizeof(unsigned long long) * n_tau));
  double* d_taus = h->xs.as<double>();
  unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(d_taus + n_tau);
  CK(cudaMemcpyAsync(h->prob.p, prob, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->region.p, truth, N, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_taus, taus, sizeof(double) * n_tau, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * n_tau, st));
  k_recall<<<(unsigned)((N + 255) / 256), 256, sizeof(unsigned) * n_tau, st>>>(
      h->prob.as<double>(), h->region.as<uint8_t>(), ny, nx, k, d_taus, n_tau, d_cnt);
  CK(cudaGetLastError());
  std::vector<unsigned long long> cnt((size_t)n_tau);
  CK(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned long long) * n_tau, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int t = 0; t < n_tau; t++) recall[t] = (double)cnt[(size_t)t] / (double)denom;  // numpy int/int
  return PSB_OK;
}

}  // extern "C"
