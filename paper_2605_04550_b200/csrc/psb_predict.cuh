// psb_predict.cuh — K2: the reference's sensitivity classifier and region selection on device.
//
//   per-point features   pseudospec/features.py:129-137 point_features_many (g1 = min|z-l|,
//                        g2 = |z - mean l|, g3 = mean|z-l|; numpy pairwise summation restated)
//                        features.py:145-151 assemble_many, 163-164 standardize
//   Fourier encoding     pseudospec/network.py:62-75 (x, y, then sin/cos at 2^1..2^6)
//   dual-path MLP        pseudospec/network.py:153-190 (_forward_cache/forward, SiLU, sigmoid),
//                        parameter layout network.py:35-52 PARAM_SHAPES (59,841 float64)
//   region               pseudospec/pipeline.py:227-231 predicted_region: dilate(prob >= tau, 5)
//                        with border clipping (core.py:224-231, scipy binary_dilation)
//
// FP64 throughout (the reference network is float64, network.py:1-14). Four lanes per point, each
// taking a quarter of a layer's outputs; weights are read with four addresses per warp (one per lane
// of a group), activations live in shared memory interleaved by point ([unit][point slot]).
#pragma once
#include "psb_algo.cuh"

namespace psb {

// parameter offsets in PARAM_SHAPES order
struct MlpOff {
  static constexpr int w_c1 = 0, b_c1 = w_c1 + 64 * 26, w_c2 = b_c1 + 64, b_c2 = w_c2 + 64 * 64;
  static constexpr int w_m1 = b_c2 + 64, b_m1 = w_m1 + 128 * 33, w_m2 = b_m1 + 128, b_m2 = w_m2 + 64 * 128;
  static constexpr int w_t1 = b_m2 + 64, b_t1 = w_t1 + 128 * 128, w_t2 = b_t1 + 128, b_t2 = w_t2 + 128 * 128;
  static constexpr int w_proj = b_t2 + 128, b_proj = w_proj + 64 * 128, w_head = b_proj + 64,
                       b_head = w_head + 64, total = b_head + 1;
};
static_assert(MlpOff::total == 59841, "PARAM_SHAPES total");

// Four warps share 32 points: lane = point, and warp w computes the outputs o = 4 m + w of every layer, so
// a 128-thread block holds 32 points and its activations (two 128-wide buffers + the three per-point
// features) take 66 KB: three blocks = 12 warps per SM, and every weight load is one warp-uniform
// (broadcast) address. (One thread per point with three 128-wide buffers needed 96 KB per warp: two warps
// per SM. Four *lanes* per point gave the same occupancy but four addresses per weight load: the LSU's
// wavefronts then bound the kernel, 3.9 ms for 65,536 points.)
constexpr int MLP_TPB = 128;  // threads per block
constexpr int MLP_GL = 4;     // warps per point group (output split)
constexpr int MLP_PB = MLP_TPB / MLP_GL;  // points per block
constexpr size_t MLP_SMEM = sizeof(double) * ((size_t)(2 * 128 + 3) * MLP_PB + 32);

__device__ __forceinline__ double expit_d(double x) { return 1.0 / (1.0 + exp(-x)); }

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src pairwise_sum, PW_BLOCKSIZE 128)
// over f(k), k in [lo, lo+len). Blocks of <= 128 terms: 8 running sums, combined as a tree.
template <class F>
__device__ double np_pairwise_leaf(F f, int lo, int len) {
  if (len < 8) {
    double res = 0.0;  // numpy starts from -0.0 for sums; identical for the non-negative terms here
    for (int i = 0; i < len; i++) res += f(lo + i);
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; j++) r[j] = f(lo + j);
  int i;
  for (i = 8; i < len - (len % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] += f(lo + i + j);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < len; i++) res += f(lo + i);
  return res;
}

// numpy's recursion (len > 128: split at n2 = len/2 rounded down to a multiple of 8, left + right)
// evaluated in post-order on an explicit stack: device recursion would live on the per-thread call
// stack (1 KB by default), which n = 2000 eigenvalues (five levels) overflowed.
template <class F>
__device__ double np_pairwise(F f, int lo, int len) {
  struct Frame { int lo, len, state; double left; };
  Frame st[32];  // depth <= log2(2^31 / 128) + 1
  int sp = 0;
  st[0] = Frame{lo, len, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& fr = st[sp];
    if (fr.len <= 128) { ret = np_pairwise_leaf(f, fr.lo, fr.len); sp--; continue; }
    int n2 = fr.len / 2;
    n2 -= n2 % 8;
    if (fr.state == 0) { fr.state = 1; st[sp + 1] = Frame{fr.lo, n2, 0, 0.0}; sp++; }
    else if (fr.state == 1) { fr.left = ret; fr.state = 2; st[sp + 1] = Frame{fr.lo + n2, fr.len - n2, 0, 0.0}; sp++; }
    else { ret = fr.left + ret; sp--; }
  }
  return ret;
}

// y[o] = act(b[o] + sum_i W[o, i] x[i]) for the block's 32 points: warp gl takes the outputs o = 4 m + gl
// in passes of eight, so eight independent FMA chains are in flight per lane (every layer's width is a
// multiple of 32). Each output keeps its own sequential sum over i (network.py:87-92's fixed per-row
// order), so the values do not depend on how the outputs are split. `xin(i)` reads input i of the
// lane's point; outputs go to y[o * MLP_PB + ps]. The caller separates layers with __syncthreads().
template <class XIn>
__device__ __forceinline__ void dense(const double* __restrict__ W, const double* __restrict__ bvec, int nin,
                                      int nout, XIn xin, double* y, int ps, int gl, bool act) {
  constexpr int C = 8;
  for (int m0 = 0; m0 * MLP_GL < nout; m0 += C) {
    double acc[C];
    const double* w[C];
#pragma unroll
    for (int k = 0; k < C; k++) { acc[k] = 0.0; w[k] = W + (int64_t)((m0 + k) * MLP_GL + gl) * nin; }
    for (int i = 0; i < nin; i++) {
      const double xi = xin(i);
#pragma unroll
      for (int k = 0; k < C; k++) acc[k] = fma(__ldg(w[k] + i), xi, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < C; k++) {
      const int o = (m0 + k) * MLP_GL + gl;
      const double v = acc[k] + __ldg(bvec + o);
      y[o * MLP_PB + ps] = act ? v * expit_d(v) : v;
    }
  }
}

struct PredictArgs {
  const double* params;
  const double* mean33;
  const double* std33;
  const double* f30;
  const double2* eig;
  double2 eig_mean;
  int n_eig;
  const double2* zs;
  int64_t P;
  double* prob;
  double* g13;  // per point: g1 = min |z - lambda|, g3 = mean |z - lambda| (k_point_features)
};

// Per-point spectral features g1, g3 (features.py:129-137): two passes over the n eigenvalues per point,
// more than half of the predictor's instructions at n = 2000. They need no shared memory, so they run as
// their own full-occupancy kernel (k_predict's 96 KB of activations per warp allow two warps per SM);
// every lane of a warp reads the same eigenvalue (broadcast). The same arithmetic as before the split.
__global__ void __launch_bounds__(128) k_point_features(PredictArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.P) return;
  const double2 z = a.zs[p];
  double g1 = INFINITY;
  for (int k = 0; k < a.n_eig; k++) {
    const double2 l = a.eig[k];
    const double d = hypot(z.x - l.x, z.y - l.y);
    g1 = fmin(g1, d);
  }
  auto dist = [&](int k) { const double2 l = a.eig[k]; return hypot(z.x - l.x, z.y - l.y); };
  const double g3 = np_pairwise(dist, 0, a.n_eig) / (double)a.n_eig;
  a.g13[2 * p] = g1;
  a.g13[2 * p + 1] = g3;
}

__global__ void __launch_bounds__(MLP_TPB) k_predict(PredictArgs a) {
  extern __shared__ double sm[];
  double* X = sm;                        // 128 x PB
  double* Y = sm + 128 * MLP_PB;         // 128 x PB
  double* Zp = sm + 256 * MLP_PB;        // 3 x PB: the standardized per-point features g1, g2, g3
  double* Zc = sm + 259 * MLP_PB;        // 30: the standardized per-matrix features (the same for every point)
  const int t = threadIdx.x;
  const int gl = t >> 5;                 // warp: which quarter of a layer's outputs
  const int ps = t & 31;                 // point slot in the block (lane)
  const int64_t p = (int64_t)blockIdx.x * MLP_PB + ps;
  const bool live = p < a.P;
  const double2 z = live ? a.zs[p] : czero();
  if (t < 30) Zc[t] = (a.f30[t] - a.mean33[t]) / a.std33[t];
  if (gl == 0) {
    // ---- features (features.py:129-137): g1, g3 from k_point_features ----
    const double g1 = live ? a.g13[2 * p] : 0.0;
    const double g3 = live ? a.g13[2 * p + 1] : 0.0;
    const double g2 = hypot(z.x - a.eig_mean.x, z.y - a.eig_mean.y);
    Zp[0 * MLP_PB + ps] = (g1 - a.mean33[30]) / a.std33[30];
    Zp[1 * MLP_PB + ps] = (g2 - a.mean33[31]) / a.std33[31];
    Zp[2 * MLP_PB + ps] = (g3 - a.mean33[32]) / a.std33[32];
    // Fourier encoding (network.py:62-75) into X[0..25]
    X[0 * MLP_PB + ps] = z.x;
    X[1 * MLP_PB + ps] = z.y;
    for (int q = 0; q < 6; q++) {
      const double f = (double)(2 << q);
      X[(2 + 4 * q) * MLP_PB + ps] = sin(f * z.x);
      X[(3 + 4 * q) * MLP_PB + ps] = sin(f * z.y);
      X[(4 + 4 * q) * MLP_PB + ps] = cos(f * z.x);
      X[(5 + 4 * q) * MLP_PB + ps] = cos(f * z.y);
    }
  }
  __syncthreads();  // Zc is shared by the block
  const double* P = a.params;
  typedef MlpOff O;
  auto inX = [&](int i) { return X[i * MLP_PB + ps]; };
  auto inY = [&](int i) { return Y[i * MLP_PB + ps]; };
  auto inZ = [&](int i) { return i < 30 ? Zc[i] : Zp[(i - 30) * MLP_PB + ps]; };
  // coordinate path: phi(26) -> 64 -> 64
  dense(P + O::w_c1, P + O::b_c1, 26, 64, inX, Y, ps, gl, true);            // Y[0..63] = h_c1
  __syncthreads();
  dense(P + O::w_c2, P + O::b_c2, 64, 64, inY, X, ps, gl, true);            // X[0..63] = h_c2
  __syncthreads();
  // matrix path: f(33) -> 128 -> 64
  dense(P + O::w_m1, P + O::b_m1, 33, 128, inZ, Y, ps, gl, true);           // Y = h_m1
  __syncthreads();
  dense(P + O::w_m2, P + O::b_m2, 128, 64, inY, X + 64 * MLP_PB, ps, gl, true);  // X[64..127] = h_m2  => X = h3
  __syncthreads();
  dense(P + O::w_t1, P + O::b_t1, 128, 128, inX, Y, ps, gl, true);          // Y = h4
  __syncthreads();
  dense(P + O::w_t2, P + O::b_t2, 128, 128, inY, X, ps, gl, true);          // X = h5 (h3 is dead)
  __syncthreads();
  for (int c = gl; c < 128; c += MLP_GL) X[c * MLP_PB + ps] = Y[c * MLP_PB + ps] + X[c * MLP_PB + ps];  // h6 = h4 + h5
  __syncthreads();
  dense(P + O::w_proj, P + O::b_proj, 128, 64, inX, Y, ps, gl, true);       // Y[0..63] = h7
  __syncthreads();
  if (gl == 0) {
    double logit = 0.0;
    for (int i = 0; i < 64; i++) logit = fma(__ldg(P + O::w_head + i), Y[i * MLP_PB + ps], logit);
    logit += __ldg(P + O::b_head);
    if (live) a.prob[p] = expit_d(logit);
  }
}

// region = dilate(prob >= tau, k) with border clipping; region[g] in {0,1}
__global__ void k_region(const double* __restrict__ prob, int ny, int nx, double tau, int k, uint8_t* region) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)ny * nx) return;
  const int i = (int)(g / nx), j = (int)(g % nx), h = k / 2;
  uint8_t v = 0;
  for (int di = -h; di <= h && !v; di++) {
    const int ii = i + di;
    if (ii < 0 || ii >= ny) continue;
    for (int dj = -h; dj <= h; dj++) {
      const int jj = j + dj;
      if (jj < 0 || jj >= nx) continue;
      if (prob[(int64_t)ii * nx + jj] >= tau) { v = 1; break; }
    }
  }
  region[g] = v;
}

// ---------------------------------------------------------------- ordered stream compaction
// idx = np.flatnonzero(mask) (core.py:204, the order restricted_field evaluates and places points in)
// on the device: (1) per-block counts from warp ballots, (2) one block scans the block counts,
// (3) every block re-ballots its elements and writes each selected grid index at block offset +
// warp offset + lane rank. Blocks of SEL_TPB elements, one element per thread.
constexpr int SEL_TPB = 1024;

__device__ __forceinline__ unsigned sel_block_scan(unsigned bal, unsigned* wsum) {
  // returns this warp's exclusive offset within the block; wsum[32] scratch (shared)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const unsigned v = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0u;
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    wsum[lane] = inc - v;  // exclusive
  }
  __syncthreads();
  return wsum[warp];
}

__global__ void __launch_bounds__(SEL_TPB) k_sel_count(const uint8_t* __restrict__ mask, int64_t N,
                                                        unsigned long long* __restrict__ blk) {
  __shared__ unsigned wsum[32];
  const int64_t g = (int64_t)blockIdx.x * SEL_TPB + threadIdx.x;
  const unsigned bal = __ballot_sync(0xffffffffu, g < N && mask[g] != 0);
  const unsigned off = sel_block_scan(bal, wsum);
  if (threadIdx.x == blockDim.x - 1) blk[blockIdx.x] = off + __popc(bal);
}

// exclusive scan of nblk block counts in place (one block of SEL_TPB threads, chunked); total -> *count
__global__ void __launch_bounds__(SEL_TPB) k_sel_scan(unsigned long long* __restrict__ blk, int64_t nblk,
                                                       int64_t* __restrict__ count) {
  __shared__ unsigned long long part[SEL_TPB];
  unsigned long long carry = 0;
  for (int64_t c0 = 0; c0 < nblk; c0 += SEL_TPB) {
    const int64_t i = c0 + threadIdx.x;
    const unsigned long long v = i < nblk ? blk[i] : 0ull;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < SEL_TPB; o <<= 1) {  // Hillis-Steele inclusive scan
      const unsigned long long y = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0ull;
      __syncthreads();
      part[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nblk) blk[i] = carry + part[threadIdx.x] - v;
    carry += part[SEL_TPB - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = (int64_t)carry;
}

__global__ void __launch_bounds__(SEL_TPB) k_sel_scatter(const uint8_t* __restrict__ mask, int64_t N,
                                                          const unsigned long long* __restrict__ blk,
                                                          int64_t* __restrict__ idx) {
  __shared__ unsigned wsum[32];
  const int64_t g = (int64_t)blockIdx.x * SEL_TPB + threadIdx.x;
  const bool on = g < N && mask[g] != 0;
  const unsigned bal = __ballot_sync(0xffffffffu, on);
  const unsigned off = sel_block_scan(bal, wsum);
  const int lane = threadIdx.x & 31;
  if (on) idx[blk[blockIdx.x] + off + __popc(bal & ((1u << lane) - 1u))] = g;
}

// canonical quiet NaN everywhere (restricted_field's unevaluated points, core.py:203)
__global__ void k_fill_nan(double* __restrict__ out, int64_t N) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < N) out[g] = __longlong_as_double(0x7ff8000000000000ll);
}

// calibrate_threshold's tau loop (pipeline.py:258-259) in one pass: dilate(prob >= tau, k) at a
// pixel is (max of prob over the clipped k x k window) >= tau, so every tau is decided from one
// window maximum. counts[t] += #{truth pixels with wmax >= taus[t]} (warp ballots, then one
// shared-memory add per warp and one global add per block and tau).
__global__ void k_recall(const double* __restrict__ prob, const uint8_t* __restrict__ truth, int ny, int nx, int k,
                         const double* __restrict__ taus, int n_tau, unsigned long long* counts) {
  extern __shared__ unsigned int cnt_s[];
  for (int t = threadIdx.x; t < n_tau; t += blockDim.x) cnt_s[t] = 0;
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool on = false;
  double m = -INFINITY;
  if (g < (int64_t)ny * nx && truth[g]) {
    on = true;
    const int i = (int)(g / nx), j = (int)(g % nx), h = k / 2;
    for (int ii = max(0, i - h); ii <= min(ny - 1, i + h); ii++)
      for (int jj = max(0, j - h); jj <= min(nx - 1, j + h); jj++) m = fmax(m, prob[(int64_t)ii * nx + jj]);
  }
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < n_tau; t++) {
    const unsigned b = __ballot_sync(0xffffffffu, on && m >= taus[t]);
    if (lane == 0 && b) atomicAdd(&cnt_s[t], (unsigned)__popc(b));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tau; t += blockDim.x)
    if (cnt_s[t]) atomicAdd(&counts[t], (unsigned long long)cnt_s[t]);
}

}  // namespace psb
