// FP64 pipe microbenchmark (development tool): the DFMA rate of (1) chains that reuse two operands
// (a = fma(a, b, c): the library's psb_fp64_peak) and (2) the bisection engine's window update
// W[r][c] -= l[r] conj(w[c]) (15 complex accumulators, 12 distinct multiplier registers: every DFMA
// reads three distinct register pairs), at 4, 8 and 16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++)
#pragma unroll
      for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += a[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_window(double* out, int iters, const double* in) {
  double2 W[6][6];
  double2 l[6], w[6];
#pragma unroll
  for (int r = 0; r < 6; r++) {
    l[r] = make_double2(in[r] * 1e-3, in[r + 6] * 1e-3 + threadIdx.x * 1e-9);
    w[r] = make_double2(in[r + 12] * 1e-3, in[r + 18] * 1e-3);
#pragma unroll
    for (int c = 0; c < 6; c++) W[r][c] = make_double2(1.0 + r, 0.5 + c);
  }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 6; r++) {
#pragma unroll
      for (int c = 0; c < r; c++) {  // 15 complex updates, 4 DFMA each
        W[r][c].x = fma(-l[r].x, w[c].x, W[r][c].x);
        W[r][c].x = fma(-l[r].y, w[c].y, W[r][c].x);
        W[r][c].y = fma(l[r].x, w[c].y, W[r][c].y);
        W[r][c].y = fma(-l[r].y, w[c].x, W[r][c].y);
      }
      W[r][r].x = fma(-l[r].x, w[r].x, fma(-l[r].y, w[r].y, W[r][r].x));  // 6 real diagonal updates, 2 DFMA
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 6; r++)
#pragma unroll
    for (int c = 0; c <= r; c++) s += W[r][c].x + W[r][c].y;
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double *out, *in;
  cudaMalloc(&out, 64);
  cudaMalloc(&in, 64 * 8);
  double h[64];
  for (int i = 0; i < 64; i++) h[i] = 0.37 + 0.01 * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double nominal = p.multiProcessorCount * 64.0 * 2.0 * p.clockRate * 1e3 / 1e12;
  printf("%s: %d SMs, %.0f MHz, nominal FP64 %.1f TF (64 DFMA/clk/SM)\n", p.name, p.multiProcessorCount, p.clockRate / 1e3, nominal);
  for (int wps : {4, 8, 16, 32}) {
    const int blocks = p.multiProcessorCount * wps / 4, threads = 128;
    for (int which = 0; which < 2; which++) {
      const int iters = which == 0 ? 8192 : 4096;
      float best = 1e30f;
      for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        if (which == 0) k_chain<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
        else k_window<<<blocks, threads>>>(out, iters, in);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      const double dfma = (which == 0 ? 64.0 : 72.0) * iters * (double)blocks * threads;
      printf("warps/SM %2d  %-7s %7.2f TF  (%.3f of nominal)\n", wps, which == 0 ? "chain" : "window", 2.0 * dfma / (best * 1e-3) / 1e12,
             2.0 * dfma / (best * 1e-3) / 1e12 / nominal);
    }
  }
  return 0;
}
