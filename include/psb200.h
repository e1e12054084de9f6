/* psb200.h — C ABI of the B200-native sigma_min(zI - A) grid evaluator.
 *
 * The reference (arxiv/paper_2605_04550, package `pseudospec`, pure Python) has no FFI:
 * its boundary is the Python function `pseudospec.core.smin_many` and the two sweeps that
 * call it by module-global name lookup. Each entry point below replaces one of them; the
 * ctypes binding that reroutes the reference onto this library is in INTEGRATION.md and
 * paper_2605_04550_b200/_lib.py.
 *
 *   psb_set_matrix        <- pseudospec/core.py:112-119 require_real_matrix (validation) and the
 *                            per-call `A` argument of smin_many (core.py:141); the band of A is
 *                            uploaded once and reused by every evaluation below
 *   psb_smin_points       <- pseudospec/core.py:141-168 smin_many(A, zs, label, chunk)
 *   psb_smin_grid         <- pseudospec/core.py:177-195 full_pseudospectrum (region == NULL) and
 *                            pseudospec/core.py:198-208 restricted_field (region != NULL)
 *   psb_smin_points_device   same as psb_smin_points on device-resident buffers (no host copies)
 *   psb_engine_split      the engine split's counts on a point set (batch scheduling estimate)
 *   psb_predict_points    <- pseudospec/pipeline.py:169-172 _predict_points (+ features.py:129-164,
 *                            network.py:62-92,153-190)
 *   psb_region_select     <- pseudospec/pipeline.py:227-231 predicted_region (+ core.py:224-231 dilate)
 *   psb_smin_selection    <- pseudospec/pipeline.py:292 restricted_field(A, grid, region) on that region
 *                            (core.py:198-208), consuming the device-side compacted index list
 *   psb_recall_sweep      <- pseudospec/pipeline.py:258-259 the calibrate_threshold tau loop
 *   psb_write_field_csv   <- pseudospec/io.py:92-102 write_field_csv (host only, no handle)
 *   psb_write_mask_csv    <- pseudospec/io.py:105-115 write_mask_csv (host only, no handle)
 *
 * Conventions (mirroring the reference):
 *   - complex values are interleaved (re, im) float64 pairs, i.e. numpy complex128 memory;
 *   - band of A: band[(d + kl) * n + i] = A[i, i + d] for d in [-kl, ku] (diagonal-major);
 *   - results are written to caller-owned host buffers; the library owns device memory;
 *   - sigma is bit-identical for the same (A, z) regardless of batch, order, region or call
 *     (the reference's worker/chunk/restriction invariance, core.py:181-182);
 *   - return codes: PSB_OK, PSB_ERR_PARAM (ParameterError, core.py:18-19), PSB_ERR_NUMERICAL
 *     (NumericalError, core.py:22-23, with *fail_index = first failing point), PSB_ERR_CUDA.
 *   - per-point status codes (optional out array): 0 converged (Lanczos engine), 1 converged
 *     (bisection engine), 2 exactly singular shift (sigma = 0), 3 not converged, 4 non-finite.
 */
#ifndef PSB200_H
#define PSB200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define PSB_OK 0
#define PSB_ERR_PARAM 1
#define PSB_ERR_NUMERICAL 2
#define PSB_ERR_CUDA 3
#define PSB_ERR_IO 4 /* file could not be opened or written (the writers below) */

typedef struct psb_handle psb_handle;

typedef struct {
  double tau;          /* engine split: sigma >= tau*X(z) -> bisection engine (default 1.5e-3 for n < 1000, else 1e-3). X is the
                          scale the bisection engine's G = (zI-A)^H (zI-A) is rounded at: for bands with a
                          diagonal-constant interior T(z), T^2 = (|z-c|+r)^2 + max off-diagonal column
                          norm^2 of A; otherwise S(z) = |z| + sqrt(||A||_1 ||A||_inf) */
  double bis_rtol;     /* bisection stop: (hi-lo) <= bis_rtol*hi on lambda = sigma^2 (default 2e-12) */
  int32_t kmax;        /* Lanczos step cap (0 -> min(3000, max(64, 4n))) */
  int32_t force_engine;/* 0 auto, 1 Lanczos engine only, 2 bisection engine only (testing) */
  int32_t refill;      /* Lanczos engine: refill a warp when this many lanes are idle (0 -> 16) */
  int32_t reserved;
} psb_opts;

typedef struct {
  int64_t n_points;       /* points evaluated in the last call */
  int64_t n_lanczos;      /* points finished by the Lanczos engine */
  int64_t n_bisect;       /* points finished by the bisection engine */
  int64_t lanczos_iters;  /* total Lanczos steps */
  int64_t pd_tests;       /* total LDL^H positive-definiteness tests (incl. classification) */
  double flops_bisect;    /* FP64 flops executed by the bisection engine's launches (classification excluded) */
  double flops_lanczos;   /* FP64 flops executed by the Lanczos engine (LU + steps) */
  double bytes_lanczos;   /* algorithmic HBM bytes moved by the Lanczos engine */
  double ms_bisect;       /* CUDA-event window of the bisection engine: its first launch's start to its last
                             launch's end (the two launches share one work counter) */
  double ms_lanczos;      /* CUDA-event window of the Lanczos kernel */
  double ms_total;        /* CUDA-event time of the whole device pipeline (incl. the list-size read-back) */
  int32_t grid_bisect, grid_lanczos; /* CTAs launched */
  double ms_classify;     /* CUDA-event time of the classification kernel */
  double flops_classify;  /* FP64 flops of the classification kernel (one LDL^H test per point) */
  double ms_fallback;     /* CUDA-event time of the fallback bisection launch (0 when not launched) */
  int32_t launches;       /* kernels launched by the last call (grid shifts, classification, engines, fallback) */
  int32_t reserved;
} psb_stats;

int psb_create(int device, psb_handle** out);
void psb_destroy(psb_handle* h);
const char* psb_last_error(const psb_handle* h);
int psb_version(void);

/* Upload the band of A (complex128, layout above). n >= 2, 0 <= kl, ku < n, kl, ku <= 16. */
int psb_set_matrix(psb_handle* h, const double* band, int32_t n, int32_t kl, int32_t ku);

/* sigma_min(z_p I - A) for P points zs (complex128[P]); sigma (float64[P]) required,
 * iters (int32[P]) and status (int8[P]) optional (may be NULL). */
int psb_smin_points(psb_handle* h, const double* zs, int64_t P, const psb_opts* opts, double* sigma,
                    int32_t* iters, int8_t* status, int64_t* fail_index);

/* Grid point (i, j) is xs[j] + 1j*ys[i] (rows = imaginary axis, core.py:42-43). xs/ys are the
 * host linspace values (passed, not recomputed, so device FMA contraction cannot change them).
 * region (uint8[ny*nx], row-major) selects points; NULL = full grid. sigma (float64[ny*nx]) gets
 * NaN off-region (core.py:203). */
int psb_smin_grid(psb_handle* h, const double* xs, int32_t nx, const double* ys, int32_t ny,
                  const uint8_t* region, const psb_opts* opts, double* sigma, int32_t* iters,
                  int8_t* status, int64_t* fail_index);

/* Device-resident variant: d_zs, d_sigma, d_iters, d_status are device pointers (iters/status
 * may be NULL); stream is a cudaStream_t (NULL = library stream). Synchronous. */
int psb_smin_points_device(psb_handle* h, const double* d_zs, int64_t P, const psb_opts* opts,
                           double* d_sigma, int32_t* d_iters, int8_t* d_status, void* stream);

/* Engine split of a point set, without sigma: the classification test alone (one LDL^H test per point,
 * the same test psb_smin_points starts with), returning how many points the bisection and Lanczos
 * engines would take. Batch scheduling uses it on a coarse subgrid as a matrix's cost estimate (no
 * reference counterpart: the reference's process pool deals fixed row blocks, core.py:186-195). */
int psb_engine_split(psb_handle* h, const double* zs, int64_t P, int64_t* n_bisect, int64_t* n_lanczos);

int psb_get_stats(const psb_handle* h, psb_stats* out);

/* Measured FP64 (DFMA) peak of this device in TFLOP/s: the roofline denominator of the
 * FP64-bound bisection engine (MEASURED_PEAKS.json carries HBM and bf16 only). */
int psb_fp64_peak(psb_handle* h, double* tflops);

/* ---- K2: fused MLP sensitivity predictor + threshold + dilation + compaction ----
 * params: the 16 arrays of network.py:35-52 PARAM_SHAPES concatenated in that order
 * (59,841 float64); mean33/std33: bundle feature statistics; f30: global_features values;
 * eig: eigenvalues (complex128[n_eig]); eig_mean: their numpy mean (complex128, passed so the
 * reduction order is numpy's). Evaluates probabilities at the points zs (complex128[P]) into
 * prob (float64[P]). */
int psb_predict_points(psb_handle* h, const double* params, const double* mean33, const double* std33,
                       const double* f30, const double* eig, int32_t n_eig, const double* eig_mean,
                       const double* zs, int64_t P, double* prob);

/* predicted_region (pipeline.py:227-231): region = dilate(prob >= tau, k) on an (ny, nx) grid,
 * plus the row-major compacted index list of selected points (idx int64[ny*nx] or NULL, *count). The
 * compaction runs on the device and its list stays there as the handle's selection (psb_smin_selection). */
int psb_region_select(psb_handle* h, const double* prob, int32_t ny, int32_t nx, double tau, int32_t k,
                      uint8_t* region, int64_t* idx, int64_t* count);

/* restricted_field (core.py:198-208) on the selection the last psb_region_select left on the device (the
 * row-major index list of its region, compacted by warp ballots and a block scan, np.flatnonzero order,
 * core.py:204): no region upload and no host compaction. Same outputs and bits as psb_smin_grid with that
 * region; PSB_ERR_PARAM when the handle holds no selection for an (ny, nx) grid. */
int psb_smin_selection(psb_handle* h, const double* xs, int32_t nx, const double* ys, int32_t ny,
                       const psb_opts* opts, double* sigma, int32_t* iters, int8_t* status, int64_t* fail_index);

/* calibrate_threshold's inner loop (pipeline.py:258-259, _recall pipeline.py:234-238): for each
 * taus[t], recall[t] = |dilate(prob >= taus[t], k) & truth| / |truth| (1.0 when truth is empty).
 * prob float64[ny*nx]; truth uint8[ny*nx] (the 3x3-dilated exact zone); n_tau <= 4096. */
int psb_recall_sweep(psb_handle* h, const double* prob, const uint8_t* truth, int32_t ny, int32_t nx, int32_t k,
                     const double* taus, int32_t n_tau, double* recall);

/* ---- field / mask export (host only; no handle, no GPU) ----
 * Byte-identical to the reference writers: header line, then one row per grid point in
 * row-major order (i over ys, j over xs), every float as Python's f"{v:.17g}" ("nan", "inf",
 * "-inf" for the special values). log10_sigma is float64[ny*nx] = numpy log10 of the field
 * (computed by the caller, as io.py:97-98); mask is uint8[ny*nx], 0 or 1. nthreads <= 0: all
 * hardware threads. Returns PSB_OK, PSB_ERR_PARAM or PSB_ERR_IO. */
int psb_write_field_csv(const char* path, const double* xs, int64_t nx, const double* ys, int64_t ny,
                        const double* log10_sigma, int32_t nthreads);
int psb_write_mask_csv(const char* path, const double* xs, int64_t nx, const double* ys, int64_t ny,
                       const uint8_t* mask, int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif
