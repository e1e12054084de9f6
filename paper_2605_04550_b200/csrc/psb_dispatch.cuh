// psb_dispatch.cuh — per-band-shape kernel sets and their registry.
//
// Each exact band shape (kl, ku) is compiled in its own translation unit (psb_shape.cu built once
// per shape with -DPSB_KL/-DPSB_KU/-DPSB_NP/-DPSB_G, or -DPSB_DYN for the runtime-shape set), so
// the library builds in parallel. Every unit registers its kernel set at load time; the C ABI picks
// the exact-shape set for the matrix's band or falls back to the runtime-shape one.
#pragma once
#include "psb_engines.cuh"

namespace psb {

typedef void (*bis_fn)(BisArgs);
typedef void (*lan_fn)(LanArgs);
// b: classification (NP = 1); bm: multisection (NP probes per thread); l: Lanczos engine.
// bt / bmt: the same for bands with a diagonal-constant interior (TZ row loop).
// bm2 / bmt2: the pair variant, the same K = 2 probes per round on two lanes (NP = 1, G = 2). Both
// variants test the same shifts with the same arithmetic, so they return the same bits and the host
// may pick either per launch (the pair for short lists, where each thread holds about one point).
// np, g: the wide variant's split. lsmem: engine-L shared memory per warp (sweep ring + LU stage). kl = -1: runtime-shape set.
// bsmem: shared-memory row stages per warp of the general-band (non-TZ) bisection kernels (BisRow).
struct KPair { int kl, ku; bis_fn b, bm, bt, bmt, bm2, bmt2; lan_fn l; int lsmem; int np, g; int bsmem; };

void register_shape(const KPair& k);  // defined in psb_capi.cu

}  // namespace psb
