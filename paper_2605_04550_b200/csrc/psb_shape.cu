// psb_shape.cu — one band shape's kernel set (see psb_dispatch.cuh). Compiled once per exact
// shape with -DPSB_KL=.. -DPSB_KU=.. -DPSB_NP=.. -DPSB_G=.., and once with -DPSB_DYN for the
// runtime-shape instantiation (any band up to 16/16).
#include "psb_dispatch.cuh"

namespace psb {
namespace {

#ifdef PSB_DYN
const KPair kSet = {-1, -1, &k_bisect<16, 16, true, 1, 1, false>, &k_bisect<16, 16, true, 1, 1, false>,
                    &k_bisect<16, 16, true, 1, 1, false>, &k_bisect<16, 16, true, 1, 1, false>,
                    &k_bisect<16, 16, true, 1, 1, false>, &k_bisect<16, 16, true, 1, 1, false>,
                    &k_lanczos<16, 16, true, 2>, 0, 1, 1, 0};
#else
constexpr int D = RingDepth<PSB_KL, PSB_KU>::D;
static_assert(PSB_NP * PSB_G == 2, "the pair variant (NP = 1, G = 2) must probe the same K = 2 shifts");
const KPair kSet = {PSB_KL, PSB_KU, &k_bisect<PSB_KL, PSB_KU, false, 1, 1, false>,
                    &k_bisect<PSB_KL, PSB_KU, false, PSB_NP, PSB_G, false>,
                    &k_bisect<PSB_KL, PSB_KU, false, 1, 1, true>,
                    &k_bisect<PSB_KL, PSB_KU, false, PSB_NP, PSB_G, true>,
                    &k_bisect<PSB_KL, PSB_KU, false, 1, 2, false>,
                    &k_bisect<PSB_KL, PSB_KU, false, 1, 2, true>, &k_lanczos<PSB_KL, PSB_KU, false, D>,
                    Ring<PSB_KL, PSB_KU, D>::BYTES + LUS<PSB_KL, PSB_KU>::BYTES, PSB_NP, PSB_G,
                    BisRow<PSB_KL, PSB_KU>::BYTES};
#endif

struct Registrar {
  Registrar() { register_shape(kSet); }
} registrar;

}  // namespace
}  // namespace psb
