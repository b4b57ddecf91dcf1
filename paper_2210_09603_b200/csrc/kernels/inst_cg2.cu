// Instantiations: CTA-pair tiles (tcgen05.mma.cta_group::2), TMA loaders only.
#include "launch_one.cuh"

namespace tmb {
bool launch_cg2(const BoundKernel& k, cudaStream_t s) {
  switch (k.bn) {
#define TMB_V(BN)                                                                 \
  case BN:                                                                        \
    if (k.tf32) launch_one<BN, stages_for(BN, 2), true, 2, true>(k, s);           \
    else if (k.generic) launch_one<BN, stages_for(BN, 2), false, 2, true>(k, s);  \
    else launch_one<BN, stages_for(BN, 2, false), false, 2, false>(k, s);                \
    return true;
    TMB_V(64) TMB_V(128) TMB_V(256)
#undef TMB_V
  }
  return false;
}
}  // namespace tmb
