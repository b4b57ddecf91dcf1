// Instantiations: single-CTA tiles, compact fast path (TMA loaders + canonical epilogue), bf16.
#include "launch_one.cuh"

namespace tmb {
bool launch_cg1_fast(const BoundKernel& k, cudaStream_t s) {
  const bool deep = k.stages == 0 || k.stages > 2;
  switch (k.bn) {
#define TMB_V(BN) \
  case BN: if (deep) launch_one<BN, stages_for(BN, 1, false), false, 1, false>(k, s); else launch_one<BN, 2, false, 1, false>(k, s); return true;
    TMB_V(64) TMB_V(96) TMB_V(128) TMB_V(192) TMB_V(256)
#undef TMB_V
  }
  return false;
}
}  // namespace tmb
