// Launch helper shared by the instantiation units (inst_*.cu): one
// tm_gemm_kernel specialisation, optionally as a CTA-pair cluster launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "../device/gemm_sm100.cuh"
#include "../host/plan.hpp"

namespace tmb {

template <int BN, int STAGES, bool TF32, int CG, bool GENERIC>
void launch_one(const BoundKernel& k, cudaStream_t s) {
  using Cfg = GemmCfg<BN, STAGES, TF32, CG, GENERIC>;
  static_assert(Cfg::SMEM_BYTES <= kMaxSmem, "shared memory budget");
  auto fn = tm_gemm_kernel<BN, STAGES, TF32, CG, GENERIC>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) != cudaSuccess)
      taskmap::fail("cudaFuncSetAttribute failed: ", cudaGetErrorString(cudaGetLastError()));
    attr_set = true;
  }
  CUtensorMap ta, tb, tc;
  std::memcpy(&ta, k.tma_a, sizeof(ta));
  std::memcpy(&tb, k.tma_b, sizeof(tb));
  std::memcpy(&tc, k.tma_c, sizeof(tc));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(k.grid);
  cfg.blockDim = dim3(Roles<GENERIC>::kThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // programmatic dependent launch: this grid's prologue overlaps the previous
  // kernel's tail (the kernel waits with griddepcontrol.wait before touching memory)
  // Programmatic dependent launch is opt-in (TMB_PDL=1): replaying the 57-launch
  // sweep graph with it hung once in ~1400 sweeps (scripts/sweep_stress.py), and
  // 3000 sweeps without it ran clean.  It is worth ~8% of the sweep, so it stays
  // available for investigation.
  static const bool pdl = std::getenv("TMB_PDL") != nullptr;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if constexpr (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, fn, k.p, ta, tb, tc) != cudaSuccess)
    taskmap::fail("cudaLaunchKernelEx failed: ", cudaGetErrorString(cudaGetLastError()));
}

// per-unit dispatchers (defined in inst_*.cu); return false if no variant matches
bool launch_cg1_generic_bf16(const BoundKernel& k, cudaStream_t s);
bool launch_cg1_generic_tf32(const BoundKernel& k, cudaStream_t s);
bool launch_cg1_fast(const BoundKernel& k, cudaStream_t s);
bool launch_cg2(const BoundKernel& k, cudaStream_t s);

}  // namespace tmb
