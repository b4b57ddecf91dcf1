// Launch helper shared by the instantiation units (inst_*.cu): one
// tm_gemm_kernel specialisation, optionally as a CTA-pair cluster launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../device/gemm_sm100.cuh"
#include "../host/plan.hpp"

namespace tmb {

constexpr int kMaxDevices = 64;

template <int BN, int STAGES, bool TF32, int CG, bool GENERIC>
void launch_one(const BoundKernel& k, cudaStream_t s) {
  using Cfg = GemmCfg<BN, STAGES, TF32, CG, GENERIC>;
  static_assert(Cfg::SMEM_BYTES <= kMaxSmem, "shared memory budget");
  auto fn = tm_gemm_kernel<BN, STAGES, TF32, CG, GENERIC>;
  // the dynamic shared-memory opt-in is a per-device (per-context) attribute:
  // set once per device this process launches on, thread-safely
  static std::once_flag attr_once[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    taskmap::fail_cuda("cudaGetDevice failed or device index out of range");
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[dev], [&] {
    attr_err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) taskmap::fail_cuda("cudaFuncSetAttribute failed: ", cudaGetErrorString(attr_err));
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
  // Programmatic dependent launch (default on; TMB_NO_PDL=1 disables): this grid's
  // prologue (barrier init, TMEM allocation, descriptor prefetch, tile list)
  // overlaps the previous kernel's tail; the kernel waits with
  // griddepcontrol.wait before touching global memory.  (Round 1 had it opt-in
  // after a rare cross-kernel hang; with the producer tail and owner-only ring
  // waits in gemm_sm100.cuh 5000-sweep stress runs are clean with it on.)
  static const bool pdl = std::getenv("TMB_NO_PDL") == nullptr;
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
    taskmap::fail_cuda("cudaLaunchKernelEx failed: ", cudaGetErrorString(cudaGetLastError()));
}

// per-unit dispatchers (defined in inst_*.cu); return false if no variant matches
bool launch_cg1_generic_bf16(const BoundKernel& k, cudaStream_t s);
bool launch_cg1_generic_tf32(const BoundKernel& k, cudaStream_t s);
bool launch_cg1_fast(const BoundKernel& k, cudaStream_t s);
bool launch_cg2(const BoundKernel& k, cudaStream_t s);
bool launch_rowband(const BoundKernel& k, cudaStream_t s);
bool launch_halo(const BoundKernel& k, cudaStream_t s);

}  // namespace tmb
