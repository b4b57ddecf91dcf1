// Instantiations and launcher of the halo implicit-GEMM conv kernel (conv_halo.cuh).
#include "../device/conv_halo.cuh"
#include "launch_one.cuh"

namespace tmb {

int halo_smem(int band_bytes, int stage_bytes, int stages, int bn, int nbands) {
  return HbLayout(band_bytes, stage_bytes, stages, bn, nbands).total;
}

template <int BN, int NB>
void launch_hb(const BoundKernel& k, cudaStream_t s) {
  auto fn = tm_halo_kernel<BN, NB>;
  static std::once_flag attr_once[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    taskmap::fail_cuda("cudaGetDevice failed or device index out of range");
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[dev], [&] {
    attr_err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  });
  if (attr_err != cudaSuccess) taskmap::fail_cuda("cudaFuncSetAttribute failed: ", cudaGetErrorString(attr_err));
  CUtensorMap tx, tw;
  std::memcpy(&tx, k.tma_a, sizeof(tx));
  std::memcpy(&tw, k.tma_b, sizeof(tw));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(k.grid);
  cfg.blockDim = dim3(kHbThreads);
  cfg.dynamicSmemBytes = k.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  static const bool pdl = std::getenv("TMB_NO_PDL") == nullptr;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (k.p.hb_mc == 2) {  // CTA pairs sharing the filter stages (multicast)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, fn, k.p, tx, tw) != cudaSuccess)
    taskmap::fail_cuda("cudaLaunchKernelEx failed: ", cudaGetErrorString(cudaGetLastError()));
}

bool launch_halo(const BoundKernel& k, cudaStream_t s) {
  const int nb = k.p.rb_steps;
  if (k.bn == 64 && nb == 4) { launch_hb<64, 4>(k, s); return true; }
  if (k.bn == 64 && nb == 2) { launch_hb<64, 2>(k, s); return true; }
  if (k.bn == 64 && nb == 1) { launch_hb<64, 1>(k, s); return true; }
  if (k.bn == 128 && nb == 2) { launch_hb<128, 2>(k, s); return true; }
  if (k.bn == 128 && nb == 1) { launch_hb<128, 1>(k, s); return true; }
  return false;
}

}  // namespace tmb
