// Instantiations and launcher of the row-band small-C conv kernel
// (conv_rowband.cuh), plus its bind-time filter-image repack.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "../device/conv_rowband.cuh"
#include "launch_one.cuh"

namespace tmb {

int rowband_smem(int rows, int rowb, int bbytes, int bn) { return RbLayout(rows, rowb, bbytes, bn).total; }

template <class T>
__global__ void pack_rowband_kernel(ConvGeom g, int cpad, int shift, int steps, int bn, T* out) {
  const int64_t n = static_cast<int64_t>(g.kh) * steps * bn * 16;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    // i = ((((fh * steps + t) * (bn/8) + fgrp) * 2 + khalf) * 8 + frow) * 8 + e
    const int e = static_cast<int>(i % 8), frow = static_cast<int>((i / 8) % 8), khalf = static_cast<int>((i / 64) % 2);
    const int64_t rest = i / 128;
    const int fgrp = static_cast<int>(rest % (bn / 8));
    const int64_t st = rest / (bn / 8);
    const int t = static_cast<int>(st % steps), fh = static_cast<int>(st / steps);
    const int f = fgrp * 8 + frow, k = t * 16 + khalf * 8 + e;
    const int c = k % cpad, fw = k / cpad - shift;
    float v = 0.f;
    if (f < g.f && c < g.c && fw >= 0 && fw < g.kw) {
      const int64_t idx = f * g.sw[0] + c * g.sw[1] + fh * g.sw[2] + fw * g.sw[3];
      v = g.w_dtype == DT_F32    ? reinterpret_cast<const float*>(g.wt)[idx]
          : g.w_dtype == DT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(g.wt)[idx])
                                 : __half2float(reinterpret_cast<const __half*>(g.wt)[idx]);
    }
    if constexpr (std::is_same<T, __half>::value) out[i] = __float2half_rn(v);
    else out[i] = __float2bfloat16_rn(v);
  }
}

void pack_rowband_filter(const ConvGeom& g, int cpad, int shift, int steps, int bn, void* out, int out_dtype) {
  if (out_dtype == TM_F16) pack_rowband_kernel<<<148, 256>>>(g, cpad, shift, steps, bn, static_cast<__half*>(out));
  else pack_rowband_kernel<<<148, 256>>>(g, cpad, shift, steps, bn, static_cast<__nv_bfloat16*>(out));
  if (cudaDeviceSynchronize() != cudaSuccess)
    taskmap::fail_cuda("row-band filter repack failed: ", cudaGetErrorString(cudaGetLastError()));
}

template <int BN, int KH, int STEPS>
void launch_rb(const BoundKernel& k, cudaStream_t s) {
  auto fn = tm_rowband_kernel<BN, KH, STEPS>;
  static std::once_flag attr_once[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    taskmap::fail_cuda("cudaGetDevice failed or device index out of range");
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[dev], [&] {
    attr_err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  });
  if (attr_err != cudaSuccess) taskmap::fail_cuda("cudaFuncSetAttribute failed: ", cudaGetErrorString(attr_err));
  CUtensorMap tx, tx0, tc;
  std::memcpy(&tx, k.tma_a, sizeof(tx));
  std::memcpy(&tx0, k.tma_b, sizeof(tx0));  // the first band's (shorter) staged-row box
  std::memcpy(&tc, k.tma_c, sizeof(tc));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(k.grid);
  cfg.blockDim = dim3(kRbThreads);
  cfg.dynamicSmemBytes = k.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  int na = 0;
  static const bool pdl = std::getenv("TMB_NO_PDL") == nullptr;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, fn, k.p, tx, tx0, tc) != cudaSuccess)
    taskmap::fail_cuda("cudaLaunchKernelEx failed: ", cudaGetErrorString(cudaGetLastError()));
}

bool launch_rowband(const BoundKernel& k, cudaStream_t s) {
  const bool stem = k.p.conv.kh == 7 && k.p.rb_steps == 2;  // 7x7 filter rows, 8-byte pixels (ResNet stem)
  switch (k.bn) {
    case 64: if (stem) launch_rb<64, 7, 2>(k, s); else launch_rb<64, 0, 0>(k, s); return true;
    case 128: launch_rb<128, 0, 0>(k, s); return true;
    case 256: launch_rb<256, 0, 0>(k, s); return true;
  }
  return false;
}

}  // namespace tmb
