// Instantiations of the task-mapped tcgen05 GEMM, TMA descriptor encoding and
// the launch path used by bound plans.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "../device/gemm_sm100.cuh"
#include "../host/plan.hpp"

namespace tmb {

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                 CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                 CUtensorMapFloatOOBfill);
using EncodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    taskmap::fail("cannot resolve driver entry point ", name);
  return reinterpret_cast<F>(fn);
}

CUtensorMapDataType tma_dtype(int dt) {
  switch (dt) {
    case TM_F32: return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    case TM_BF16: return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    default: return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  }
}

void check_cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) taskmap::fail(what, " failed with CUresult ", static_cast<int>(r));
}

}  // namespace

int num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) return 148;
  return n;
}

void make_tma_2d3d(void* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box) {
  static EncodeTiled enc = driver_fn<EncodeTiled>("cuTensorMapEncodeTiled");
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  check_cu(enc(reinterpret_cast<CUtensorMap*>(map), tma_dtype(dtype), rank, const_cast<void*>(ptr), d, s, b,
               e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled");
}

void make_tma_im2col(void* map, const void* ptr, int dtype, const uint64_t* dims_cwhn,
                     const uint64_t* strides_bytes, int pad_lo, int upper_corner, int stride,
                     uint32_t channels, uint32_t pixels) {
  static EncodeIm2col enc = driver_fn<EncodeIm2col>("cuTensorMapEncodeIm2col");
  cuuint64_t d[4] = {dims_cwhn[0], dims_cwhn[1], dims_cwhn[2], dims_cwhn[3]};
  cuuint64_t s[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  int lower[2] = {-pad_lo, -pad_lo};
  int upper[2] = {upper_corner, upper_corner};
  cuuint32_t e[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  check_cu(enc(reinterpret_cast<CUtensorMap*>(map), tma_dtype(dtype), 4, const_cast<void*>(ptr), d, s, lower,
               upper, channels, pixels, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeIm2col");
}

namespace {

template <int BN, int STAGES, bool TF32, int CG>
void launch_one(const BoundKernel& k, cudaStream_t s) {
  using Cfg = GemmCfg<BN, STAGES, TF32, CG>;
  auto fn = tm_gemm_kernel<BN, STAGES, TF32, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) != cudaSuccess)
      taskmap::fail("cudaFuncSetAttribute failed: ", cudaGetErrorString(cudaGetLastError()));
    attr_set = true;
  }
  CUtensorMap ta, tb;
  std::memcpy(&ta, k.tma_a, sizeof(ta));
  std::memcpy(&tb, k.tma_b, sizeof(tb));
  if constexpr (CG == 1) {
    fn<<<k.grid, kNumThreads, Cfg::SMEM_BYTES, s>>>(k.p, ta, tb);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(k.grid);
    cfg.blockDim = dim3(kNumThreads);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, fn, k.p, ta, tb) != cudaSuccess)
      taskmap::fail("cudaLaunchKernelEx (cluster) failed: ", cudaGetErrorString(cudaGetLastError()));
  }
}

// stage counts chosen to fill ~200 KB of shared memory (per-CTA stage bytes
// are 16 KB of A + BN/CG rows of B)
constexpr int stages_for(int bn, int cg) {
  const int kb = 16 + bn / cg / 8;  // KB per stage
  return (192 / kb) > 8 ? 8 : (192 / kb);
}

}  // namespace

void launch_bound(const BoundKernel& k, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool deep = k.stages == 0 || k.stages > 2;
#define TMB_CASE(BN)                                                               \
  case BN:                                                                         \
    if (k.tf32) {                                                                  \
      if (deep) launch_one<BN, stages_for(BN, 1), true, 1>(k, s);                  \
      else launch_one<BN, 2, true, 1>(k, s);                                       \
    } else {                                                                       \
      if (deep) launch_one<BN, stages_for(BN, 1), false, 1>(k, s);                 \
      else launch_one<BN, 2, false, 1>(k, s);                                      \
    }                                                                              \
    break;
#define TMB_CASE2(BN)                                                              \
  case BN:                                                                         \
    if (k.tf32) launch_one<BN, stages_for(BN, 2), true, 2>(k, s);                  \
    else launch_one<BN, stages_for(BN, 2), false, 2>(k, s);                        \
    break;
  if (k.cg == 2) {
    switch (k.bn) {
      TMB_CASE2(128)
      TMB_CASE2(256)
      default: taskmap::fail("no 2-CTA kernel instantiated for block_n=", k.bn);
    }
  } else {
    switch (k.bn) {
      TMB_CASE(64)
      TMB_CASE(128)
      TMB_CASE(192)
      TMB_CASE(256)
      default: taskmap::fail("no kernel instantiated for block_n=", k.bn);
    }
  }
#undef TMB_CASE
#undef TMB_CASE2
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) taskmap::fail("kernel launch failed: ", cudaGetErrorString(e));
}

}  // namespace tmb
