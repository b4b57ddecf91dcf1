// TMA descriptor encoding, helper kernels (filter repack, tuner gates) and the
// launch dispatch of bound plans onto the tm_gemm_kernel instantiations
// (inst_*.cu).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <mutex>
#include <type_traits>

#include "launch_one.cuh"

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
  if (r != CUDA_SUCCESS) taskmap::fail_cuda(what, " failed with CUresult ", static_cast<int>(r));
}

}  // namespace

int num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) return 148;
  return n;
}

void make_tma_2d3d(void* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, int swizzle) {
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
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(map), tma_dtype(dtype), rank, const_cast<void*>(ptr), d, s, b,
                         e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swizzle == 128   ? CU_TENSOR_MAP_SWIZZLE_128B
                         : swizzle == kSwizzle128Atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                         : swizzle == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::string dims_s, str_s, box_s;
    for (int i = 0; i < rank; ++i) {
      dims_s += std::to_string(dims[i]) + " ";
      box_s += std::to_string(box[i]) + " ";
      if (i < rank - 1) str_s += std::to_string(strides_bytes[i]) + " ";
    }
    taskmap::fail_cuda("cuTensorMapEncodeTiled failed with CUresult ", static_cast<int>(r), " (rank ", rank, ", dims ",
                       dims_s, ", strides ", str_s, ", box ", box_s, ", swizzle ", swizzle, ", address ",
                       reinterpret_cast<uintptr_t>(ptr) % 128, " mod 128)");
  }
}

void make_tma_im2col(void* map, const void* ptr, int dtype, const uint64_t* dims_cwhn,
                     const uint64_t* strides_bytes, int pad_lo, int upper_corner, int stride,
                     uint32_t channels, uint32_t pixels, bool swizzle128) {
  static EncodeIm2col enc = driver_fn<EncodeIm2col>("cuTensorMapEncodeIm2col");
  cuuint64_t d[4] = {dims_cwhn[0], dims_cwhn[1], dims_cwhn[2], dims_cwhn[3]};
  cuuint64_t s[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  int lower[2] = {-pad_lo, -pad_lo};
  int upper[2] = {upper_corner, upper_corner};
  cuuint32_t e[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  check_cu(enc(reinterpret_cast<CUtensorMap*>(map), tma_dtype(dtype), 4, const_cast<void*>(ptr), d, s, lower,
               upper, channels, pixels, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeIm2col");
}

// Filter repack into the GEMM's K order (bind-time; see fusion.cpp): out[f][k]
// bf16 or fp16 (the MMA operand format), K-major, row length kp (multiple of 8),
// zero where the K order pads.
template <class T>
__global__ void pack_filter_kernel(ConvGeom g, int kp, T* out) {
  const int64_t n = static_cast<int64_t>(g.f) * kp;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int f = static_cast<int>(i / kp), k = static_cast<int>(i % kp);
    int c, fh, fw;
    if (g.korder == 0) {
      c = k / (g.kh * g.kw);
      fh = (k / g.kw) % g.kh;
      fw = k % g.kw;
    } else {
      const int tap = k / g.cpad;
      c = k % g.cpad;
      fh = tap / g.kw;
      fw = tap % g.kw;
    }
    float v = 0.f;
    if (c < g.c && fh < g.kh) {
      const int64_t idx = f * g.sw[0] + c * g.sw[1] + fh * g.sw[2] + fw * g.sw[3];
      v = g.w_dtype == DT_F32    ? reinterpret_cast<const float*>(g.wt)[idx]
          : g.w_dtype == DT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(g.wt)[idx])
                                 : __half2float(reinterpret_cast<const __half*>(g.wt)[idx]);
    }
    if constexpr (sizeof(T) == 2 && std::is_same<T, __half>::value) out[i] = __float2half_rn(v);
    else out[i] = __float2bfloat16_rn(v);
  }
}

void pack_filter(const ConvGeom& g, int kp, void* out, int out_dtype) {
  if (out_dtype == TM_F16) pack_filter_kernel<<<148, 256>>>(g, kp, static_cast<__half*>(out));
  else pack_filter_kernel<<<148, 256>>>(g, kp, static_cast<__nv_bfloat16*>(out));
  if (cudaDeviceSynchronize() != cudaSuccess) taskmap::fail_cuda("filter repack kernel failed: ", cudaGetErrorString(cudaGetLastError()));
}

__global__ void mismatch_kernel(const uint4* a, const uint4* b, size_t n16, const uint8_t* ta, const uint8_t* tb,
                                size_t tail, unsigned long long* out) {
  unsigned long long bad = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    bad += (x.x != y.x) + (x.y != y.y) + (x.z != y.z) + (x.w != y.w);
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) bad += ta[threadIdx.x] != tb[threadIdx.x];
  if (bad) atomicAdd(out, bad);
}

// Bitwise comparison of two device byte ranges (the tuner's correctness gate).
unsigned long long device_mismatch(const void* a, const void* b, size_t bytes, void* stream) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) taskmap::fail_cuda("cudaMalloc failed in device_mismatch");
  cudaMemsetAsync(d, 0, 8, static_cast<cudaStream_t>(stream));
  const bool aligned = (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (reinterpret_cast<uintptr_t>(b) % 16 == 0);
  const size_t n16 = aligned ? bytes / 16 : 0;
  const size_t tail = bytes - n16 * 16;
  if (tail > 1024) taskmap::fail("device_mismatch: unaligned ranges are limited to 1 KB");
  mismatch_kernel<<<296, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(a), static_cast<const uint4*>(b), n16, static_cast<const uint8_t*>(a) + n16 * 16,
      static_cast<const uint8_t*>(b) + n16 * 16, tail, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  cudaFree(d);
  return h;
}

__global__ void max_rel_error_kernel(const void* a, const void* b, size_t n, int dtype, unsigned int* out) {
  float worst = 0.f;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    float x, y;
    if (dtype == DT_F32) {
      x = static_cast<const float*>(a)[i];
      y = static_cast<const float*>(b)[i];
    } else if (dtype == DT_BF16) {
      x = __bfloat162float(static_cast<const __nv_bfloat16*>(a)[i]);
      y = __bfloat162float(static_cast<const __nv_bfloat16*>(b)[i]);
    } else {
      x = __half2float(static_cast<const __half*>(a)[i]);
      y = __half2float(static_cast<const __half*>(b)[i]);
    }
    const float e = (x == y) ? 0.f : fabsf(x - y) / fmaxf(1.f, fabsf(y));  // tensor.cpp:71-86 metric
    worst = fmaxf(worst, e != e ? 3.0e38f : e);                          // NaN counts as failure
  }
  atomicMax(out, __float_as_uint(worst));  // non-negative floats order like their bits
}

// max |a-b| / max(1, |b|) over n elements of dtype (the tuner's tolerance gate).
float device_max_rel_error(const void* a, const void* b, size_t n, int dtype, void* stream) {
  unsigned int* d = nullptr;
  if (cudaMalloc(&d, 4) != cudaSuccess) taskmap::fail_cuda("cudaMalloc failed in device_max_rel_error");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(d, 0, 4, s);
  max_rel_error_kernel<<<296, 1024, 0, s>>>(a, b, n, dtype, d);
  unsigned int h = 0;
  cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFree(d);
  float f;
  std::memcpy(&f, &h, 4);
  return f;
}

int kernel_stages(const BoundKernel& k) {
  if (k.simt) return 2;
  if (k.cg == 2) return k.tf32 || k.generic ? stages_for(k.bn, 2) : stages_for(k.bn, 2, false);
  const bool deep = k.stages == 0 || k.stages > 2;
  if (!deep) return 2;
  return k.tf32 ? stages_for(k.bn, 1) : stages_for(k.bn, 1, k.generic != 0);
}

void launch_bound(const BoundKernel& k, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  bool ok;
  if (k.simt) {
    launch_simt(k, stream);
    ok = true;
  } else if (k.rule) {
    if (k.rfn) launch_rule_compiled(k.rfn, k.rp, k.rgrid, k.rblock, stream);
    else launch_rule(k.rj, k.rule_threads, k.grid, stream);
    ok = true;
  } else if (k.rowband == 2) ok = launch_halo(k, s);
  else if (k.rowband) ok = launch_rowband(k, s);
  else if (k.cg == 2) ok = launch_cg2(k, s);
  else if (k.tf32) ok = launch_cg1_generic_tf32(k, s);
  else if (!k.generic) ok = launch_cg1_fast(k, s);
  else ok = launch_cg1_generic_bf16(k, s);
  if (!ok) taskmap::fail("no kernel instantiated for block_n=", k.bn, " cta_group=", k.cg);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) taskmap::fail_cuda("kernel launch failed: ", cudaGetErrorString(e));
}

}  // namespace tmb
