// fp32 CUDA-core GEMM scheduled with the paper's task mappings (K4a).
//
// Block tile 128x128x8 (or 128x64x8 when the 128x128 grid under-fills the SMs), 256 threads.  Every index in this kernel comes from a
// task mapping (taskmap.cuh, the algebra of proj/src/mapping.cpp):
//   compute:  spatial(4,2) * repeat(2,2) * spatial(4,8) * repeat(4,4)
//             (Hidet's CUDA-core matmul mapping): 256
//             workers x 64 outputs each over the 128x128 tile;
//   A load:   repeat(4,1) * spatial(32,8) over the 128x8 A tile (Fig. 5 style
//             cooperative load);
//   B load:   repeat(1,4) * spatial(8,32) over the 8x128 B tile.
// Double buffering is Fig. 6's register-staged form: the
// next K-tile is loaded into registers while the current one is computed from
// shared memory, then committed to the other buffer.  Loads are predicated
// (zero outside the matrix), so any M, N, K works.  The epilogue
// runs the fused op program element by element, exact fp32 throughout.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../device/gemm_params.h"
#include "../device/taskmap.cuh"
#include "../host/plan.hpp"

namespace tmb {
namespace {

// BN = 128: the paper's mapping; BN = 64 (twice the CTAs for small grids, e.g.
// config 1's 1024^2 output = 64 tiles of 128^2 on 148 SMs): one repeat atom
// halved along N.
// K-tile depth TBK = 8 (the paper's) or 16: the loads repeat TBK/8 times along k.
template <int BN, int TBK>
struct SimtMaps;
template <int TBK>
struct SimtMaps<128, TBK> {
  using Compute = tm::Chain<tm::Spatial<4, 2>, tm::Repeat<2, 2>, tm::Spatial<4, 8>, tm::Repeat<4, 4>>;
  using LoadA = tm::Compose<tm::Repeat<4, TBK / 8>, tm::Spatial<32, 8>>;
  using LoadB = tm::Compose<tm::Repeat<TBK / 8, 4>, tm::Spatial<8, 32>>;
};
template <int TBK>
struct SimtMaps<64, TBK> {
  using Compute = tm::Chain<tm::Spatial<4, 2>, tm::Repeat<2, 1>, tm::Spatial<4, 8>, tm::Repeat<4, 4>>;
  using LoadA = tm::Compose<tm::Repeat<4, TBK / 8>, tm::Spatial<32, 8>>;
  using LoadB = tm::Compose<tm::Repeat<TBK / 8, 2>, tm::Spatial<8, 32>>;
};
using ComputeMap = SimtMaps<128, 8>::Compute;
using LoadA = SimtMaps<128, 8>::LoadA;
using LoadB = SimtMaps<128, 8>::LoadB;
static_assert(ComputeMap::workers == 256 && ComputeMap::tasks == 64, "CUDA-core mapping shape");
static_assert(ComputeMap::dim(0) == 128 && ComputeMap::dim(1) == 128, "covers the 128x128 tile");
static_assert(SimtMaps<64, 8>::Compute::workers == 256 && SimtMaps<64, 8>::Compute::dim(1) == 64, "128x64 tile");
static_assert(SimtMaps<128, 16>::LoadA::dim(1) == 16 && SimtMaps<128, 16>::LoadB::dim(0) == 16, "16-deep K tile");
static_assert(LoadA::workers == 256 && LoadA::dim(0) == 128 && LoadA::dim(1) == 8, "A tile 128x8");
static_assert(LoadB::workers == 256 && LoadB::dim(0) == 8 && LoadB::dim(1) == 128, "B tile 8x128");

constexpr int TBM = 128;

__device__ __forceinline__ float ld_elem(const void* base, int64_t idx, int32_t dt) {
  if (dt == DT_F32) return __ldg(reinterpret_cast<const float*>(base) + idx);
  if (dt == DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
  return __half2float(reinterpret_cast<const __half*>(base)[idx]);
}

// operand element with its arithmetic prologue applied (fuse_prologue)
__device__ __forceinline__ float ld_operand(const Strided& s, int64_t idx) {
  float v = ld_elem(s.ptr, idx, s.dtype);
  for (int i = 0; i < s.n_pre; ++i) {
    const float c = s.pre[i].c;
    switch (s.pre[i].kind) {
      case EPI_ADD_C: v = v + c; break;
      case EPI_SUB_C: v = v - c; break;
      case EPI_RSUB_C: v = c - v; break;
      case EPI_MUL_C: v = v * c; break;
      case EPI_DIV_C: v = v / c; break;
      case EPI_RDIV_C: v = c / v; break;
      case EPI_MAX_C: v = fmaxf(v, c); break;
      case EPI_MIN_C: v = fminf(v, c); break;
      case EPI_RELU: v = fmaxf(v, 0.f); break;
      case EPI_NEG: v = -v; break;
      case EPI_EXP: v = expf(v); break;
      case EPI_SQRT: v = sqrtf(v); break;
      case EPI_GELU_TANH: {
        const float u = 0.7978845608028654f * (v + 0.044715f * v * v * v);
        v = 0.5f * v * (1.0f + (1.0f - 2.0f / (expf(2.0f * u) + 1.0f)));
        break;
      }
      default: break;
    }
  }
  return v;
}

__device__ __forceinline__ int64_t row_part(int64_t P, int64_t hi, int64_t lo, int64_t r) {
  return (r / P) * hi + (r % P) * lo;
}

__device__ __forceinline__ float side_val(const EpiOp& op, int64_t r, int64_t c, int64_t b) {
  const int64_t idx = row_part(op.a.P, op.a.s_hi, op.a.s_lo, r) + c * op.a.s_col + b * op.a.s_batch + op.a.offset;
  return ld_elem(op.ptr, idx, op.dtype);
}

// Element-wise form of the fused epilogue program (same op semantics as the
// tcgen05 kernel's interpreter).
__device__ float epilogue1(const GemmParams& p, float v, int64_t r, int64_t c, int64_t b) {
  for (int o = 0; o < p.n_ops; ++o) {
    const EpiOp& op = p.ops[o];
    const float s = (op.kind >= EPI_ADD_T && op.kind <= EPI_MIN_T) ? side_val(op, r, c, b) : op.c;
    switch (op.kind) {
      case EPI_ADD_C: case EPI_ADD_T: v = v + s; break;
      case EPI_SUB_C: case EPI_SUB_T: v = v - s; break;
      case EPI_RSUB_C: case EPI_RSUB_T: v = s - v; break;
      case EPI_MUL_C: case EPI_MUL_T: v = v * s; break;
      case EPI_DIV_C: case EPI_DIV_T: v = v / s; break;
      case EPI_RDIV_C: case EPI_RDIV_T: v = s / v; break;
      case EPI_MAX_C: case EPI_MAX_T: v = fmaxf(v, s); break;
      case EPI_MIN_C: case EPI_MIN_T: v = fminf(v, s); break;
      case EPI_RELU: v = fmaxf(v, 0.f); break;
      case EPI_GELU_TANH: {
        const float u = 0.7978845608028654f * (v + 0.044715f * v * v * v);
        v = 0.5f * v * (1.0f + (1.0f - 2.0f / (expf(2.0f * u) + 1.0f)));
        break;
      }
      case EPI_EXP: v = expf(v); break;
      case EPI_SQRT: v = sqrtf(v); break;
      case EPI_NEG: v = -v; break;
      case EPI_ROUND_BF16: v = __bfloat162float(__float2bfloat16_rn(v)); break;
      default: break;
    }
  }
  return v;
}

template <int TBN, int TBK>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const __grid_constant__ GemmParams p) {
  using CMap = typename SimtMaps<TBN, TBK>::Compute;
  using AMap = typename SimtMaps<TBN, TBK>::LoadA;
  using BMap = typename SimtMaps<TBN, TBK>::LoadB;
  constexpr int CN = TBN / 16;  // columns per thread (4 per repeat(4,4) block, TBN / 64 blocks)
  __shared__ __align__(16) float As[2][TBK][TBM + 4];  // A tile stored k-major (transposed) for fragment reads
  __shared__ __align__(16) float Bs[2][TBK][TBN + 4];
  const uint32_t t = threadIdx.x;
  const int tiles_mn = p.tiles_m * p.tiles_n;
  const int b = static_cast<int>(blockIdx.x / tiles_mn);
  const int tm_ = static_cast<int>((blockIdx.x % tiles_mn) / p.tiles_n), tn = static_cast<int>(blockIdx.x % p.tiles_n);
  const int64_t m0 = int64_t(tm_) * TBM, n0 = int64_t(tn) * TBN;
  const Strided& A = p.a;
  const Strided& B = p.b;
  // Each thread's load tasks touch fixed rows (A) / columns (B) and fixed k offsets
  // inside a K-tile: their element offsets are computed once, and a K-tile only
  // adds k0 * s_k (no per-element div/mod of the strided address map).
  int64_t abase[AMap::tasks], bbase[BMap::tasks];
  int ak[AMap::tasks], bk[BMap::tasks];
  bool aok[AMap::tasks], bok[BMap::tasks];
#pragma unroll
  for (uint32_t i = 0; i < AMap::tasks; ++i) {
    int c[2];
    AMap::task(t, i, c);  // (m, k) within the tile
    const int64_t m = m0 + c[0];
    aok[i] = m < p.M;
    abase[i] = (aok[i] ? row_part(A.P, A.s_hi, A.s_lo, m) : 0) + c[1] * A.s_k + b * A.s_batch + A.offset;
    ak[i] = c[1];
  }
#pragma unroll
  for (uint32_t i = 0; i < BMap::tasks; ++i) {
    int c[2];
    BMap::task(t, i, c);  // (k, n) within the tile
    const int64_t n = n0 + c[1];
    bok[i] = n < p.N;
    bbase[i] = (bok[i] ? row_part(B.P, B.s_hi, B.s_lo, n) : 0) + c[0] * B.s_k + b * B.s_batch + B.offset;
    bk[i] = c[0];
  }
  const bool plain = A.n_pre == 0 && B.n_pre == 0 && A.dtype == DT_F32 && B.dtype == DT_F32;
  float ra[AMap::tasks], rb[BMap::tasks];
  auto load_tiles = [&](int k0) {
    const int64_t ka = int64_t(k0) * A.s_k, kb = int64_t(k0) * B.s_k;
#pragma unroll
    for (uint32_t i = 0; i < AMap::tasks; ++i) {
      const bool ok = aok[i] && k0 + ak[i] < p.K;
      ra[i] = !ok ? 0.f : plain ? __ldg(reinterpret_cast<const float*>(A.ptr) + abase[i] + ka) : ld_operand(A, abase[i] + ka);
    }
#pragma unroll
    for (uint32_t i = 0; i < BMap::tasks; ++i) {
      const bool ok = bok[i] && k0 + bk[i] < p.K;
      rb[i] = !ok ? 0.f : plain ? __ldg(reinterpret_cast<const float*>(B.ptr) + bbase[i] + kb) : ld_operand(B, bbase[i] + kb);
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (uint32_t i = 0; i < AMap::tasks; ++i) {
      int c[2];
      AMap::task(t, i, c);
      As[buf][c[1]][c[0]] = ra[i];
    }
#pragma unroll
    for (uint32_t i = 0; i < BMap::tasks; ++i) {
      int c[2];
      BMap::task(t, i, c);
      Bs[buf][c[0]][c[1]] = rb[i];
    }
  };

  // this thread's rows / columns under the compute mapping: the innermost
  // repeat(4,4) atom makes each group of 4 consecutive, so fragments are read
  // as float4 (rows: 2 groups; columns: TBN/64 groups)
  int rows[8], cols[CN];
#pragma unroll
  for (int r1 = 0; r1 < 2; ++r1)
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      int c[2];
      CMap::task(t, (r1 * (TBN / 64)) * 16 + r2 * 4, c);
      rows[r1 * 4 + r2] = c[0];
    }
#pragma unroll
  for (int j = 0; j < CN; ++j) {
    int c[2];
    CMap::task(t, (j / 4) * 16 + (j % 4), c);
    cols[j] = c[1];
  }

  float acc[8][CN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < CN; ++j) acc[i][j] = 0.f;

  const int ktiles = (p.K + TBK - 1) / TBK;
  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tiles((kt + 1) * TBK);  // Fig. 6: preload next tile into registers
#pragma unroll
    for (int k = 0; k < TBK; ++k) {
      float af[8], bf[CN];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(&As[buf][k][rows[4 * g]]);
        af[4 * g] = v.x; af[4 * g + 1] = v.y; af[4 * g + 2] = v.z; af[4 * g + 3] = v.w;
      }
#pragma unroll
      for (int g = 0; g < CN / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(&Bs[buf][k][cols[4 * g]]);
        bf[4 * g] = v.x; bf[4 * g + 1] = v.y; bf[4 * g + 2] = v.z; bf[4 * g + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < CN; ++j) acc[i][j] = fmaf(af[i], bf[j], acc[i][j]);
    }
    if (kt + 1 < ktiles) {
      store_tiles(buf ^ 1);  // commit the staged tile to the other buffer
      __syncthreads();
    }
  }
  // fused epilogue + predicated store through the output address map
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = m0 + rows[i];
    if (r >= p.M) continue;
    const int64_t obase = row_part(p.out_a.P, p.out_a.s_hi, p.out_a.s_lo, r) + b * p.out_a.s_batch + p.out_a.offset;
#pragma unroll
    for (int j = 0; j < CN; ++j) {
      const int64_t c = n0 + cols[j];
      if (c >= p.N) continue;
      const float v = epilogue1(p, acc[i][j], r, c, b);
      const int64_t o = obase + c * p.out_a.s_col;
      if (p.out_dtype == DT_F32) reinterpret_cast<float*>(p.out)[o] = v;
      else if (p.out_dtype == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16_rn(v);
      else reinterpret_cast<__half*>(p.out)[o] = __float2half_rn(v);
    }
  }
}

}  // namespace

// Host-side evaluation of the compile-time mappings compiled into this kernel
// (0: compute, 1: A load, 2: B load), for parity tests against TaskMapping.
int kernel_mapping_assign(int which, uint32_t worker, int* buf, int cap) {
  auto run = [&](auto tag, int dims) {
    using M = decltype(tag);
    if (worker >= M::workers || static_cast<int>(M::tasks) * dims > cap) return -1;
    for (uint32_t i = 0; i < M::tasks; ++i) M::task(worker, i, buf + i * dims);
    return static_cast<int>(M::tasks);
  };
  if (which == 0) return run(ComputeMap{}, 2);
  if (which == 1) return run(LoadA{}, 2);
  if (which == 2) return run(LoadB{}, 2);
  return -1;
}

void launch_simt(const BoundKernel& k, void* stream) {
  const GemmParams& p = k.p;
  const int64_t blocks = int64_t(p.batch) * p.tiles_m * p.tiles_n;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = static_cast<unsigned>(blocks);
  if (k.bn == 64) {
    if (k.stages == 16) simt_gemm_kernel<64, 16><<<g, 256, 0, s>>>(p);
    else simt_gemm_kernel<64, 8><<<g, 256, 0, s>>>(p);
  } else {
    if (k.stages == 16) simt_gemm_kernel<128, 16><<<g, 256, 0, s>>>(p);
    else simt_gemm_kernel<128, 8><<<g, 256, 0, s>>>(p);
  }
}

}  // namespace tmb
