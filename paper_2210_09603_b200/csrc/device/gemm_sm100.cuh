// Fused task-mapped GEMM for sm_100a (tcgen05 + TMEM + TMA + mbarrier ring).
//
// This is the B200 form of the spec's matmul_template (SPEC.md:291-299,
// design :326-331) and of Hidet's tiled matmul with double buffering
// (PAPER.md:289-291):
//   * block -> tile assignment is a task mapping (GemmParams::tile_map),
//     evaluated in closed form (taskmap.cuh); out-of-domain tasks are skipped,
//     i.e. predicated, which is what makes the space input-size agnostic;
//   * the double buffer becomes an S-stage shared-memory ring guarded by
//     full/empty mbarriers, filled by TMA (or by a predicated gather warp
//     group for operands TMA cannot describe: odd strides, casts, im2col);
//   * the inner product runs on the 5th-gen tensor core (tcgen05.mma issued by
//     one thread) into a double-buffered TMEM accumulator;
//   * the epilogue warps drain TMEM -> registers, apply the fused epilogue op
//     list (bias / scale / BN-fold / ReLU / GELU / residual ...) and store
//     through the epilogue's output address map (NCHW re-index etc.).
//
// Warp roles (9 warps): 0-3 loaders, 4-7 epilogue (TMEM lane groups 0-3),
// 8 MMA issuer + TMEM owner.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gemm_params.h"
#include "ptx.cuh"

namespace tmb {

constexpr int kBM = 128;          // tile rows (TMEM lanes)
constexpr int kRowBytes = 128;    // one swizzle-128B row of K
constexpr int kNumThreads = 288;  // 9 warps

template <int BN, int STAGES, bool TF32>
struct GemmCfg {
  static constexpr int kElem = TF32 ? 4 : 2;
  static constexpr int BK = kRowBytes / kElem;        // 64 bf16 / 32 tf32
  static constexpr int KSTEP = TF32 ? 8 : 16;          // K per tcgen05.mma
  static constexpr int NSTEP = BK / KSTEP;             // 4
  static constexpr int A_BYTES = kBM * kRowBytes;      // 16 KB
  static constexpr int B_BYTES = BN * kRowBytes;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 must be 16..256 step 16");
};

namespace detail {

__device__ __forceinline__ int64_t addr_rowpart(const Addr& a, int64_t row, int64_t batch) {
  return (row / a.P) * a.s_hi + (row % a.P) * a.s_lo + batch * a.s_batch + a.offset;
}

// Raw bits of one element converted to the MMA input format.
template <bool TF32>
__device__ __forceinline__ uint32_t load_bits(const void* base, int64_t idx, int32_t dt) {
  if (TF32) {
    float f;
    if (dt == DT_F32) f = __ldg(reinterpret_cast<const float*>(base) + idx);
    else if (dt == DT_BF16) f = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
    else f = __half2float(reinterpret_cast<const __half*>(base)[idx]);
    return __float_as_uint(f);
  } else {
    if (dt == DT_BF16) return __ldg(reinterpret_cast<const unsigned short*>(base) + idx);
    float f = dt == DT_F32 ? __ldg(reinterpret_cast<const float*>(base) + idx)
                           : __half2float(reinterpret_cast<const __half*>(base)[idx]);
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<unsigned short*>(&h);
  }
}

// Store one 16-byte chunk (chunk index c of a 128-byte K row) of tile row r
// into a SWIZZLE_128B K-major tile (the layout TMA would have produced).
__device__ __forceinline__ void st_sw128(uint8_t* tile, int r, int c, uint4 v) {
  uint8_t* p = tile + r * kRowBytes + ((c ^ (r & 7)) << 4);
  *reinterpret_cast<uint4*>(p) = v;
}

template <bool TF32>
__device__ __forceinline__ uint4 pack_chunk(const uint32_t* bits) {
  uint4 v;
  if (TF32) {
    v.x = bits[0]; v.y = bits[1]; v.z = bits[2]; v.w = bits[3];
  } else {
    v.x = bits[0] | (bits[1] << 16);
    v.y = bits[2] | (bits[3] << 16);
    v.z = bits[4] | (bits[5] << 16);
    v.w = bits[6] | (bits[7] << 16);
  }
  return v;
}

// Predicated gather of one tile row of a strided operand (prologue = load/cast).
template <bool TF32, int BK>
__device__ __forceinline__ void gather_row_strided(uint8_t* tile, int r, const Strided& s,
                                                   int64_t row, bool row_ok, int64_t batch,
                                                   int k0, int K) {
  constexpr int PER = TF32 ? 4 : 8;
  const int64_t base = row_ok ? ((row / s.P) * s.s_hi + (row % s.P) * s.s_lo +
                                 batch * s.s_batch + s.offset)
                              : 0;
#pragma unroll
  for (int c = 0; c < BK / PER; ++c) {
    uint32_t bits[8];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int k = k0 + c * PER + j;
      bits[j] = (row_ok && k < K) ? load_bits<TF32>(s.ptr, base + (int64_t)k * s.s_k, s.dtype) : 0u;
    }
    st_sw128(tile, r, c, pack_chunk<TF32>(bits));
  }
}

// Predicated im2col gather of one tile row (= one output pixel), the
// reference Col node (compute_ir.cpp:532-557): zero outside the padded image.
template <bool TF32, int BK>
__device__ __forceinline__ void gather_row_im2col(uint8_t* tile, int r, const ConvGeom& g,
                                                  int64_t pix, bool row_ok, int k0, int K) {
  constexpr int PER = TF32 ? 4 : 8;
  const int hw = g.ho * g.wo;
  const int img = row_ok ? static_cast<int>(pix / hw) : 0;
  const int rem = row_ok ? static_cast<int>(pix % hw) : 0;
  const int oh = rem / g.wo, ow = rem % g.wo;
  const int bh = oh * g.stride - g.pad, bw = ow * g.stride - g.pad;
  const int64_t xbase = static_cast<int64_t>(img) * g.sx[0];
  const int khw = g.kh * g.kw;
  int ch, fh, fw;
  if (g.korder == 0) {
    ch = k0 / khw;
    const int rr = k0 % khw;
    fh = rr / g.kw;
    fw = rr % g.kw;
  } else {
    const int tap = k0 / g.c;
    ch = k0 % g.c;
    fh = tap / g.kw;
    fw = tap % g.kw;
  }
#pragma unroll 1
  for (int c = 0; c < BK / PER; ++c) {
    uint32_t bits[8];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int k = k0 + c * PER + j;
      const int ih = bh + fh, iw = bw + fw;
      const bool ok = row_ok && k < K && ih >= 0 && ih < g.h && iw >= 0 && iw < g.w;
      bits[j] = ok ? load_bits<TF32>(g.x, xbase + ch * g.sx[1] + ih * g.sx[2] + iw * g.sx[3],
                                     g.x_dtype)
                   : 0u;
      if (g.korder == 0) {
        if (++fw == g.kw) { fw = 0; if (++fh == g.kh) { fh = 0; ++ch; } }
      } else {
        if (++ch == g.c) { ch = 0; if (++fw == g.kw) { fw = 0; ++fh; } }
      }
    }
    st_sw128(tile, r, c, pack_chunk<TF32>(bits));
  }
}

// Filter gather of one tile row (= one output channel f) of Wf (the flatten
// node, compute_ir.cpp:558-569), any strides of W, either K order.
template <bool TF32, int BK>
__device__ __forceinline__ void gather_row_filter(uint8_t* tile, int r, const ConvGeom& g,
                                                  int64_t f, bool row_ok, int k0, int K) {
  constexpr int PER = TF32 ? 4 : 8;
  const int khw = g.kh * g.kw;
  int ch, fh, fw;
  if (g.korder == 0) {
    ch = k0 / khw;
    const int rr = k0 % khw;
    fh = rr / g.kw;
    fw = rr % g.kw;
  } else {
    const int tap = k0 / g.c;
    ch = k0 % g.c;
    fh = tap / g.kw;
    fw = tap % g.kw;
  }
  const int64_t wbase = f * g.sw[0];
#pragma unroll 1
  for (int c = 0; c < BK / PER; ++c) {
    uint32_t bits[8];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int k = k0 + c * PER + j;
      const bool ok = row_ok && k < K;
      bits[j] = ok ? load_bits<TF32>(g.wt, wbase + ch * g.sw[1] + fh * g.sw[2] + fw * g.sw[3],
                                     g.w_dtype)
                   : 0u;
      if (g.korder == 0) {
        if (++fw == g.kw) { fw = 0; if (++fh == g.kh) { fh = 0; ++ch; } }
      } else {
        if (++ch == g.c) { ch = 0; if (++fw == g.kw) { fw = 0; ++fh; } }
      }
    }
    st_sw128(tile, r, c, pack_chunk<TF32>(bits));
  }
}

__device__ __forceinline__ float gelu_tanh(float x) {
  // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))), tanh(u) = 1 - 2/(exp(2u)+1)
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = 1.0f - 2.0f / (__expf(2.0f * u) + 1.0f);
  return 0.5f * x * (1.0f + t);
}

__device__ __forceinline__ float load_side(const void* p, int64_t idx, int32_t dt) {
  if (dt == DT_F32) return __ldg(reinterpret_cast<const float*>(p) + idx);
  if (dt == DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return __half2float(reinterpret_cast<const __half*>(p)[idx]);
}

// Applies the fused epilogue op list to 16 consecutive columns of one row.
__device__ __forceinline__ void apply_epilogue(const GemmParams& p, float (&v)[16],
                                               const int64_t* rowpart, int64_t col0,
                                               bool row_ok) {
  for (int o = 0; o < p.n_ops; ++o) {
    const EpiOp& op = p.ops[o];
    const int kind = op.kind;
    if (kind >= EPI_ADD_T && kind <= EPI_MIN_T) {
      float s[16];
      if (op.a.s_col == 0) {
        const float x = row_ok ? load_side(op.ptr, rowpart[o], op.dtype) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) s[j] = x;
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          s[j] = (row_ok && col0 + j < p.N)
                     ? load_side(op.ptr, rowpart[o] + (col0 + j) * op.a.s_col, op.dtype)
                     : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        switch (kind) {
          case EPI_ADD_T: v[j] = v[j] + s[j]; break;
          case EPI_SUB_T: v[j] = v[j] - s[j]; break;
          case EPI_RSUB_T: v[j] = s[j] - v[j]; break;
          case EPI_MUL_T: v[j] = v[j] * s[j]; break;
          case EPI_DIV_T: v[j] = v[j] / s[j]; break;
          case EPI_RDIV_T: v[j] = s[j] / v[j]; break;
          case EPI_MAX_T: v[j] = fmaxf(v[j], s[j]); break;
          default: v[j] = fminf(v[j], s[j]); break;
        }
      }
      continue;
    }
    const float c = op.c;
    switch (kind) {
#define TMB_EW(K, EXPR) \
  case K:               \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) { const float x = v[j]; v[j] = (EXPR); } break;
      TMB_EW(EPI_ADD_C, x + c)
      TMB_EW(EPI_SUB_C, x - c)
      TMB_EW(EPI_RSUB_C, c - x)
      TMB_EW(EPI_MUL_C, x * c)
      TMB_EW(EPI_DIV_C, x / c)
      TMB_EW(EPI_RDIV_C, c / x)
      TMB_EW(EPI_MAX_C, fmaxf(x, c))
      TMB_EW(EPI_MIN_C, fminf(x, c))
      TMB_EW(EPI_RELU, fmaxf(x, 0.f))
      TMB_EW(EPI_GELU_TANH, gelu_tanh(x))
      TMB_EW(EPI_EXP, __expf(x))
      TMB_EW(EPI_SQRT, sqrtf(x))
      TMB_EW(EPI_NEG, -x)
      TMB_EW(EPI_ROUND_BF16, __bfloat162float(__float2bfloat16_rn(x)))
#undef TMB_EW
      default: break;
    }
  }
}

__device__ __forceinline__ void store_out(const GemmParams& p, const float (&v)[16], int64_t base,
                                          int64_t col0, bool row_ok) {
  if (!row_ok) return;
  const int64_t sc = p.out_a.s_col;
  const bool full = col0 + 16 <= p.N;
  if (p.out_dtype == DT_BF16) {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out);
    if (sc == 1 && full && ((reinterpret_cast<uintptr_t>(o + base + col0) & 15) == 0)) {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      uint4* dst = reinterpret_cast<uint4*>(o + base + col0);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (col0 + j < p.N) o[base + (col0 + j) * sc] = __float2bfloat16_rn(v[j]);
    }
  } else if (p.out_dtype == DT_F32) {
    float* o = reinterpret_cast<float*>(p.out);
    if (sc == 1 && full && ((reinterpret_cast<uintptr_t>(o + base + col0) & 15) == 0)) {
      float4* dst = reinterpret_cast<float4*>(o + base + col0);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (col0 + j < p.N) o[base + (col0 + j) * sc] = v[j];
    }
  } else {
    __half* o = reinterpret_cast<__half*>(p.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (col0 + j < p.N) o[base + (col0 + j) * sc] = __float2half_rn(v[j]);
  }
}

// Decodes task `i` of this CTA into (batch, tile_m, tile_n); false once the
// CTA's task list is exhausted.  Out-of-range tasks are reported via `valid`.
__device__ __forceinline__ bool next_tile(const GemmParams& p, uint32_t i, int& b, int& tm_,
                                          int& tn, bool& valid) {
  if (i >= p.tile_map.tasks) return false;
  int32_t c[tm::kMaxRank];
  tm::dev_task(p.tile_map, blockIdx.x, i, c);
  b = c[0];
  tm_ = c[1];
  tn = c[2];
  valid = b < p.batch && tm_ < p.tiles_m && tn < p.tiles_n;
  return true;
}

}  // namespace detail

template <int BN, int STAGES, bool TF32>
__global__ void __launch_bounds__(kNumThreads, 1)
    tm_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB) {
  using Cfg = GemmCfg<BN, STAGES, TF32>;
  constexpr int BK = Cfg::BK;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool a_tma = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA;
  const bool b_tma = p.b_loader == LD_TMA_K || p.b_loader == LD_TMA_MN;
  const bool all_tma = a_tma && b_tma;

  if (threadIdx.x == 0) {
    if (a_tma) ptx::tma_prefetch_desc(&tmA);
    if (b_tma) ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], all_tma ? 1 : 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    // ===================== loaders (prologue splice) =====================
    const int t = threadIdx.x;  // 0..127
    if (all_tma && t != 0) {
      // idle: single-thread TMA producer
    } else {
      int stage = 0;
      uint32_t phase = 0;
      int b, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile(p, i, b, tm_, tn, valid); ++i) {
        if (!valid) continue;
        const int m0 = tm_ * kBM, n0 = tn * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* a_tile = smA + stage * Cfg::A_BYTES;
          uint8_t* b_tile = smB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (all_tma) {
            ptx::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          } else if (t == 0) {
            // mixed mode: announce the TMA bytes now, arrive after the gather
            const uint32_t tx = (a_tma ? Cfg::A_BYTES : 0) + (b_tma ? Cfg::B_BYTES : 0);
            if (tx) ptx::mbar_expect_tx(&full[stage], tx);
          }
          if (t == 0) {
            if (p.a_loader == LD_TMA_K) {
              ptx::tma_load_3d(a_tile, &tmA, &full[stage], k0, m0, b);
            } else if (p.a_loader == LD_IM2COL_TMA) {
              // K block = (tap, channel block); rows = 128 consecutive output pixels.
              const int cblocks = p.conv.c / BK;
              const int tap = kb / cblocks, cb = kb % cblocks;
              const int fh = tap / p.conv.kw, fw = tap % p.conv.kw;
              const int hw = p.conv.ho * p.conv.wo;
              const int img = m0 / hw, rem = m0 % hw;
              const int oh = rem / p.conv.wo, ow = rem % p.conv.wo;
              ptx::tma_load_im2col_4d(a_tile, &tmA, &full[stage], cb * BK,
                                      ow * p.conv.stride - p.conv.pad,
                                      oh * p.conv.stride - p.conv.pad, img,
                                      static_cast<uint16_t>(fw), static_cast<uint16_t>(fh));
            }
            if (p.b_loader == LD_TMA_K) {
              ptx::tma_load_3d(b_tile, &tmB, &full[stage], k0, n0, b);
            } else if (p.b_loader == LD_TMA_MN) {
#pragma unroll 1
              for (int j = 0; j < BN / 64; ++j)
                ptx::tma_load_3d(b_tile + j * (64 * kRowBytes), &tmB, &full[stage], n0 + 64 * j,
                                 k0, b);
            }
          }
          if (!all_tma) {
            // predicated gather of the non-TMA operand(s), one tile row per thread
            if (!a_tma) {
              const int64_t row = m0 + t;
              const bool ok = row < p.M;
              if (p.a_loader == LD_GATHER)
                detail::gather_row_strided<TF32, BK>(a_tile, t, p.a, row, ok, b, k0, p.K);
              else
                detail::gather_row_im2col<TF32, BK>(a_tile, t, p.conv, row, ok, k0, p.K);
            }
            if (!b_tma) {
#pragma unroll 1
              for (int r = t; r < BN; r += 128) {
                const int64_t row = n0 + r;
                const bool ok = row < p.N;
                if (p.b_loader == LD_GATHER)
                  detail::gather_row_strided<TF32, BK>(b_tile, r, p.b, row, ok, b, k0, p.K);
                else
                  detail::gather_row_filter<TF32, BK>(b_tile, r, p.conv, row, ok, k0, p.K);
              }
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&full[stage]);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp < 8) {
    // ===================== epilogue (epilogue splice) =====================
    const int lg = warp - 4;  // TMEM lane group
    int acc = 0;
    uint32_t acc_phase = 0;
    int b, tm_, tn;
    bool valid;
    int64_t rowpart[kMaxEpiOps];
    for (uint32_t i = 0; detail::next_tile(p, i, b, tm_, tn, valid); ++i) {
      if (!valid) continue;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t row = static_cast<int64_t>(tm_) * kBM + lg * 32 + lane;
      const bool row_ok = row < p.M;
      const int64_t rr = row_ok ? row : 0;
      for (int o = 0; o < p.n_ops; ++o) rowpart[o] = detail::addr_rowpart(p.ops[o].a, rr, b);
      const int64_t obase = detail::addr_rowpart(p.out_a, rr, b);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        const int64_t col0 = static_cast<int64_t>(tn) * BN + c * 16;
        if (col0 >= p.N) break;  // warp-uniform
        uint32_t r[16];
        ptx::tmem_ld16(taddr + c * 16, r);
        ptx::tmem_wait_ld();
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        detail::apply_epilogue(p, v, rowpart, col0, row_ok);
        detail::store_out(p, v, obase, col0, row_ok);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
  } else {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      const bool b_mn = p.b_loader == LD_TMA_MN;
      const uint32_t idesc = ptx::make_idesc(kBM, BN, TF32 ? 2u : 1u, false, b_mn);
      const uint32_t mn_lbo = p.mn_lbo_sbo_swap ? 1024u : 64u * kRowBytes;
      const uint32_t mn_sbo = p.mn_lbo_sbo_swap ? 64u * kRowBytes : 1024u;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int b, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile(p, i, b, tm_, tn, valid); ++i) {
        if (!valid) continue;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = ptx::smem_u32(smB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < Cfg::NSTEP; ++kk) {
            const uint64_t adesc = ptx::smem_desc_sw128(a_addr + kk * Cfg::KSTEP * Cfg::kElem, 16, 1024);
            const uint64_t bdesc =
                b_mn ? ptx::smem_desc_sw128(b_addr + kk * Cfg::KSTEP * kRowBytes, mn_lbo, mn_sbo)
                     : ptx::smem_desc_sw128(b_addr + kk * Cfg::KSTEP * Cfg::kElem, 16, 1024);
            const uint32_t accum = (kb | kk) != 0;
            if (TF32) ptx::mma_tf32(d_tmem, adesc, bdesc, idesc, accum);
            else ptx::mma_f16(d_tmem, adesc, bdesc, idesc, accum);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        ptx::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tmb
