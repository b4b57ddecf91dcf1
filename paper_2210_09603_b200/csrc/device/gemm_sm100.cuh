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
// Warp roles (13 warps): 0-3 loaders, 4-11 epilogue (TMEM lane group = warp%4,
// interleaved 16-column chunks), 12 MMA issuer + TMEM owner.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gemm_params.h"
#include "ptx.cuh"

namespace tmb {

constexpr int kBM = 128;          // tile rows (TMEM lanes)
constexpr int kRowBytes = 128;    // one swizzle-128B row of K
constexpr int kEpiWarps = 8;       // epilogue warps (2 per TMEM lane group)
constexpr int kNumThreads = 32 * (4 + kEpiWarps + 1);  // loaders + epilogue + MMA

// CG = CTAs per MMA (cta_group): 1, or 2 for the SM-pair form where the tile
// is (2*128) x BN, each CTA stages its 128 rows of A and BN/2 rows of B, and
// the pair leader issues tcgen05.mma.cta_group::2 over both CTAs' smem.
template <int BN, int STAGES, bool TF32, int CG = 1>
struct GemmCfg {
  static constexpr int kElem = TF32 ? 4 : 2;
  static constexpr int BK = kRowBytes / kElem;        // 64 bf16 / 32 tf32
  static constexpr int KSTEP = TF32 ? 8 : 16;          // K per tcgen05.mma
  static constexpr int NSTEP = BK / KSTEP;             // 4
  static constexpr int A_BYTES = kBM * kRowBytes;      // 16 KB
  static constexpr int B_BYTES = (BN / CG) * kRowBytes;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int COLBUF_BYTES = kMaxEpiOps * BN * 4;  // staged per-column epilogue operands
  static constexpr int OUTBUF_BYTES = kEpiWarps * 32 * 16 * 4;  // per-warp 32x16 output chunk (<= f32)
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + COLBUF_BYTES + OUTBUF_BYTES;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 must be 16..256 step 16");
};

namespace detail {

__device__ __forceinline__ int64_t addr_rowpart(const Addr& a, int64_t row, int64_t batch) {
  int64_t q, r;
  if (a.P < (int64_t(1) << 31) && row < (int64_t(1) << 31)) {  // 32-bit divide fast path
    const uint32_t rr = static_cast<uint32_t>(row), pp = static_cast<uint32_t>(a.P);
    const uint32_t qq = rr / pp;
    q = qq;
    r = rr - qq * pp;
  } else {
    q = row / a.P;
    r = row % a.P;
  }
  return q * a.s_hi + r * a.s_lo + batch * a.s_batch + a.offset;
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
  } else {  // (tap, channel) with cpad >= c channels per tap; padded channels are zero
    const int tap = k0 / g.cpad;
    ch = k0 % g.cpad;
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
      const bool ok = row_ok && k < K && ch < g.c && fh < g.kh;
      bits[j] = ok ? load_bits<TF32>(g.wt, wbase + ch * g.sw[1] + fh * g.sw[2] + fw * g.sw[3],
                                     g.w_dtype)
                   : 0u;
      if (g.korder == 0) {
        if (++fw == g.kw) { fw = 0; if (++fh == g.kh) { fh = 0; ++ch; } }
      } else {
        if (++ch == g.cpad) { ch = 0; if (++fw == g.kw) { fw = 0; ++fh; } }
      }
    }
    st_sw128(tile, r, c, pack_chunk<TF32>(bits));
  }
}

__device__ __forceinline__ float gelu_tanh(float x) {
  // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))), tanh(u) = 1 - 2/(exp(2u)+1);
  // __fdividef(2, inf) = 0 gives the right limit when exp overflows.
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = 1.0f - __fdividef(2.0f, __expf(2.0f * u) + 1.0f);
  return 0.5f * x * (1.0f + t);
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// one MUFU op per element; used when the output is bf16 (|err| ~ 2^-11 << bf16 ulp)
__device__ __forceinline__ float gelu_tanh_fast(float x) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(u), hx);
}

__device__ __forceinline__ float load_side(const void* p, int64_t idx, int32_t dt) {
  if (dt == DT_F32) return __ldg(reinterpret_cast<const float*>(p) + idx);
  if (dt == DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return __half2float(reinterpret_cast<const __half*>(p)[idx]);
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4 u, float* o) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// 16 consecutive columns of a matrix side operand for one row (vectorised
// when contiguous and 16-byte aligned, otherwise predicated scalar loads).
__device__ __forceinline__ void load_mat16(const EpiOp& op, int64_t rowpart, int64_t col0, int N,
                                           bool row_ok, float (&out)[16]) {
  if (!row_ok) {
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = 0.f;
    return;
  }
  const int64_t base = rowpart + col0 * op.a.s_col;
  if (op.a.s_col == 1 && col0 + 16 <= N) {
    if (op.dtype == DT_BF16 && ((reinterpret_cast<uintptr_t>(op.ptr) + base * 2) & 15) == 0) {
      const uint4* q = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(op.ptr) + base);
      bf16x8_to_f32(__ldg(q), out);
      bf16x8_to_f32(__ldg(q + 1), out + 8);
      return;
    }
    if (op.dtype == DT_F32 && ((reinterpret_cast<uintptr_t>(op.ptr) + base * 4) & 15) == 0) {
      const float4* q = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(op.ptr) + base);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = __ldg(q + i);
        out[4 * i] = f.x; out[4 * i + 1] = f.y; out[4 * i + 2] = f.z; out[4 * i + 3] = f.w;
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    out[j] = (col0 + j < N) ? load_side(op.ptr, base + j * op.a.s_col, op.dtype) : 0.f;
}

// Applies the fused epilogue op list to 16 consecutive columns of one row.
// Side operands come from: smem column buffers (SIDE_COL), a per-row register
// (SIDE_ROW) or the prefetched matrix chunk (SIDE_MAT).
template <int BN>
__device__ __forceinline__ void apply_epilogue(const GemmParams& p, float (&v)[16], const float* colbuf,
                                               int cbase, const float* rowv, const float (&mat)[kMaxMatOps][16]) {
  for (int o = 0; o < p.n_ops; ++o) {
    const EpiOp& op = p.ops[o];
    const int kind = op.kind;
    if (kind >= EPI_ADD_T && kind <= EPI_MIN_T) {
      float s[16];
      if (op.side == SIDE_COL) {
        const float4* cb = reinterpret_cast<const float4*>(colbuf + o * BN + cbase);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 f = cb[i];
          s[4 * i] = f.x; s[4 * i + 1] = f.y; s[4 * i + 2] = f.z; s[4 * i + 3] = f.w;
        }
      } else if (op.side == SIDE_ROW) {
        const float x = rowv[o];
#pragma unroll
        for (int j = 0; j < 16; ++j) s[j] = x;
      } else {
        const int sl = op.slot;
#pragma unroll
        for (int j = 0; j < 16; ++j) s[j] = sl == 0 ? mat[0][j] : mat[1][j];
      }
      switch (kind) {
#define TMB_TW(K, EXPR) \
  case K:               \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) { const float x = v[j], y = s[j]; v[j] = (EXPR); } break;
        TMB_TW(EPI_ADD_T, x + y)
        TMB_TW(EPI_SUB_T, x - y)
        TMB_TW(EPI_RSUB_T, y - x)
        TMB_TW(EPI_MUL_T, x * y)
        TMB_TW(EPI_DIV_T, x / y)
        TMB_TW(EPI_RDIV_T, y / x)
        TMB_TW(EPI_MAX_T, fmaxf(x, y))
        TMB_TW(EPI_MIN_T, fminf(x, y))
#undef TMB_TW
        default: break;
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
      TMB_EW(EPI_GELU_TANH, p.fast_math ? gelu_tanh_fast(x) : gelu_tanh(x))
      TMB_EW(EPI_EXP, __expf(x))
      TMB_EW(EPI_SQRT, sqrtf(x))
      TMB_EW(EPI_NEG, -x)
      TMB_EW(EPI_ROUND_BF16, __bfloat162float(__float2bfloat16_rn(x)))
#undef TMB_EW
      default: break;
    }
  }
}

// Canonical epilogue: v = act(acc * S[c] + T[c]) (+ R), S/T staged in smem.
template <int BN>
__device__ __forceinline__ void apply_canon(const GemmParams& p, float (&v)[16], const float* colbuf, int cbase,
                                            const float (&mat)[kMaxMatOps][16]) {
  const float4* S = reinterpret_cast<const float4*>(colbuf + cbase);
  const float4* T = reinterpret_cast<const float4*>(colbuf + BN + cbase);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 s = S[q], t = T[q];
    v[4 * q] = fmaf(v[4 * q], s.x, t.x);
    v[4 * q + 1] = fmaf(v[4 * q + 1], s.y, t.y);
    v[4 * q + 2] = fmaf(v[4 * q + 2], s.z, t.z);
    v[4 * q + 3] = fmaf(v[4 * q + 3], s.w, t.w);
  }
  if (p.canon_act == 1) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
  } else if (p.canon_act == 2) {
    if (p.fast_math) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = gelu_tanh_fast(v[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = gelu_tanh(v[j]);
    }
  }
  if (p.canon_res_slot == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += mat[0][j];
  } else if (p.canon_res_slot == 1) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += mat[1][j];
  }
}

// GENERIC = false compiles only the canonical epilogue (and, in the kernel, only
// TMA operand loaders): the hot loops then fit the instruction cache, which the
// full interpreter + gather code (~370 KB of SASS per instantiation) does not.
template <int BN, bool GENERIC>
__device__ __forceinline__ void epilogue16(const GemmParams& p, float (&v)[16], const float* colbuf, int cbase,
                                           const float* rowv, const float (&mat)[kMaxMatOps][16]) {
  if constexpr (GENERIC) {
    if (p.canon) apply_canon<BN>(p, v, colbuf, cbase, mat);
    else apply_epilogue<BN>(p, v, colbuf, cbase, rowv, mat);
  } else {
    apply_canon<BN>(p, v, colbuf, cbase, mat);
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
__device__ __forceinline__ void trace(const GemmParams& p, uint32_t i, int ev, long long t0) {
  if (p.trace != nullptr && i < static_cast<uint32_t>(kTraceTiles))
    p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + i) * kTraceEvents + ev] = clock64() - t0;
}

template <int CG>
__device__ __forceinline__ bool next_tile(const GemmParams& p, uint32_t i, int& b, int& ks, int& tm_,
                                          int& tn, bool& valid) {
  if (i >= p.tile_map.tasks) return false;
  int32_t c[tm::kMaxRank];
  tm::dev_task(p.tile_map, blockIdx.x / CG, i, c);  // workers = CTA pairs when CG == 2
  b = c[0] / p.split_k;
  ks = c[0] % p.split_k;
  tm_ = c[1];
  tn = c[2];
  valid = b < p.batch && tm_ < p.tiles_m && tn < p.tiles_n;
  return true;
}

}  // namespace detail

template <int BN, int STAGES, bool TF32, int CG, bool GENERIC>
__global__ void __launch_bounds__(kNumThreads, 1)
    tm_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC) {
  using Cfg = GemmCfg<BN, STAGES, TF32, CG>;
  constexpr int BK = Cfg::BK;
  constexpr int kTileM = kBM * CG;  // rows per tile (both CTAs of a pair)
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
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
  uint32_t* split_flag = tmem_slot + 1;
  float* colbuf = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES + 256);
  uint8_t* outbuf = smem + STAGES * Cfg::STAGE_BYTES + 256 + Cfg::COLBUF_BYTES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool a_tma = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA || p.a_loader == LD_IM2COL_TMA8;
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
      ptx::mbar_init(&tempty[a], kEpiWarps * CG);  // both CTAs' epilogues drain before reuse
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4 + kEpiWarps) {
    if constexpr (CG == 2) ptx::tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
    else ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer barriers initialised before any TMA/arrive
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long t0 = clock64();
  if (p.trace != nullptr && threadIdx.x == 0)
    p.trace[static_cast<int64_t>(blockIdx.x) * kTraceTiles * kTraceEvents + TR_CTA_START] =
        static_cast<long long>(ptx::globaltimer());

  if (warp < 4) {
    // ===================== loaders (prologue splice) =====================
    const int t = threadIdx.x;  // 0..127
    if (all_tma && t != 0) {
      // idle: single-thread TMA producer
    } else {
      int stage = 0;
      uint32_t phase = 0;
      int b, ks, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile<CG>(p, i, b, ks, tm_, tn, valid); ++i) {
        if (!valid) continue;
        // this CTA's rows of A and columns of B (half of each tile's B when CG == 2)
        const int m0 = tm_ * kTileM + rank * kBM, n0 = tn * BN + rank * (BN / CG);
        for (int kb0 = ks * p.kb_per_split, kb = kb0, kb_end = min(p.num_kb, kb0 + p.kb_per_split); kb < kb_end; ++kb) {
          if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&empty[stage], phase ^ 1u);
          else ptx::mbar_wait(&empty[stage], phase ^ 1u);
          if (kb == kb0 && t == 0) detail::trace(p, i, TR_PROD_FIRST, t0);
          if (kb == kb_end - 1 && t == 0) detail::trace(p, i, TR_PROD_LAST, t0);
          uint8_t* a_tile = smA + stage * Cfg::A_BYTES;
          uint8_t* b_tile = smB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if constexpr (CG == 2) {
            // both CTAs' TMA bytes complete on the leader's full barrier
            const uint32_t lead_full = ptx::mapa_shared(ptx::smem_u32(&full[stage]), 0);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * Cfg::STAGE_BYTES);
            if (p.a_loader == LD_TMA_K) {
              ptx::tma_load_3d_2sm(a_tile, &tmA, lead_full, k0, m0, b);
            } else {
              const int cblocks = p.conv.c / BK;
              const int tap = kb / cblocks, cb = kb % cblocks;
              const int fh = tap / p.conv.kw, fw = tap % p.conv.kw;
              const int hw = p.conv.ho * p.conv.wo;
              const int img = m0 / hw, rem = m0 % hw;
              const int oh = rem / p.conv.wo, ow = rem % p.conv.wo;
              ptx::tma_load_im2col_4d_2sm(a_tile, &tmA, lead_full, cb * BK, ow * p.conv.stride - p.conv.pad,
                                          oh * p.conv.stride - p.conv.pad, img, static_cast<uint16_t>(fw),
                                          static_cast<uint16_t>(fh));
            }
            if (p.b_loader == LD_TMA_K) {
              ptx::tma_load_3d_2sm(b_tile, &tmB, lead_full, k0, n0, b);
            } else {
#pragma unroll 1
              for (int j = 0; j < BN / CG / 64; ++j)
                ptx::tma_load_3d_2sm(b_tile + j * (64 * kRowBytes), &tmB, lead_full, n0 + 64 * j, k0, b);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            continue;
          }
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
            } else if (p.a_loader == LD_IM2COL_TMA8) {
              // 8 taps per k-block, one {8 ch x 128 px} box each (2 KB, dense rows of
              // 16 B = one core-matrix column); taps past the window repeat the last
              // one (the filter is zero there, and the data is finite)
              const int hw = p.conv.ho * p.conv.wo;
              const int img = m0 / hw, rem = m0 % hw;
              const int oh = rem / p.conv.wo, ow = rem % p.conv.wo;
              const int taps = p.conv.kh * p.conv.kw;
#pragma unroll 1
              for (int j = 0; j < BK / 8; ++j) {
                const int tap = min(kb * (BK / 8) + j, taps - 1);
                ptx::tma_load_im2col_4d(a_tile + j * 2048, &tmA, &full[stage], 0, ow * p.conv.stride - p.conv.pad,
                                        oh * p.conv.stride - p.conv.pad, img,
                                        static_cast<uint16_t>(tap % p.conv.kw), static_cast<uint16_t>(tap / p.conv.kw));
              }
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
          if (GENERIC && !all_tma) {
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
  } else if (warp < 4 + kEpiWarps) {
    // ===================== epilogue (epilogue splice) =====================
    const int e = warp - 4;          // 0..7
    const int lg = warp & 3;         // TMEM lane group this warp may access
    const int half = e >> 2;         // which interleaved half of the 16-column chunks
    const int et = threadIdx.x - 128;
    constexpr int kChunks = BN / 16;
    int acc = 0;
    uint32_t acc_phase = 0;
    int b, ks, tm_, tn;
    bool valid;
    int64_t rowpart[kMaxEpiOps];
    float rowv[kMaxEpiOps];
    bool has_col = false;
    for (int o = 0; o < p.n_ops; ++o) has_col = has_col || p.ops[o].side == SIDE_COL;
    int staged_tn = -1, staged_b = -1;
    // this warp's 32x16 output staging: 2 KB, a 2-deep ring of 1 KB bf16 chunks
    // (one outstanding TMA store while the next chunk is written) or one f32 chunk
    uint8_t* obuf_base = outbuf + e * (32 * 16 * 4);
    const int obytes = p.out_dtype == DT_F32 ? 4 : 2;
    uint32_t n_emit = 0;
    auto emit = [&](const float (&v)[16], int64_t obase_, int64_t col0, bool row_ok_, int tile_row0) {
      if (!p.out_tma) {
        detail::store_out(p, v, obase_, col0, row_ok_);
        return;
      }
      uint8_t* obuf = obuf_base + (obytes == 2 ? (n_emit & 1u) * 1024 : 0);
      if (lane == 0) {  // the store that last used this buffer has read it
        if (obytes == 2) ptx::bulk_wait_read<1>();
        else ptx::bulk_wait_read<0>();
      }
      ++n_emit;
      __syncwarp();
      if (obytes == 2) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          w[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        uint4* dst = reinterpret_cast<uint4*>(obuf + lane * 32);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      } else {
        float4* dst = reinterpret_cast<float4*>(obuf + lane * 64);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(&tmC, obuf, static_cast<int32_t>(col0), tile_row0, b);
        ptx::bulk_commit();
      }
    };
    for (uint32_t i = 0; detail::next_tile<CG>(p, i, b, ks, tm_, tn, valid); ++i) {
      if (!valid) continue;
      const int64_t n0 = static_cast<int64_t>(tn) * BN;
      const int row0 = tm_ * kTileM + rank * kBM + lg * 32;  // this warp's first row
      const int64_t row = static_cast<int64_t>(row0) + lane;
      const bool row_ok = row < p.M;
      const int64_t rr = row_ok ? row : 0;
      // Stage this tile's column vectors while the MMA works on it; skipped when
      // the previous tile had the same columns (e.g. every tile of a conv whose
      // F fits one tile), which keeps the load latency off the critical path.
      const bool restage = (staged_tn < 0 && (has_col || p.canon)) || (has_col && (tn != staged_tn || b != staged_b));
      if (restage) ptx::named_bar_sync(1, 32 * kEpiWarps);  // previous tile's readers are done
      if (restage && p.canon) {  // S and T column vectors of the canonical epilogue
        for (int c = et; c < BN; c += 32 * kEpiWarps) {
          const bool in = n0 + c < p.N;
          float s = p.canon_s, t = p.canon_t;
          if (p.canon_s_op >= 0 && in) {
            const EpiOp& op = p.ops[p.canon_s_op];
            s = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, b) + (n0 + c) * op.a.s_col, op.dtype);
          }
          if (p.canon_t_op >= 0 && in) {
            const EpiOp& op = p.ops[p.canon_t_op];
            t = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, b) + (n0 + c) * op.a.s_col, op.dtype);
          }
          colbuf[c] = s;
          colbuf[BN + c] = t;
        }
      }
      for (int o = 0; o < p.n_ops; ++o) {
        const EpiOp& op = p.ops[o];
        rowpart[o] = detail::addr_rowpart(op.a, rr, b);
        if (op.side == SIDE_COL && restage && !p.canon) {
          const int64_t cb = detail::addr_rowpart(op.a, 0, b);
          for (int c = et; c < BN; c += 32 * kEpiWarps)
            colbuf[o * BN + c] = (n0 + c < p.N) ? detail::load_side(op.ptr, cb + (n0 + c) * op.a.s_col, op.dtype) : 0.f;
        } else if (op.side == SIDE_ROW) {
          rowv[o] = row_ok ? detail::load_side(op.ptr, rowpart[o], op.dtype) : 0.f;
        }
      }
      const int64_t obase = detail::addr_rowpart(p.out_a, rr, b);
      if (restage) {
        ptx::named_bar_sync(1, 32 * kEpiWarps);  // column buffers ready
        staged_tn = tn;
        staged_b = b;
      }
      if (et == 0) detail::trace(p, i, TR_EPI_READY, t0);
      float mat[kMaxMatOps][16];
      auto prefetch = [&](int c, float (&dst)[kMaxMatOps][16]) {
        for (int o = 0; o < p.n_ops; ++o)
          if (p.ops[o].side == SIDE_MAT) {
            float tmp[16];
            detail::load_mat16(p.ops[o], rowpart[o], n0 + c * 16, p.N, row_ok, tmp);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (p.ops[o].slot == 0) dst[0][j] = tmp[j];
              else dst[1][j] = tmp[j];
            }
          }
      };
      if (p.has_mat && p.split_k == 1) prefetch(2 * half, mat);
      if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&tfull[acc], acc_phase);
      else ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN;
      if (et == 0) detail::trace(p, i, TR_EPI_ACC, t0);
      if (p.split_k > 1) {
        // ---- split-K: park the raw partial tile, last unit reduces + runs the epilogue
        const int64_t tile_id = ((static_cast<int64_t>(b) * p.tiles_m + tm_) * p.tiles_n + tn) * CG + rank;
        const float* ws = p.workspace + tile_id * p.split_k * static_cast<int64_t>(kBM * BN);
        const int rloc = lg * 32 + lane;
#pragma unroll 1
        for (int c = half; c < kChunks; c += 2) {
          uint32_t r[16];
          ptx::tmem_ld16(taddr + c * 16, r);
          ptx::tmem_wait_ld();
          // chunk-major layout: a warp writes 32 consecutive 64-byte rows
          float4* dst = reinterpret_cast<float4*>(const_cast<float*>(ws) + ks * static_cast<int64_t>(kBM * BN) +
                                                  (static_cast<int64_t>(c) * kBM + rloc) * 16);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            __stcg(dst + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // TMEM is free again: the MMA can start the next unit
          if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
          else ptx::mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        __threadfence();
        ptx::named_bar_sync(2, 32 * kEpiWarps);
        if (et == 0) *split_flag = (atomicAdd(&p.counters[tile_id], 1) == p.split_k - 1) ? 1u : 0u;
        ptx::named_bar_sync(2, 32 * kEpiWarps);
        if (*reinterpret_cast<volatile uint32_t*>(split_flag) == 0u) continue;
        __threadfence();
#pragma unroll 1
        for (int c = half; c < kChunks; c += 2) {
          const int64_t col0 = n0 + c * 16;
          if (col0 >= p.N) break;
          if (p.has_mat) prefetch(c, mat);
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
          for (int s = 0; s < p.split_k; ++s) {  // fixed order: deterministic
            const float4* src = reinterpret_cast<const float4*>(ws + s * static_cast<int64_t>(kBM * BN) +
                                                                (static_cast<int64_t>(c) * kBM + rloc) * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = __ldcg(src + q);
              v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
            }
          }
          detail::epilogue16<BN, GENERIC>(p, v, colbuf, c * 16, rowv, mat);
          emit(v, obase, col0, row_ok, row0);
        }
        if (et == 0) p.counters[tile_id] = 0;  // self-resetting for the next launch
        continue;
      }
      // 32 columns per TMEM round trip (one wait per 32 columns); the two warps
      // of a lane group interleave 32-column chunks
#pragma unroll 1
      for (int c2 = half; c2 < BN / 32; c2 += 2) {
        const int64_t colA = n0 + c2 * 32;
        if (colA >= p.N) break;  // warp-uniform
        float nxt[kMaxMatOps][16];
        if (p.has_mat && colA + 16 < p.N) prefetch(2 * c2 + 1, nxt);
        uint32_t r[32];
        // fine-grained epilogue timeline: warp 4 of every CTA, first 32-column chunk
        // of each tile -> trace events 8..13 (kTraceEvents = 16)
        const bool fine = p.trace != nullptr && warp == 4 && c2 == half && i < static_cast<uint32_t>(kTraceTiles);
        auto tick = [&](int ev) {
          if (fine && lane == 0)
            p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + i) * kTraceEvents + ev] = clock64() - t0;
        };
        tick(8);
        ptx::tmem_ld32(taddr + c2 * 32, r);
        ptx::tmem_wait_ld();
        tick(9);
        {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
          detail::epilogue16<BN, GENERIC>(p, v, colbuf, c2 * 32, rowv, mat);
          tick(10);
          emit(v, obase, colA, row_ok, row0);
          tick(11);
        }
        if (colA + 16 < p.N) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[16 + j]);
          if (p.has_mat && c2 + 2 < BN / 32 && colA + 64 < p.N) prefetch(2 * (c2 + 2), mat);
          detail::epilogue16<BN, GENERIC>(p, v, colbuf, c2 * 32 + 16, rowv, nxt);
          tick(12);
          emit(v, obase, colA + 16, row_ok, row0);
          tick(13);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // the (leader's) MMA may overwrite this accumulator once both CTAs drained it
        if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
        else ptx::mbar_arrive(&tempty[acc]);
      }
      if (et == 0) detail::trace(p, i, TR_EPI_DONE, t0);
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    if (p.out_tma && lane == 0) ptx::bulk_wait<0>();  // all output tiles written before exit
  } else {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0 && rank == 0) {
      const bool b_mn = p.b_loader == LD_TMA_MN;
      const bool a_noswz = p.a_loader == LD_IM2COL_TMA8;
      const uint32_t idesc = ptx::make_idesc(kTileM, BN, TF32 ? 2u : 1u, false, b_mn);
      const uint32_t mn_lbo = p.mn_lbo_sbo_swap ? 1024u : 64u * kRowBytes;
      const uint32_t mn_sbo = p.mn_lbo_sbo_swap ? 64u * kRowBytes : 1024u;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int b, ks, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile<CG>(p, i, b, ks, tm_, tn, valid); ++i) {
        if (!valid) continue;
        if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&tempty[acc], acc_phase ^ 1u);
        else ptx::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb0 = ks * p.kb_per_split, kb = kb0, kb_end = min(p.num_kb, kb0 + p.kb_per_split); kb < kb_end; ++kb) {
          if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&full[stage], phase);
          else ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (kb == kb0) detail::trace(p, i, TR_MMA_FIRST, t0);
          const uint32_t a_addr = ptx::smem_u32(smA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = ptx::smem_u32(smB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < Cfg::NSTEP; ++kk) {
            const uint64_t adesc =
                a_noswz ? ptx::smem_desc_noswz(a_addr + kk * 2 * 2048, 2048, 128)  // 2 taps (2 x 16 B chunks) per K16
                        : ptx::smem_desc_sw128(a_addr + kk * Cfg::KSTEP * Cfg::kElem, 16, 1024);
            const uint64_t bdesc =
                b_mn ? ptx::smem_desc_sw128(b_addr + kk * Cfg::KSTEP * kRowBytes, mn_lbo, mn_sbo)
                     : ptx::smem_desc_sw128(b_addr + kk * Cfg::KSTEP * Cfg::kElem, 16, 1024);
            const uint32_t accum = (kb != kb0 || kk != 0);
            if constexpr (CG == 2) {
              if (TF32) ptx::mma_tf32_2sm(d_tmem, adesc, bdesc, idesc, accum);
              else ptx::mma_f16_2sm(d_tmem, adesc, bdesc, idesc, accum);
            } else {
              if (TF32) ptx::mma_tf32(d_tmem, adesc, bdesc, idesc, accum);
              else ptx::mma_f16(d_tmem, adesc, bdesc, idesc, accum);
            }
          }
          // frees this ring slot in both CTAs of the pair
          if constexpr (CG == 2) ptx::mma_commit_2sm(&empty[stage], 0x3);
          else ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        if constexpr (CG == 2) ptx::mma_commit_2sm(&tfull[acc], 0x3);
        else ptx::mma_commit(&tfull[acc]);
        detail::trace(p, i, TR_MMA_LAST, t0);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer done with its TMEM before the pair frees it
  else __syncthreads();
  if (warp == 4 + kEpiWarps) {
    ptx::tc_fence_after();
    if constexpr (CG == 2) ptx::tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
    else ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tmb
