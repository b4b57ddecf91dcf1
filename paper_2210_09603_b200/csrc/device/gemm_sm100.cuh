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
// Warp roles (13 warps): 0-3 loaders, 4-11 epilogue (two groups of 4, one per
// TMEM accumulator buffer; TMEM lane group = warp%4), 12 MMA issuer + TMEM owner.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gemm_params.h"
#include "ptx.cuh"

namespace tmb {

constexpr int kBM = 128;          // tile rows (TMEM lanes)
constexpr int kRowBytes = 128;    // one swizzle-128B row of K
constexpr int kEpiWarps = 8;       // epilogue warps (2 groups x 4 TMEM lane groups)
constexpr int kNumThreads = 32 * (4 + kEpiWarps + 1);  // loaders + epilogue + MMA
// The CTA's task list (tile coordinates), decoded once into shared memory at
// kernel start instead of by every role for every tile: 8 bytes per task.
constexpr int kTileListMax = 128;
constexpr int kTileListBytes = kTileListMax * 8;

// Warp roles.  Generic kernel (13 warps): 0-3 loaders (128 gather threads),
// 4-11 epilogue, 12 MMA.  Compact kernel (all-TMA operands, 12 warps = 384
// threads, which raises the register budget from 128 to 168 per thread):
// 0-2 TMA loaders, 3 MMA, 4-11 epilogue.  Epilogue warps stay 4-11 in both
// (TMEM lane group = warp % 4).
template <bool GENERIC>
struct Roles {
  static constexpr int kLoadWarps = GENERIC ? 4 : 3;
  static constexpr int kMmaWarp = GENERIC ? 4 + kEpiWarps : 3;
  static constexpr int kThreads = 32 * (GENERIC ? 4 + kEpiWarps + 1 : 4 + kEpiWarps);
};

// CG = CTAs per MMA (cta_group): 1, or 2 for the SM-pair form where the tile
// is (2*128) x BN, each CTA stages its 128 rows of A and BN/2 rows of B, and
// the pair leader issues tcgen05.mma.cta_group::2 over both CTAs' smem.
template <int BN, int STAGES, bool TF32, int CG = 1, bool GENERIC = true>
struct GemmCfg {
  static constexpr int kElem = TF32 ? 4 : 2;
  static constexpr int BK = kRowBytes / kElem;        // 64 bf16 / 32 tf32
  static constexpr int KSTEP = TF32 ? 8 : 16;          // K per tcgen05.mma
  static constexpr int NSTEP = BK / KSTEP;             // 4
  static constexpr int A_BYTES = kBM * kRowBytes;      // 16 KB
  static constexpr int B_BYTES = (BN / CG) * kRowBytes;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  // per epilogue warp group (one per TMEM accumulator): staged per-column operands
  static constexpr int COL_OPS = GENERIC ? kMaxEpiOps : 2;
  static constexpr int COLBUF_BYTES = 2 * COL_OPS * BN * 4;
  static constexpr int OUT_ROW = out_stage_row_bytes(BN, CG);      // bytes per lane per column group
  static constexpr int OUTBUF_BYTES = kEpiWarps * 32 * OUT_ROW;  // one staging buffer per epilogue warp
  // layout: [STAGES x (A | B)] [outbuf] [barriers 256 B] [colbuf]; the base is
  // 1024-byte aligned (checked at run time) as SWIZZLE_128B requires
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OUTBUF_BYTES + 256 + COLBUF_BYTES + kTileListBytes;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 must be 16..256 step 16");
};


// deepest ring (<= 8 stages) that fits next to the epilogue buffers
constexpr int stages_for(int bn, int cg, bool generic = true) {
  const int stage = kBM * kRowBytes + (bn / cg) * kRowBytes;
  const int fixed = kEpiWarps * 32 * out_stage_row_bytes(bn, cg) + 256 + 2 * (generic ? kMaxEpiOps : 2) * bn * 4 +
                    kTileListBytes;
  const int n = (kMaxSmem - fixed) / stage;
  return n > 8 ? 8 : n;
}

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

// Raw bits of one element converted to the MMA input format: fp32 (tf32
// kind), or the 16-bit format of the kind::f16 MMA -- bf16, or fp16 when `f16`.
// Same-format elements are copied bit for bit; others are rounded to nearest.
template <bool TF32>
__device__ __forceinline__ uint32_t load_bits(const void* base, int64_t idx, int32_t dt, bool f16) {
  if (TF32) {
    float f;
    if (dt == DT_F32) f = __ldg(reinterpret_cast<const float*>(base) + idx);
    else if (dt == DT_BF16) f = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
    else f = __half2float(reinterpret_cast<const __half*>(base)[idx]);
    return __float_as_uint(f);
  } else {
    if (dt == (f16 ? DT_F16 : DT_BF16)) return __ldg(reinterpret_cast<const unsigned short*>(base) + idx);
    const float f = dt == DT_F32 ? __ldg(reinterpret_cast<const float*>(base) + idx)
                    : dt == DT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx])
                                    : __half2float(reinterpret_cast<const __half*>(base)[idx]);
    if (f16) {
      __half h = __float2half_rn(f);
      return *reinterpret_cast<unsigned short*>(&h);
    }
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<unsigned short*>(&h);
  }
}

__device__ __forceinline__ float gelu_tanh(float x);

// Arithmetic prologue: load one element as fp32, apply the ops, convert to the
// MMA input format (tf32 bits, bf16 or fp16).
template <bool TF32>
__device__ __noinline__ uint32_t load_pre(const Strided& s, int64_t idx, bool f16) {
  float v = s.dtype == DT_F32    ? __ldg(reinterpret_cast<const float*>(s.ptr) + idx)
            : s.dtype == DT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(s.ptr)[idx])
                                 : __half2float(reinterpret_cast<const __half*>(s.ptr)[idx]);
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
      case EPI_EXP: v = __expf(v); break;
      case EPI_SQRT: v = sqrtf(v); break;
      case EPI_GELU_TANH: v = gelu_tanh(v); break;
      default: break;
    }
  }
  if (TF32) return __float_as_uint(v);
  if (f16) {
    __half h = __float2half_rn(v);
    return *reinterpret_cast<unsigned short*>(&h);
  }
  __nv_bfloat16 h = __float2bfloat16_rn(v);
  return *reinterpret_cast<unsigned short*>(&h);
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
                                                   int k0, int K, bool f16) {
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
      bits[j] = !(row_ok && k < K) ? 0u
                : s.n_pre ? load_pre<TF32>(s, base + (int64_t)k * s.s_k, f16)
                          : load_bits<TF32>(s.ptr, base + (int64_t)k * s.s_k, s.dtype, f16);
    }
    st_sw128(tile, r, c, pack_chunk<TF32>(bits));
  }
}

// Predicated im2col gather of one tile row (= one output pixel), the
// reference Col node (compute_ir.cpp:532-557): zero outside the padded image.
template <bool TF32, int BK>
__device__ __forceinline__ void gather_row_im2col(uint8_t* tile, int r, const ConvGeom& g,
                                                  int64_t pix, bool row_ok, int k0, int K, bool f16) {
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
                                     g.x_dtype, f16)
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

// Small-C im2col gather of one tile row (one output pixel) for k-block kb:
// BK/8 taps of one 16-byte pixel each (C <= 8 channels stored 16-byte padded,
// channels-last), as cp.async copies into the no-swizzle layout of
// LD_IM2COL_TMA8 ([tap][pixel][16 B]).  Asynchronous, so a loader thread runs
// ahead over the whole ring instead of waiting for each stage's loads.
// Padding taps and channels >= C are zero, as the reference Col node's select
// (compute_ir.cpp:539-553).
struct G8Row {
  int64_t base;  // pixel index of (img, 0, 0) in 16-byte units
  int bh, bw;    // top-left input coordinate of the output pixel's window
  bool ok;
};

// per tile: this thread's output pixel (tile row r)
__device__ __forceinline__ G8Row g8_row(const ConvGeom& g, int64_t pix, int64_t M) {
  G8Row rw;
  rw.ok = pix < M;
  const int hw = g.ho * g.wo;
  const int img = rw.ok ? static_cast<int>(pix / hw) : 0;
  const int rem = rw.ok ? static_cast<int>(pix - static_cast<int64_t>(img) * hw) : 0;
  const int oh = rem / g.wo, ow = rem - (rem / g.wo) * g.wo;
  rw.bh = oh * g.stride - g.pad;
  rw.bw = ow * g.stride - g.pad;
  rw.base = static_cast<int64_t>(img) * (g.sx[0] >> 3);
  return rw;
}

template <int BK>
__device__ __forceinline__ void gather_g8(uint8_t* tile, int r, const ConvGeom& g, const G8Row& rw, int kb) {
  static_assert(BK == 64, "8 taps of 8 channels per k-block");
  const uint4* x = reinterpret_cast<const uint4*>(g.x);  // one pixel = 16 B (pixel stride 8 elements)
  const int64_t s_h = g.sx[2] >> 3, s_w = g.sx[3] >> 3;
  const uint32_t nb = 2u * static_cast<uint32_t>(g.c);  // bytes of the c < C channels of a pixel
  const int taps = g.kh * g.kw;
  int tap = kb * 8;
  int fh = tap / g.kw, fw = tap - fh * g.kw;
  uint8_t* dst = tile + (r >> 3) * 1024 + (r & 7) * 16;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ih = rw.bh + fh, iw = rw.bw + fw;
    const bool ok = rw.ok && tap < taps && static_cast<unsigned>(ih) < static_cast<unsigned>(g.h) &&
                    static_cast<unsigned>(iw) < static_cast<unsigned>(g.w);
    // tap-adjacent no-swizzle layout: core matrix (8 rows x 16 B) of (row group, tap)
    // at (r / 8) * 1024 + j * 128 (LBO = 128 along K, SBO = 1024 along M);
    // padding taps copy 0 bytes (all zero), channels >= C are zero-filled
    ptx::cp_async16_ca(dst + j * 128, ok ? static_cast<const void*>(x + rw.base + ih * s_h + iw * s_w) : g.x,
                       ok ? nb : 0u);
    ++tap;
    if (++fw == g.kw) { fw = 0; ++fh; }
  }
}

// Filter gather of one tile row (= one output channel f) of Wf (the flatten
// node, compute_ir.cpp:558-569), any strides of W, either K order.
template <bool TF32, int BK>
__device__ __forceinline__ void gather_row_filter(uint8_t* tile, int r, const ConvGeom& g,
                                                  int64_t f, bool row_ok, int k0, int K, bool f16) {
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
                                     g.w_dtype, f16)
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

// strided / unaligned / ragged-edge fallback, one element per call and kept out
// of line (rare, and large once unrolled; scalar arguments stay in registers)
static __device__ __noinline__ float load_mat1(const void* ptr, int64_t idx, int32_t dt, bool ok) {
  return ok ? load_side(ptr, idx, dt) : 0.f;
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
  for (int j = 0; j < 16; ++j) out[j] = load_mat1(op.ptr, base + j * op.a.s_col, op.dtype, col0 + j < N);
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

// exp-based GELU (fp32 outputs), out of line: rare, and large unrolled 16x
static __device__ __noinline__ float gelu_precise1(float x) { return gelu_tanh(x); }

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
  const bool pre = p.canon_res_pre != 0;
  if (pre && p.canon_res_slot == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += mat[0][j];
  } else if (pre && p.canon_res_slot == 1) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += mat[1][j];
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
      for (int j = 0; j < 16; ++j) v[j] = gelu_precise1(v[j]);
    }
  }
  if (!pre && p.canon_res_slot == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += mat[0][j];
  } else if (!pre && p.canon_res_slot == 1) {
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

// one element of any output dtype (scalar fallback of store_out, out of line)
static __device__ __noinline__ void store1(void* out, int32_t dt, int64_t idx, float x) {
  if (dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(x);
  else if (dt == DT_F32) reinterpret_cast<float*>(out)[idx] = x;
  else reinterpret_cast<__half*>(out)[idx] = __float2half_rn(x);
}

// direct (non-TMA) store of 16 columns of one row
__device__ __forceinline__ void store_out(const GemmParams& p, const float (&v)[16], int64_t base,
                                          int64_t col0, bool row_ok) {
  if (!row_ok) return;
  const int64_t sc = p.out_a.s_col;
  const bool full = col0 + 16 <= p.N && sc == 1;
  if (full && p.out_dtype == DT_BF16) {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out);
    if ((reinterpret_cast<uintptr_t>(o + base + col0) & 15) == 0) {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      uint4* dst = reinterpret_cast<uint4*>(o + base + col0);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      return;
    }
  } else if (full && p.out_dtype == DT_F32) {
    float* o = reinterpret_cast<float*>(p.out);
    if ((reinterpret_cast<uintptr_t>(o + base + col0) & 15) == 0) {
      float4* dst = reinterpret_cast<float4*>(o + base + col0);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      return;
    }
  }
  // strided (e.g. NCHW: lanes = consecutive pixels, still coalesced) or ragged
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (col0 + j < p.N) store1(p.out, p.out_dtype, base + (col0 + j) * sc, v[j]);
}

// Fast-path drain of one accumulator tile for one warp (32 rows x ncols):
// canonical epilogue v = act(acc * S[c] + T[c]) (+ R[row, c]) with the
// activation / residual fixed at compile time, so each 32-column step is
// straight-line code: TMEM load (x32) -> FMA with the staged S/T -> act ->
// (+ bf16 residual, prefetched one step ahead) -> bf16 pack -> swizzled smem
// staging -> one TMA store per OUT_ROW-byte column group.  The accumulator is
// handed back to the MMA right after the last TMEM load.
// bf16x2 pack with ReLU folded into the conversion (one instruction per 2 outputs)
__device__ __forceinline__ uint32_t pack_relu_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// + the bf16 residual elements 4q .. 4q+3 of the 32 (words 2q, 2q+1 of rq[])
__device__ __forceinline__ void add_res4(float (&x)[4], const uint4 (&rq)[4], int q) {
  const uint32_t* rw = reinterpret_cast<const uint32_t*>(rq);
  const uint32_t w0 = rw[2 * q], w1 = rw[2 * q + 1];
  x[0] += __uint_as_float(w0 << 16);
  x[1] += __uint_as_float(w0 & 0xFFFF0000u);
  x[2] += __uint_as_float(w1 << 16);
  x[3] += __uint_as_float(w1 & 0xFFFF0000u);
}

#ifdef TMB_FINE_TRACE
// diagnostics build only (-DTMB_FINE_TRACE): clock64 at each drain step of the
// first epilogue warp, into trace rows 48.. of the CTA (tracing must be on)
#define TMB_FT(i) do { if (fine != nullptr && threadIdx.x == 128 && (i) < 256) fine[(i)] = clock64(); } while (0)
#else
#define TMB_FT(i) do { } while (0)
#endif

// F32OUT: fp32 output rows (OUT_ROW == 128: one 32-column group per TMEM load; no
// residual, no direct stores -- the host admits only those), the same FMA / ReLU.
template <int BN, int CG, int OUT_ROW, int ACT, int RES, bool F32OUT = false>
__device__ __forceinline__ void drain_fast(const CUtensorMap* tmC, uint32_t taddr, const float* colbuf,
                                           uint8_t* obuf, int ncols, int32_t col_base, int32_t row0,
                                           int32_t b, int lane, const uint4* res, uint64_t* tempty_bar,
                                           long long* fine = nullptr, __nv_bfloat16* drow = nullptr,
                                           int dcols = 0) {
  static_assert(!F32OUT || (OUT_ROW == 128 && RES == 0 && ACT <= 1), "fp32 lean drain: 128-byte rows, no residual");
  constexpr int GC = OUT_ROW / (F32OUT ? 4 : 2);  // output columns per TMA store group (32 or 64)
  int ft = 0;
  (void)fine;
  (void)ft;
  auto release = [&]() {  // the MMA may reuse this accumulator buffer
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(tempty_bar), 0));
      else ptx::mbar_arrive(tempty_bar);
    }
  };
  if (ncols <= 0) {  // nothing of this column range is inside the output
    release();
    return;
  }
  // this lane's staged row: OUT_ROW bytes, 16-byte chunks XOR-swizzled as the TMA store expects
  uint8_t* const orow = obuf + lane * OUT_ROW;
  const int swz = OUT_ROW == 128 ? (lane & 7) : ((lane >> 1) & 3);
  uint4 rq[4];
  if constexpr (RES) {
#pragma unroll
    for (int q = 0; q < 4; ++q) rq[q] = __ldg(res + q);
  }
#pragma unroll 1
  for (int c = 0; c < ncols; c += 32) {
    uint32_t r[32];
    TMB_FT(ft++);
    ptx::tmem_ld32(taddr + c, r);
    uint4 rn[4];
    if constexpr (RES) {
      if (c + 32 < ncols) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rn[q] = __ldg(res + (c + 32) / 8 + q);
      }
    }
    ptx::tmem_wait_ld();
    TMB_FT(ft++);
    if (c + 32 >= ncols) release();  // last TMEM read of this tile
    if (drow == nullptr && dcols >= 0 && c % GC == 0) {  // the previous store from this buffer has read it
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    }
    TMB_FT(ft++);
    if constexpr (F32OUT) {
      // 32 fp32 columns = the whole 128-byte staged row: 8 swizzled 16-byte chunks
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 sv = *reinterpret_cast<const float4*>(colbuf + c + 4 * q);
        const float4 tv = *reinterpret_cast<const float4*>(colbuf + BN + c + 4 * q);
        float x[4] = {fmaf(__uint_as_float(r[4 * q]), sv.x, tv.x), fmaf(__uint_as_float(r[4 * q + 1]), sv.y, tv.y),
                      fmaf(__uint_as_float(r[4 * q + 2]), sv.z, tv.z), fmaf(__uint_as_float(r[4 * q + 3]), sv.w, tv.w)};
        if constexpr (ACT == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) x[j] = fmaxf(x[j], 0.f);
        }
        *reinterpret_cast<uint4*>(orow + ((q ^ swz) << 4)) =
            make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(tmC, obuf, col_base + c, row0, b);
        ptx::bulk_commit();
      }
      continue;
    }
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 sv = *reinterpret_cast<const float4*>(colbuf + c + 4 * q);
      const float4 tv = *reinterpret_cast<const float4*>(colbuf + BN + c + 4 * q);
      float x[4] = {fmaf(__uint_as_float(r[4 * q]), sv.x, tv.x), fmaf(__uint_as_float(r[4 * q + 1]), sv.y, tv.y),
                    fmaf(__uint_as_float(r[4 * q + 2]), sv.z, tv.z), fmaf(__uint_as_float(r[4 * q + 3]), sv.w, tv.w)};
      if constexpr (ACT == 1 && !RES) {
        w[2 * q] = pack_relu_bf16x2(x[0], x[1]);
        w[2 * q + 1] = pack_relu_bf16x2(x[2], x[3]);
        continue;
      }
      if constexpr (RES == 2) add_res4(x, rq, q);  // act(acc*S + T + R)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (ACT == 1) x[j] = fmaxf(x[j], 0.f);
        if constexpr (ACT == 2) x[j] = gelu_tanh_fast(x[j]);
      }
      if constexpr (RES == 1) add_res4(x, rq, q);  // act(acc*S + T) + R
      w[2 * q] = pack_bf16x2(x[0], x[1]);
      w[2 * q + 1] = pack_bf16x2(x[2], x[3]);
    }
    TMB_FT(ft++);
    if (drow != nullptr || dcols < 0) {
      // direct: this lane's row segment straight from registers (16-byte stores,
      // whole 32-byte sectors over the 4 stores); no staging, proxy fence or TMA
      if (drow != nullptr) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c + 8 * k < dcols)
            *reinterpret_cast<uint4*>(drow + c + 8 * k) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
      }
      if constexpr (RES) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rq[q] = rn[q];
      }
      continue;
    }
    const int j0 = (c % GC) / 8;  // first 16-byte chunk of these 32 columns in the staged row
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(orow + (((j0 + k) ^ swz) << 4)) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    TMB_FT(ft++);
    if ((c + 32) % GC == 0 || c + 32 >= ncols) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(tmC, obuf, col_base + (c / GC) * GC, row0, b);
        ptx::bulk_commit();
      }
    }
    TMB_FT(ft++);
    if constexpr (RES) {
#pragma unroll
      for (int q = 0; q < 4; ++q) rq[q] = rn[q];
    }
  }
}

// Split-K final unit, lean form: sums the split partials of this warp's rows
// and column half from the fp32 workspace (chunk-major [split][col/16][128][16]),
// all of a 32-column chunk's loads in flight together, then the same canonical
// math / bf16 staging / TMA store as drain_fast.
template <int BN, int CG, int OUT_ROW, int ACT, int RES>
__device__ __forceinline__ void drain_reduce(const CUtensorMap* tmC, const float* ws, int split_k, int rloc,
                                             int cofs, const float* colbuf, uint8_t* obuf, int ncols,
                                             int32_t col_base, int32_t row0, int32_t b, int lane, const uint4* res,
                                             long long* tk = nullptr, long long t0 = 0) {
  constexpr int GC = OUT_ROW / 2;
  uint8_t* const orow = obuf + lane * OUT_ROW;
  const int swz = OUT_ROW == 128 ? (lane & 7) : ((lane >> 1) & 3);
#pragma unroll 1
  for (int c = 0; c < ncols; c += 32) {
    float x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = 0.f;
    // the workspace round trip is an L2 latency (~1-2k clk under load): issue
    // every split of a 16-column half-chunk before adding (up to 4 splits per
    // batch), then add in split order (deterministic)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll 1
      for (int sp0 = 0; sp0 < split_k; sp0 += 4) {
        float4 f[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4* src = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(min(sp0 + u, split_k - 1)) *
                                                                         (kBM * BN)) +
                              (static_cast<int64_t>((cofs + c) / 4 + 4 * h) * kBM + rloc);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            f[u][q] = sp0 + u < split_k ? __ldcg(src + q * kBM) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            x[16 * h + 4 * q] += f[u][q].x; x[16 * h + 4 * q + 1] += f[u][q].y;
            x[16 * h + 4 * q + 2] += f[u][q].z; x[16 * h + 4 * q + 3] += f[u][q].w;
          }
      }
    }
    if (tk != nullptr && c == 0 && lane == 0) tk[12] = clock64() - t0 + (static_cast<long long>(__float_as_int(x[0]) & 0) );
    uint4 rq[4];
    if constexpr (RES) {
#pragma unroll
      for (int q = 0; q < 4; ++q) rq[q] = __ldg(res + c / 8 + q);
    }
    if (c % GC == 0) {
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    }
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 sv = *reinterpret_cast<const float4*>(colbuf + c + 4 * q);
      const float4 tv = *reinterpret_cast<const float4*>(colbuf + BN + c + 4 * q);
      float y[4] = {fmaf(x[4 * q], sv.x, tv.x), fmaf(x[4 * q + 1], sv.y, tv.y), fmaf(x[4 * q + 2], sv.z, tv.z),
                    fmaf(x[4 * q + 3], sv.w, tv.w)};
      if constexpr (RES == 2) add_res4(y, rq, q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (ACT == 1) y[j] = fmaxf(y[j], 0.f);
        if constexpr (ACT == 2) y[j] = gelu_tanh_fast(y[j]);
      }
      if constexpr (RES == 1) add_res4(y, rq, q);
      w[2 * q] = pack_bf16x2(y[0], y[1]);
      w[2 * q + 1] = pack_bf16x2(y[2], y[3]);
    }
    const int j0 = (c % GC) / 8;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(orow + (((j0 + k) ^ swz) << 4)) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    if ((c + 32) % GC == 0 || c + 32 >= ncols) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(tmC, obuf, col_base + (c / GC) * GC, row0, b);
        ptx::bulk_commit();
      }
    }
    if (tk != nullptr && c == 0 && lane == 0) tk[13] = clock64() - t0;
  }
}

// Split-K final step with the tile's partials staged in shared memory (sk_spin):
// `stage` holds split_k slabs of this warp's 32 rows x ncols columns, layout
// [split][col/4][32 lanes] of float4 (slab_f4 float4 each); sums in split order
// (deterministic), then the same canonical math / staging / TMA store as
// drain_fast.
template <int BN, int CG, int OUT_ROW, int ACT, int RES>
__device__ __forceinline__ void drain_reduce_smem(const CUtensorMap* tmC, const float4* stage, int split_k,
                                                  int slab_f4, const float* colbuf, uint8_t* obuf, int ncols,
                                                  int32_t col_base, int32_t row0, int32_t b, int lane,
                                                  const uint4* res) {
  constexpr int GC = OUT_ROW / 2;
  uint8_t* const orow = obuf + lane * OUT_ROW;
  const int swz = OUT_ROW == 128 ? (lane & 7) : ((lane >> 1) & 3);
#pragma unroll 1
  for (int c = 0; c < ncols; c += 32) {
    float x[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 f = stage[(c / 4 + q) * 32 + lane];
      x[4 * q] = f.x; x[4 * q + 1] = f.y; x[4 * q + 2] = f.z; x[4 * q + 3] = f.w;
    }
#pragma unroll 1
    for (int sp = 1; sp < split_k; ++sp) {
      const float4* sl = stage + static_cast<int64_t>(sp) * slab_f4;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = sl[(c / 4 + q) * 32 + lane];
        x[4 * q] += f.x; x[4 * q + 1] += f.y; x[4 * q + 2] += f.z; x[4 * q + 3] += f.w;
      }
    }
    uint4 rq[4];
    if constexpr (RES) {
#pragma unroll
      for (int q = 0; q < 4; ++q) rq[q] = __ldg(res + c / 8 + q);
    }
    if (c % GC == 0) {
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    }
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 sv = *reinterpret_cast<const float4*>(colbuf + c + 4 * q);
      const float4 tv = *reinterpret_cast<const float4*>(colbuf + BN + c + 4 * q);
      float y[4] = {fmaf(x[4 * q], sv.x, tv.x), fmaf(x[4 * q + 1], sv.y, tv.y), fmaf(x[4 * q + 2], sv.z, tv.z),
                    fmaf(x[4 * q + 3], sv.w, tv.w)};
      if constexpr (RES == 2) add_res4(y, rq, q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (ACT == 1) y[j] = fmaxf(y[j], 0.f);
        if constexpr (ACT == 2) y[j] = gelu_tanh_fast(y[j]);
      }
      if constexpr (RES == 1) add_res4(y, rq, q);
      w[2 * q] = pack_bf16x2(y[0], y[1]);
      w[2 * q + 1] = pack_bf16x2(y[2], y[3]);
    }
    const int j0 = (c % GC) / 8;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(orow + (((j0 + k) ^ swz) << 4)) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    if ((c + 32) % GC == 0 || c + 32 >= ncols) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(tmC, obuf, col_base + (c / GC) * GC, row0, b);
        ptx::bulk_commit();
      }
    }
  }
}

// Decodes task `i` of this CTA into (batch, tile_m, tile_n); false once the
// CTA's task list is exhausted.  Out-of-range tasks are reported via `valid`.
__device__ __forceinline__ void trace(const GemmParams& p, uint32_t i, int ev, long long t0) {
  if (p.trace != nullptr && i < static_cast<uint32_t>(kTraceTiles))
    p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + i) * kTraceEvents + ev] = clock64() - t0;
}

template <int CG>
__device__ __forceinline__ bool decode_tile(const GemmParams& p, uint32_t i, int& b, int& ks, int& tm_, int& tn,
                                            bool& valid) {
  if (i >= p.tile_map.tasks) return false;
  int32_t c[tm::kMaxRank];
  tm::dev_task_fixed<2, 3>(p.tile_map, blockIdx.x / CG, i, c);  // workers = CTA pairs when CG == 2
  b = c[0] / p.split_k;
  ks = c[0] % p.split_k;
  tm_ = c[1];
  tn = c[2];
  valid = b < p.batch && tm_ < p.tiles_m && tn < p.tiles_n;
  return true;
}

__device__ __forceinline__ bool use_tile_list(const GemmParams& p) {
  return p.tile_map.tasks <= static_cast<uint32_t>(kTileListMax) && p.tiles_m < 65536 && p.tiles_n < 65536;
}

// task i of this CTA from the shared-memory list (entry: tm:16 | tn:16 | b*split_k+ks:31 | valid:1),
// or decoded when the list overflowed
template <int CG>
__device__ __forceinline__ bool next_tile(const GemmParams& p, const uint2* list, uint32_t i, int& b, int& ks,
                                          int& tm_, int& tn, bool& valid) {
  if (i >= p.tile_map.tasks) return false;
  if (!use_tile_list(p)) return decode_tile<CG>(p, i, b, ks, tm_, tn, valid);
  const uint2 e = list[i];
  tm_ = static_cast<int>(e.x & 0xFFFFu);
  tn = static_cast<int>(e.x >> 16);
  const int bk = static_cast<int>(e.y >> 1);
  b = bk / p.split_k;
  ks = bk - b * p.split_k;
  valid = (e.y & 1u) != 0u;
  return true;
}

}  // namespace detail

template <int BN, int STAGES, bool TF32, int CG, bool GENERIC>
__global__ void __launch_bounds__(Roles<GENERIC>::kThreads, 1)
    tm_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC) {
  using Cfg = GemmCfg<BN, STAGES, TF32, CG, GENERIC>;
  constexpr int BK = Cfg::BK;
  constexpr int kTileM = kBM * CG;  // rows per tile (both CTAs of a pair)
  // MN-major B: one 128-byte swizzle row holds MNB elements along N (64 bf16 / 32
  // tf32); a block of MNB columns x BK k-rows occupies BK * 128 bytes of the slot
  constexpr int MNB = kRowBytes / Cfg::kElem;
  constexpr int MN_BLOCK_BYTES = BK * kRowBytes;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((ptx::smem_u32(smem_raw) & 1023u) != 0u) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint8_t* smem = smem_raw;
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* outbuf = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + Cfg::OUTBUF_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* split_flag = tmem_slot + 1;  // [2], one per epilogue warp group
  // [8] per epilogue warp: partial slabs bulk-copied into the idle ring (sk_spin)
  uint64_t* rbar = reinterpret_cast<uint64_t*>(outbuf + Cfg::OUTBUF_BYTES) + 22;
  float* colbuf_all = reinterpret_cast<float*>(outbuf + Cfg::OUTBUF_BYTES + 256);
  uint2* tile_list = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(colbuf_all) + Cfg::COLBUF_BYTES);

  const uint64_t gt_entry = p.trace != nullptr ? ptx::globaltimer() : 0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool a_tma = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA || p.a_loader == LD_IM2COL_TMA8;
  const bool b_tma = p.b_loader == LD_TMA_K || p.b_loader == LD_TMA_MN;
  const bool all_tma = a_tma && b_tma;

  const int skip = p.dbg == 1 ? p.dbg_skip : 0;
  if (threadIdx.x == 0 && !(skip & 2)) {
    if (a_tma) ptx::tma_prefetch_desc(&tmA);
    if (b_tma) ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      // all-TMA: the A and B issuing warps; gather: every loader thread (dbg 4: one per warp)
      ptx::mbar_init(&full[s], all_tma ? 2 : (p.dbg == 4 ? 4 : 128));
      ptx::mbar_init(&empty[s], 1);
    }
    for (int w = 0; w < kEpiWarps; ++w) ptx::mbar_init(&rbar[w], 1);
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      // drained by: the group's 4 warps, or all 8 when the groups split columns (of both CTAs)
      ptx::mbar_init(&tempty[a], ((!GENERIC || p.epi_fast) && (CG == 1 || p.split_k == 1) && BN % 64 == 0 ? 8 : 4) * CG);
    }
    ptx::fence_mbar_init();
  }
  using R = Roles<GENERIC>;
  if (detail::use_tile_list(p) && p.tile_tab != nullptr) {
    // the bind-time table: one 8-byte load per task (L2-resident after the first launch)
    const uint2* tab = reinterpret_cast<const uint2*>(p.tile_tab) + static_cast<size_t>(blockIdx.x / CG) * p.tile_map.tasks;
    for (uint32_t i = threadIdx.x; i < p.tile_map.tasks; i += blockDim.x) tile_list[i] = __ldg(tab + i);
  } else if (detail::use_tile_list(p) && !(skip & 1)) {
    for (uint32_t i = threadIdx.x; i < p.tile_map.tasks; i += blockDim.x) {
      int b, ks, tm_, tn;
      bool valid;
      detail::decode_tile<CG>(p, i, b, ks, tm_, tn, valid);
      tile_list[i] = valid ? make_uint2(static_cast<uint32_t>(tm_) | (static_cast<uint32_t>(tn) << 16),
                                        (static_cast<uint32_t>(b * p.split_k + ks) << 1) | 1u)
                           : make_uint2(0u, 0u);
    }
  }
  if (warp == R::kMmaWarp && !(skip & 4)) {
    if constexpr (CG == 2) ptx::tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
    else ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer barriers initialised before any TMA/arrive
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, descriptor prefetch) overlapped the previous kernel's tail;
  // from here on this grid reads its inputs and writes its outputs, so wait
  // for the previous grid, and let the next one start placing CTAs.
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  // ring depth in use (a multiple of num_kb for weight-stationary B, else STAGES)
  const int ring = (p.ring > 0 && p.ring <= STAGES) ? p.ring : STAGES;
  const long long t0 = clock64();
  if (p.trace != nullptr && threadIdx.x == 0) {  // ns: kernel entry, setup done (tile 0's slots 7, 14)
    long long* tr0 = p.trace + static_cast<int64_t>(blockIdx.x) * kTraceTiles * kTraceEvents;
    tr0[TR_CTA_START] = static_cast<long long>(gt_entry);
    tr0[14] = static_cast<long long>(ptx::globaltimer());
  }

  if (p.dbg == 1) {
    // diagnostics: setup + teardown only
  } else if (warp < R::kLoadWarps) {
    // ===================== loaders (prologue splice) =====================
    // All-TMA operands: lane 0 of each of the 4 loader warps issues every 4th
    // ring slot (slot q -> warp q % 4).  TMA copies issued by one thread are
    // serviced one after another (~600 clk per box, nearly size-independent,
    // measured by scripts/tmabench.cu), so a single issuing thread caps a CTA
    // near 30 B/clk; four issuing warps run four copy streams in parallel.
    const int t = threadIdx.x;  // 0..127
    const uint32_t lw = static_cast<uint32_t>(t >> 5);
    if (all_tma && (t & 31) != 0) {
      // idle lanes
    } else {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t q = 0;  // ring slot sequence number
      int b, ks, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile<CG>(p, tile_list, i, b, ks, tm_, tn, valid); ++i) {
        if (!valid) continue;
        // this CTA's rows of A and columns of B (half of each tile's B when CG == 2)
        const int m0 = tm_ * kTileM + rank * kBM, n0 = tn * BN + rank * (BN / CG);
        detail::G8Row g8{};
        if (GENERIC && p.a_loader == LD_IM2COL_G8) g8 = detail::g8_row(p.conv, m0 + t, p.M);
        for (int kb0 = ks * p.kb_per_split, kb = kb0, kb_end = min(p.num_kb, kb0 + p.kb_per_split); kb < kb_end; ++kb, ++q) {
          // all-TMA: slot q's A comes from warp 2q mod L, its B from warp 2q+1 mod L
          // (full barrier count 2).  Only those two warps wait for the slot's empty
          // barrier.  A warp that also polled the slots it does not own could be
          // lapped: the owners refill slot q and the MMA consumes it before the
          // bystander polls, the barrier is then two phases past the one it waits
          // for, the parity test aliases, and the bystander -- owner of slot q+1 --
          // never issues again (the round-1 intermittent hang).  A warp owns at
          // least one slot of every `ring` consecutive ones (L <= 4, ring >= 2), so
          // an owner is never more than one phase ahead of the barrier either.
          const bool do_a = (2u * q) % R::kLoadWarps == lw, do_b = (2u * q + 1u) % R::kLoadWarps == lw;
          if (all_tma && !do_a && !do_b) {
            if (++stage == ring) { stage = 0; phase ^= 1u; }
            continue;
          }
          if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&empty[stage], phase ^ 1u);
          // loader warps poll their empty slots instead of parking on them: the ring's
          // MMA-commit -> refill round trip is what bounds small tiles (measured: ~300
          // clk per slot with no copies and no MMAs), and a parked warp adds its
          // wake-up latency to it (-3..4% on the ResNet layers); the MMA warp keeps the
          // suspending wait (polling it measured no better)
          else ptx::mbar_wait_poll(&empty[stage], phase ^ 1u);
          uint8_t* a_tile = smA + stage * Cfg::A_BYTES;
          uint8_t* b_tile = smB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          const bool b_stays = p.b_resident && q >= static_cast<uint32_t>(ring);
          if (all_tma) {
            if (p.dbg == 3 || p.dbg == 7) {  // diagnostics: no copies (MMA on stale smem) -> MMA + epilogue floor
              if (do_a || do_b) {
                if constexpr (CG == 2) {
                  if (rank == 0) ptx::mbar_arrive(&full[stage]);
                } else {
                  ptx::mbar_arrive(&full[stage]);
                }
              }
            } else if (do_a || do_b) {
              if (kb == kb0) detail::trace(p, i, TR_PROD_FIRST, t0);
              if (kb == kb_end - 1) detail::trace(p, i, TR_PROD_LAST, t0);
              if constexpr (CG == 2) {
                // both CTAs' TMA bytes complete on the leader's full barrier
                const uint32_t lead_full = ptx::mapa_shared(ptx::smem_u32(&full[stage]), 0);
                if (do_a) {
                  if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * Cfg::A_BYTES);
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
                }
                if (do_b && b_stays) {
                  if (rank == 0) ptx::mbar_arrive(&full[stage]);  // B already resident in this slot
                } else if (do_b) {
                  if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * Cfg::B_BYTES);
                  if (p.b_loader == LD_TMA_K) {
                    ptx::tma_load_3d_2sm(b_tile, &tmB, lead_full, k0, n0, b);
                  } else {
                    if (p.b_mn4d) {
                      ptx::tma_load_4d_2sm(b_tile, &tmB, lead_full, 0, k0, n0 / MNB, b);
                    } else {
#pragma unroll 1
                      for (int j = 0; j < BN / CG / MNB; ++j)
                        ptx::tma_load_3d_2sm(b_tile + j * MN_BLOCK_BYTES, &tmB, lead_full, n0 + MNB * j, k0, b);
                    }
                  }
                }
              } else {
                if (do_a) {
                  ptx::mbar_arrive_expect_tx(&full[stage], Cfg::A_BYTES);
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
                    ptx::tma_load_im2col_4d(a_tile, &tmA, &full[stage], cb * BK, ow * p.conv.stride - p.conv.pad,
                                            oh * p.conv.stride - p.conv.pad, img, static_cast<uint16_t>(fw),
                                            static_cast<uint16_t>(fh));
                  } else {  // LD_IM2COL_TMA8
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
                      ptx::tma_load_im2col_4d(a_tile + j * 2048, &tmA, &full[stage], 0,
                                              ow * p.conv.stride - p.conv.pad, oh * p.conv.stride - p.conv.pad, img,
                                              static_cast<uint16_t>(tap % p.conv.kw),
                                              static_cast<uint16_t>(tap / p.conv.kw));
                    }
                  }
                }
                if (do_b && b_stays) {
                  ptx::mbar_arrive(&full[stage]);  // B already resident in this slot
                } else if (do_b) {
                  ptx::mbar_arrive_expect_tx(&full[stage], Cfg::B_BYTES);
                  if (p.b_loader == LD_TMA_K) {
                    ptx::tma_load_3d(b_tile, &tmB, &full[stage], k0, n0, b);
                  } else {
                    if (p.b_mn4d) {
                      ptx::tma_load_4d(b_tile, &tmB, &full[stage], 0, k0, n0 / MNB, b);
                    } else {
#pragma unroll 1
                      for (int j = 0; j < BN / MNB; ++j)
                        ptx::tma_load_3d(b_tile + j * MN_BLOCK_BYTES, &tmB, &full[stage], n0 + MNB * j, k0, b);
                    }
                  }
                }
              }
            }
            if (++stage == ring) { stage = 0; phase ^= 1u; }
            continue;
          }
          // ---- mixed / gather mode (GENERIC): lane 0 of warp q % 4 issues the slot's
          // TMA operand (TMA copies from one thread are serviced serially), all 128 gather
          const bool issuer = t == static_cast<int>((q & 3u) << 5);
          if (kb == kb0 && issuer) detail::trace(p, i, TR_PROD_FIRST, t0);
          if (kb == kb_end - 1 && issuer) detail::trace(p, i, TR_PROD_LAST, t0);
          if constexpr (CG == 2) {
            __trap();  // the CTA-pair form is instantiated for TMA operands only
          }
          if (issuer) {
            // mixed mode: announce the TMA bytes now, arrive after the gather
            const uint32_t tx = (a_tma ? Cfg::A_BYTES : 0) + (b_tma && !b_stays ? Cfg::B_BYTES : 0);
            if (tx) ptx::mbar_expect_tx(&full[stage], tx);
          }
          if (issuer) {
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
            if (b_stays) {
              // weight-stationary: this slot's B is already resident
            } else if (p.b_loader == LD_TMA_K) {
              ptx::tma_load_3d(b_tile, &tmB, &full[stage], k0, n0, b);
            } else if (p.b_loader == LD_TMA_MN) {
              if (p.b_mn4d) {
                ptx::tma_load_4d(b_tile, &tmB, &full[stage], 0, k0, n0 / MNB, b);
              } else {
#pragma unroll 1
                for (int j = 0; j < BN / MNB; ++j)
                  ptx::tma_load_3d(b_tile + j * MN_BLOCK_BYTES, &tmB, &full[stage], n0 + MNB * j,
                                   k0, b);
              }
            }
          }
          if (GENERIC && !all_tma) {
            // predicated gather of the non-TMA operand(s), one tile row per thread
            if (!a_tma) {
              const int64_t row = m0 + t;
              const bool ok = row < p.M;
              if (p.a_loader == LD_GATHER)
                detail::gather_row_strided<TF32, BK>(a_tile, t, p.a, row, ok, b, k0, p.K, p.ab_f16 != 0);
              else if (p.a_loader == LD_IM2COL_G8) {
                if constexpr (!TF32) {
                  if (p.dbg != 3 && p.dbg != 4) detail::gather_g8<BK>(a_tile, t, p.conv, g8, kb);  // async, arrives below
                }
              } else {
                detail::gather_row_im2col<TF32, BK>(a_tile, t, p.conv, row, ok, k0, p.K, p.ab_f16 != 0);
              }
            }
            if (!b_tma && !b_stays) {
#pragma unroll 1
              for (int r = t; r < BN; r += 128) {
                const int64_t row = n0 + r;
                const bool ok = row < p.N;
                if (p.b_loader == LD_GATHER)
                  detail::gather_row_strided<TF32, BK>(b_tile, r, p.b, row, ok, b, k0, p.K, p.ab_f16 != 0);
                else
                  detail::gather_row_filter<TF32, BK>(b_tile, r, p.conv, row, ok, k0, p.K, p.ab_f16 != 0);
              }
            }
            if (p.dbg == 4) {  // diagnostics: no gather, one arrival per warp
              __syncwarp();
              if ((t & 31) == 0) ptx::mbar_arrive(&full[stage]);
            } else if (p.a_loader == LD_IM2COL_G8 && b_tma) {
              ptx::cp_async_arrive_noinc(&full[stage]);  // when this thread's copies land
            } else {
              if (p.a_loader == LD_IM2COL_G8) asm volatile("cp.async.wait_all;" ::: "memory");
              ptx::fence_proxy_async_smem();
              ptx::mbar_arrive(&full[stage]);
            }
          }
          if (++stage == ring) { stage = 0; phase ^= 1u; }
        }
      }
      // Producer tail: wait until the MMA's commits for the last `ring` slots have
      // arrived on this CTA's empty barriers (the pair leader multicasts them to
      // both CTAs).  Without it a commit can still be in flight when the CTA exits
      // and land in the shared memory of the next CTA placed on this SM -- e.g.
      // the barriers a programmatically launched successor has just initialised.
      for (int j = 0; j < ring; ++j, ++q) {
        const bool own = !all_tma || (2u * q) % R::kLoadWarps == lw || (2u * q + 1u) % R::kLoadWarps == lw;
        if (own) {
          if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&empty[stage], phase ^ 1u);
          // loader warps poll their empty slots instead of parking on them: the ring's
          // MMA-commit -> refill round trip is what bounds small tiles (measured: ~300
          // clk per slot with no copies and no MMAs), and a parked warp adds its
          // wake-up latency to it (-3..4% on the ResNet layers); the MMA warp keeps the
          // suspending wait (polling it measured no better)
          else ptx::mbar_wait_poll(&empty[stage], phase ^ 1u);
        }
        if (++stage == ring) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    // ===================== epilogue (epilogue splice) =====================
    // Two warp groups, one per TMEM accumulator buffer: group h drains the
    // CTA's tiles 1 mod 2 == h, so two tiles' epilogues overlap and each warp
    // (TMEM lane group lg = warp % 4: rows lg*32 .. +32 of the tile) walks the
    // whole tile width.  Output columns go out in groups of OUT_ROW bytes per
    // row: 32 rows are staged in this warp's swizzled smem buffer and written
    // by one TMA store.
    const int e = warp - 4;                // 0..7
    const int lg = warp & 3;               // TMEM lane group this warp may access
    const int grp = e >> 2;                // warp group = accumulator buffer it drains
    const int gt = threadIdx.x - 128 - grp * 128;  // thread index within the group (0..127)
    const bool lead = (e & 3) == 0 && lane == 0;  // traces / counters
    constexpr int kChunks = BN / 16;
    float* colbuf = colbuf_all + grp * (Cfg::COL_OPS * BN);
    uint32_t acc_phase = 0;
    int b, ks, tm_, tn;
    bool valid;
    int64_t rowpart[kMaxEpiOps];
    float rowv[kMaxEpiOps];
    bool has_col = false;
    for (int o = 0; o < p.n_ops; ++o) has_col = has_col || p.ops[o].side == SIDE_COL;
    int staged_tn = -1, staged_b = -1;
    uint8_t* obuf = outbuf + e * (32 * Cfg::OUT_ROW);
    const int obytes = p.out_dtype == DT_F32 ? 4 : 2;
    const int gcols = Cfg::OUT_ROW / obytes;  // columns per TMA-store group
    // 16-byte chunk j of this lane's staged row, with the TMA swizzle applied
    auto stage_at = [&](int j) -> uint4* {
      uint32_t a = static_cast<uint32_t>(lane * Cfg::OUT_ROW + j * 16);
      a ^= ((a >> 7) & (Cfg::OUT_ROW == 128 ? 7u : 3u)) << 4;
      return reinterpret_cast<uint4*>(obuf + a);
    };
    // 16 finished columns (tile column c) -> staging buffer or global memory
    auto put16 = [&](const float (&v)[16], int c, int64_t obase_, int64_t n0_, bool row_ok_) {
      if (p.dbg == 2) return;  // diagnostics: no output stores
      if (!p.out_tma) {
        detail::store_out(p, v, obase_, n0_ + c, row_ok_);
        return;
      }
      const int j0 = (c % gcols) * obytes / 16;
      if (obytes == 2) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          w[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        *stage_at(j0) = make_uint4(w[0], w[1], w[2], w[3]);
        *stage_at(j0 + 1) = make_uint4(w[4], w[5], w[6], w[7]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *stage_at(j0 + q) = make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                                         __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
      }
    };
    // before the first put16 of a column group: the previous store has read the buffer
    auto group_begin = [&]() {
      if (!p.out_tma) return;
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    };
    auto group_end = [&](int64_t col0, int tile_row0) {
      if (!p.out_tma || p.dbg == 2) return;
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(&tmC, obuf, static_cast<int32_t>(col0), tile_row0, b);
        ptx::bulk_commit();
      }
    };
    auto release_acc = [&](uint32_t buf) {
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // the (leader's) MMA may overwrite this accumulator once both CTAs drained it
        if constexpr (CG == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&tempty[buf]), 0));
        else ptx::mbar_arrive(&tempty[buf]);
      }
    };
    uint32_t nvalid = 0;
    // (CTA-pair split-K keeps the one-group-per-unit path: the lean split form hung in
    // back-to-back launches of the CG=2 FFN chain, scripts/space_probe.py config 56)
    // lean drain (drain_fast) for canonical bf16 epilogues; the two groups split each
    // tile's columns when the halves are whole 32-column chunks (BN % 64 == 0),
    // otherwise they alternate tiles, full width
    const bool lean = !GENERIC || p.epi_fast;
    const bool colsplit = lean && (CG == 1 || p.split_k == 1) && BN % 64 == 0;
    uint32_t acc_phase2[2] = {0u, 0u};  // colsplit: per-buffer phase
    // canonical S / T of columns gt and gt + 128 of tile column block tn_ (batch b_)
    auto fetch_st = [&](int tn_, int b_, float (&s_v)[2], float (&t_v)[2]) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = static_cast<int64_t>(tn_) * BN + gt + 128 * h;
        const bool in = gt + 128 * h < BN && col < p.N;
        s_v[h] = p.canon_s;
        t_v[h] = p.canon_t;
        if (p.canon_s_op >= 0 && in) {
          const EpiOp& op = p.ops[p.canon_s_op];
          s_v[h] = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, b_) + col * op.a.s_col, op.dtype);
        }
        if (p.canon_t_op >= 0 && in) {
          const EpiOp& op = p.ops[p.canon_t_op];
          t_v[h] = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, b_) + col * op.a.s_col, op.dtype);
        }
      }
    };
    float pf_s[2] = {0.f, 0.f}, pf_t[2] = {0.f, 0.f};
    int pf_tn = -1, pf_b = -1;
    for (uint32_t i = 0; detail::next_tile<CG>(p, tile_list, i, b, ks, tm_, tn, valid); ++i) {
      if (!valid) continue;
      // accumulator buffer = tile parity.  Compact kernel (no split-K): both groups
      // drain every tile, group g the column half g (a tile's drain takes half as
      // long, which is what the last tile of a CTA exposes); otherwise group g
      // drains the tiles of parity g, full width.
      const uint32_t abuf = nvalid++ & 1u;
      if (!colsplit && abuf != static_cast<uint32_t>(grp)) continue;  // the other group's tile
      const int64_t n0 = static_cast<int64_t>(tn) * BN;
      const int tile_row0 = tm_ * kTileM + rank * kBM;
      const int row0 = tile_row0 + lg * 32;  // this warp's first row
      const int64_t row = static_cast<int64_t>(row0) + lane;
      const bool row_ok = row < p.M;
      const int64_t rr = row_ok ? row : 0;
      // Stage this tile's column vectors while the MMA works on it; skipped when
      // the group's previous tile had the same columns (e.g. every tile of a conv
      // whose F fits one tile), which keeps the load latency off the critical path.
      const bool restage = (staged_tn < 0 && (has_col || p.canon)) || (has_col && (tn != staged_tn || b != staged_b));
      if (restage) ptx::named_bar_sync(1 + grp, 128);  // the group's previous readers are done
      if (restage && p.canon) {  // S and T column vectors of the canonical epilogue
        float s_v[2], t_v[2];
        if (pf_tn == tn && pf_b == b) {  // prefetched while the previous tile drained
          s_v[0] = pf_s[0]; s_v[1] = pf_s[1]; t_v[0] = pf_t[0]; t_v[1] = pf_t[1];
        } else {
          fetch_st(tn, b, s_v, t_v);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = gt + 128 * h;
          if (c < BN) {
            colbuf[c] = s_v[h];
            colbuf[BN + c] = t_v[h];
          }
        }
      }
      if (p.canon && has_col) {
        // look ahead to this group's next tile; if its columns differ, start
        // loading its S / T now so the loads overlap this tile's drain
        pf_tn = -1;
        int nb_, nks_, ntm_, ntn_;
        bool nv_;
        uint32_t need = colsplit ? 1u : 2u;
        for (uint32_t j = i + 1; detail::next_tile<CG>(p, tile_list, j, nb_, nks_, ntm_, ntn_, nv_); ++j) {
          if (!nv_) continue;
          if (--need == 0) {
            if (ntn_ != tn || nb_ != b) {
              fetch_st(ntn_, nb_, pf_s, pf_t);
              pf_tn = ntn_;
              pf_b = nb_;
            }
            break;
          }
        }
      }
      if constexpr (GENERIC) {
#pragma unroll 1
        for (int o = 0; o < p.n_ops; ++o) {
          const EpiOp& op = p.ops[o];
          rowpart[o] = detail::addr_rowpart(op.a, rr, b);
          if (op.side == SIDE_COL && restage && !p.canon) {
            const int64_t cb = detail::addr_rowpart(op.a, 0, b);
            for (int c = gt; c < BN; c += 128)
              colbuf[o * BN + c] = (n0 + c < p.N) ? detail::load_side(op.ptr, cb + (n0 + c) * op.a.s_col, op.dtype) : 0.f;
          } else if (op.side == SIDE_ROW) {
            rowv[o] = row_ok ? detail::load_side(op.ptr, rowpart[o], op.dtype) : 0.f;
          }
        }
      } else if (p.canon_res_op >= 0) {  // canonical form: the residual is the only per-element operand
        rowpart[0] = detail::addr_rowpart(p.ops[p.canon_res_op].a, rr, b);
      }
      const int64_t obase = p.out_tma ? 0 : detail::addr_rowpart(p.out_a, rr, b);
      if (restage) {
        ptx::named_bar_sync(1 + grp, 128);  // column buffers ready
        staged_tn = tn;
        staged_b = b;
      }
      if (lead) detail::trace(p, i, TR_EPI_READY, t0);
      float mat[kMaxMatOps][16];
      auto prefetch = [&](int c, float (&dst)[kMaxMatOps][16]) {
        if constexpr (!GENERIC) {
          if (p.canon_res_op >= 0)  // slot 0: the canonical form has one matrix operand
            detail::load_mat16(p.ops[p.canon_res_op], rowpart[0], n0 + c * 16, p.N, row_ok, dst[0]);
          return;
        }
#pragma unroll 1
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
      if (GENERIC && !colsplit && p.has_mat && p.split_k == 1) prefetch(0, mat);
      if (colsplit) {
        if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&tfull[abuf], acc_phase2[abuf]);
        else ptx::mbar_wait(&tfull[abuf], acc_phase2[abuf]);
        acc_phase2[abuf] ^= 1u;
      } else {
        if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&tfull[grp], acc_phase);
        else ptx::mbar_wait(&tfull[grp], acc_phase);
        acc_phase ^= 1u;
      }
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + abuf * BN;
      if (lead) detail::trace(p, i, TR_EPI_ACC, t0);
      const int ncols = static_cast<int>(min(static_cast<int64_t>(BN), p.N - n0));  // valid columns
      if (CG == 1 && p.split_k > 1 && colsplit) {
        // ---- split-K, lean form: each group parks its column half of the raw partial
        // tile; the group that completes a (tile, half) last reduces it and stores
        constexpr int kHalf = BN / 2;
        const int cofs = grp * kHalf;
        const int hcols = max(0, min(kHalf, ncols - cofs));
        const int64_t tile_id = ((static_cast<int64_t>(b) * p.tiles_m + tm_) * p.tiles_n + tn) * CG + rank;
        const float* ws = p.workspace + tile_id * p.split_k * static_cast<int64_t>(kBM * BN);
        const int rloc = lg * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < kHalf; c += 32) {
          uint32_t r[32];
          ptx::tmem_ld32(taddr + cofs + c, r);
          ptx::tmem_wait_ld();
          // layout [split][col/4][128 rows] of float4: each store instruction of a
          // warp writes 512 contiguous bytes (whole lines), and the reader uses the
          // same lane -> row mapping
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4* split_base = reinterpret_cast<float4*>(const_cast<float*>(ws) + ks * static_cast<int64_t>(kBM * BN));
              // sk_spin: per-warp slabs [grp][lg][col/4][32 lanes] (one contiguous block
              // per 32 rows x half, bulk-copied by the reducer)
              float4* dst = p.sk_spin
                                ? split_base + ((grp * 4 + lg) * (kHalf / 4) + (c / 4 + 4 * h + q)) * 32 + lane
                                : split_base + (static_cast<int64_t>((cofs + c) / 4 + 4 * h + q) * kBM + rloc);
              __stcg(dst, make_float4(__uint_as_float(r[16 * h + 4 * q]), __uint_as_float(r[16 * h + 4 * q + 1]),
                                      __uint_as_float(r[16 * h + 4 * q + 2]), __uint_as_float(r[16 * h + 4 * q + 3])));
            }
          }
        }
        release_acc(abuf);  // TMEM is free again: the MMA can start the next unit
        if (lead) detail::trace(p, i, 8, t0);
        __threadfence();
        if (lead) detail::trace(p, i, 9, t0);
        ptx::named_bar_sync(3 + grp, 128);
        if (p.sk_spin) {
          if (gt == 0) {
            uint32_t* ctr = reinterpret_cast<uint32_t*>(&p.counters[tile_id * 2 + grp]);
            const uint32_t sk = static_cast<uint32_t>(p.split_k);
            const uint32_t target = (atomicAdd(ctr, 1u) / sk + 1u) * sk;
            while (static_cast<int32_t>(ptx::ld_acquire_u32(ctr) - target) < 0) __nanosleep(64);
          }
          ptx::named_bar_sync(3 + grp, 128);
          if (lead) detail::trace(p, i, 10, t0);
          if (lg % p.split_k != ks) continue;  // another unit of this tile reduces these rows
        } else {
          if (gt == 0) split_flag[grp] = (atomicAdd(&p.counters[tile_id * 2 + grp], 1) == p.split_k - 1) ? 1u : 0u;
          ptx::named_bar_sync(3 + grp, 128);
          if (lead) detail::trace(p, i, 10, t0);
          if (*reinterpret_cast<volatile uint32_t*>(&split_flag[grp]) == 0u) continue;
        }
        __threadfence();
        const uint4* res = nullptr;
        if (p.canon_res_op >= 0)  // rr is row 0 for rows past M (their stores are clipped)
          res = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ops[p.canon_res_op].ptr) +
                                               detail::addr_rowpart(p.ops[p.canon_res_op].a, rr, b) + n0 + cofs);
        const int32_t cbase = static_cast<int32_t>(n0) + cofs;
        long long* tk = (p.trace != nullptr && e == 0 && i < static_cast<uint32_t>(kTraceTiles))
                            ? p.trace + (static_cast<int64_t>(blockIdx.x) * kTraceTiles + i) * kTraceEvents
                            : nullptr;
        if (tk != nullptr && lane == 0) tk[7] = clock64() - t0;  // reduce start (after the fence)
        if (p.sk_spin) {
          // the ring is idle (one unit per CTA): this warp's split_k slabs of 32 rows x
          // the half's columns land there by bulk copies (full bandwidth, no register
          // round trips), then sum from shared memory
          const int slab_f4 = (kHalf / 4) * 32;
          const int reducer = grp * (4 / p.split_k) + lg / p.split_k;
          float4* stage = reinterpret_cast<float4*>(smA) + static_cast<int64_t>(reducer) * p.split_k * slab_f4;
          if (lane == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");  // peers' stores -> async-proxy reads
            const uint32_t slab_b = static_cast<uint32_t>(slab_f4 * 16);
            ptx::mbar_arrive_expect_tx(&rbar[e], slab_b * static_cast<uint32_t>(p.split_k));
            for (int sp = 0; sp < p.split_k; ++sp)
              ptx::bulk_load(stage + static_cast<int64_t>(sp) * slab_f4,
                             reinterpret_cast<const float4*>(p.workspace + tile_id * p.split_k * static_cast<int64_t>(kBM * BN) +
                                                             sp * static_cast<int64_t>(kBM * BN)) +
                                 (grp * 4 + lg) * slab_f4,
                             slab_b, &rbar[e]);
          }
          ptx::mbar_wait(&rbar[e], 0);
          switch (p.canon_act * 3 + (p.canon_res_op < 0 ? 0 : p.canon_res_pre ? 2 : 1)) {
#define TMB_REDS(A, R)                                                                                             \
  case A * 3 + R:                                                                                                  \
    detail::drain_reduce_smem<BN, CG, Cfg::OUT_ROW, A, R>(&tmC, stage, p.split_k, slab_f4, colbuf + cofs, obuf,    \
                                                          hcols, cbase, row0, b, lane, res);                      \
    break;
            TMB_REDS(0, 0) TMB_REDS(0, 1) TMB_REDS(1, 0) TMB_REDS(1, 1) TMB_REDS(1, 2) TMB_REDS(2, 0) TMB_REDS(2, 1)
#undef TMB_REDS
            default: __trap();
          }
          if (lead) detail::trace(p, i, 11, t0);
          continue;
        }
        switch (p.canon_act * 3 + (p.canon_res_op < 0 ? 0 : p.canon_res_pre ? 2 : 1)) {
#define TMB_RED(A, R)                                                                                              \
  case A * 3 + R:                                                                                                  \
    detail::drain_reduce<BN, CG, Cfg::OUT_ROW, A, R>(&tmC, ws, p.split_k, rloc, cofs, colbuf + cofs, obuf, hcols,  \
                                                     cbase, row0, b, lane, res, tk, t0);                           \
    break;
          TMB_RED(0, 0) TMB_RED(0, 1) TMB_RED(1, 0) TMB_RED(1, 1) TMB_RED(1, 2) TMB_RED(2, 0) TMB_RED(2, 1)
#undef TMB_RED
          default: __trap();
        }
        if (gt == 0 && !p.sk_spin) p.counters[tile_id * 2 + grp] = 0;  // self-resetting for the next launch
        if (lead) detail::trace(p, i, 11, t0);
        continue;
      }
      if (p.split_k > 1) {
        // ---- split-K: park the raw partial tile, last unit reduces + runs the epilogue
        const int64_t tile_id = ((static_cast<int64_t>(b) * p.tiles_m + tm_) * p.tiles_n + tn) * CG + rank;
        const float* ws = p.workspace + tile_id * p.split_k * static_cast<int64_t>(kBM * BN);
        const int rloc = lg * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < kChunks; ++c) {
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
        release_acc(abuf);  // TMEM is free again: the MMA can start the next unit
        __threadfence();
        ptx::named_bar_sync(3 + grp, 128);
        if (gt == 0) split_flag[grp] = (atomicAdd(&p.counters[tile_id * 2], 1) == p.split_k - 1) ? 1u : 0u;
        ptx::named_bar_sync(3 + grp, 128);
        if (*reinterpret_cast<volatile uint32_t*>(&split_flag[grp]) == 0u) continue;
        __threadfence();
#pragma unroll 1
        for (int c = 0; c * 16 < ncols; ++c) {
          if (c % (gcols / 16) == 0) group_begin();
          if (p.has_mat) prefetch(c, mat);
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
          for (int sp = 0; sp < p.split_k; ++sp) {  // fixed order: deterministic
            const float4* src = reinterpret_cast<const float4*>(ws + sp * static_cast<int64_t>(kBM * BN) +
                                                                (static_cast<int64_t>(c) * kBM + rloc) * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = __ldcg(src + q);
              v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
            }
          }
          detail::epilogue16<BN, GENERIC>(p, v, colbuf, c * 16, rowv, mat);
          put16(v, c * 16, obase, n0, row_ok);
          if ((c + 1) % (gcols / 16) == 0 || (c + 1) * 16 >= ncols)
            group_end(n0 + (c * 16 / gcols) * gcols, row0);
        }
        if (gt == 0) p.counters[tile_id * 2] = 0;  // self-resetting for the next launch
        continue;
      }
      // 32 columns per TMEM load; the accumulator is released right after the
      // last load, before the math of the last columns
      if (lean) {
        // lean drain (host guarantees via epi_fast: canonical epilogue, bf16 TMA-stored
        // output, residual absent or bf16 contiguous 16-byte aligned with N % 32 == 0)
        // this group's column half of the tile
        const int kHalf = colsplit ? BN / 2 : BN;
        const int cofs = colsplit ? grp * kHalf : 0;
        const int hcols = max(0, min(kHalf, ncols - cofs));
        const uint4* res = nullptr;
        if (p.canon_res_op >= 0)
          res = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ops[p.canon_res_op].ptr) +
                                               detail::addr_rowpart(p.ops[p.canon_res_op].a, rr, b) + n0 + cofs);
        const int32_t cb = static_cast<int32_t>(n0) + cofs;
        // direct stores (p.out_direct): this lane's row of the output; dcols = valid
        // columns of the half (multiple of 8 by the host's check), -1 = row outside M
        __nv_bfloat16* drow = nullptr;
        int dcols = 0;
        if (p.out_direct) {
          if (row_ok) {
            drow = static_cast<__nv_bfloat16*>(p.out) + detail::addr_rowpart(p.out_a, rr, b) + n0 + cofs;
            dcols = hcols;
          } else {
            dcols = -1;
          }
        }
        long long* fine = nullptr;
#ifdef TMB_FINE_TRACE
        if (p.trace != nullptr && nvalid <= 4)
          fine = p.trace + (static_cast<int64_t>(blockIdx.x) * kTraceTiles + 48) * kTraceEvents + (nvalid - 1) * 64;
#endif
        if constexpr (Cfg::OUT_ROW == 128) {
          if (p.out_dtype == DT_F32) {  // fp32 rows: identity or ReLU, no residual (host-checked)
            if (p.canon_act == 1)
              detail::drain_fast<BN, CG, Cfg::OUT_ROW, 1, 0, true>(&tmC, taddr + cofs, colbuf + cofs, obuf, hcols, cb,
                                                                   row0, b, lane, nullptr, &tempty[abuf]);
            else
              detail::drain_fast<BN, CG, Cfg::OUT_ROW, 0, 0, true>(&tmC, taddr + cofs, colbuf + cofs, obuf, hcols, cb,
                                                                   row0, b, lane, nullptr, &tempty[abuf]);
            if (lead) detail::trace(p, i, TR_EPI_DONE, t0);
            continue;
          }
        }
        switch (p.canon_act * 3 + (res == nullptr ? 0 : p.canon_res_pre ? 2 : 1)) {
#define TMB_DRAIN(A, R)                                                                                          \
  case A * 3 + R:                                                                                                \
    detail::drain_fast<BN, CG, Cfg::OUT_ROW, A, R>(&tmC, taddr + cofs, colbuf + cofs, obuf, hcols, cb, row0, b,  \
                                                   lane, res, &tempty[abuf], fine, drow, dcols);                 \
    break;
          TMB_DRAIN(0, 0) TMB_DRAIN(0, 1) TMB_DRAIN(1, 0) TMB_DRAIN(1, 1) TMB_DRAIN(1, 2) TMB_DRAIN(2, 0) TMB_DRAIN(2, 1)
#undef TMB_DRAIN
          default: __trap();
        }
        if (lead) detail::trace(p, i, TR_EPI_DONE, t0);
        continue;
      }
#pragma unroll 1
      for (int c2 = 0; c2 * 32 < ncols; ++c2) {
        uint32_t r[32];
        ptx::tmem_ld32(taddr + c2 * 32, r);
        ptx::tmem_wait_ld();
        if ((c2 + 1) * 32 >= ncols) release_acc(abuf);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c = c2 * 32 + hh * 16;
          if (c >= ncols) break;
          if (c % gcols == 0) group_begin();
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[hh * 16 + j]);
          float nxt[kMaxMatOps][16];
          if (p.has_mat && c + 16 < ncols) prefetch(c / 16 + 1, nxt);
          detail::epilogue16<BN, GENERIC>(p, v, colbuf, c, rowv, mat);
          put16(v, c, obase, n0, row_ok);
          if (p.has_mat) {
#pragma unroll
            for (int o = 0; o < kMaxMatOps; ++o)
#pragma unroll
              for (int j = 0; j < 16; ++j) mat[o][j] = nxt[o][j];
          }
          if ((c + 16) % gcols == 0 || c + 16 >= ncols) group_end(n0 + (c / gcols) * gcols, row0);
        }
      }
      if (lead) detail::trace(p, i, TR_EPI_DONE, t0);
    }
    if (p.out_tma && lane == 0) ptx::bulk_wait<0>();  // all output tiles written before exit
  } else {
    // ===================== MMA issuer =====================
    // The whole warp walks the ring (warp-uniform control flow); one elected
    // lane issues each k-block's tcgen05.mma group and its commit.  Descriptors
    // are built once: per stage / per K16 step they only move the start address
    // field (addr >> 4 in bits [0,14)), so the issue loop is adds on uniform
    // registers.
    if (rank == 0) {
      const bool b_mn = p.b_loader == LD_TMA_MN;
      const bool a_noswz = p.a_loader == LD_IM2COL_TMA8;
      const bool a_g8 = p.a_loader == LD_IM2COL_G8;
      // operand format: tf32 (kind::tf32) / fp16 (0) or bf16 (1) for kind::f16
      const uint32_t idesc = ptx::make_idesc(kTileM, BN, TF32 ? 2u : (p.ab_f16 ? 0u : 1u), false, b_mn);
      const uint32_t mn_lbo = p.mn_lbo_sbo_swap ? 1024u : static_cast<uint32_t>(MN_BLOCK_BYTES);
      const uint32_t mn_sbo = p.mn_lbo_sbo_swap ? static_cast<uint32_t>(MN_BLOCK_BYTES) : 1024u;
      const uint32_t a0 = ptx::smem_u32(smA), b0 = ptx::smem_u32(smB);
      // 2 taps (2 x 16 B chunks of 2 KB boxes) per K16 for the C<=8 im2col layout
      // G8: taps adjacent (LBO 128 B along K, SBO 1024 B per 8 rows), 2 taps per K16
      const uint64_t adesc0 = a_noswz ? ptx::smem_desc_noswz(a0, 2048, 128)
                                      : a_g8 ? ptx::smem_desc_noswz(a0, 128, 1024) : ptx::smem_desc_sw128(a0, 16, 1024);
      const uint64_t bdesc0 = !b_mn ? ptx::smem_desc_sw128(b0, 16, 1024)
                              : TF32 ? ptx::smem_desc_sw128_base32b(b0, static_cast<uint32_t>(MN_BLOCK_BYTES), 512u)
                                     : ptx::smem_desc_sw128(b0, mn_lbo, mn_sbo);
      const uint32_t a_kstep = a_noswz ? (2u * 2048u) >> 4
                                       : a_g8 ? (2u * 128u) >> 4 : static_cast<uint32_t>(Cfg::KSTEP * Cfg::kElem) >> 4;
      const uint32_t b_kstep = b_mn ? static_cast<uint32_t>(Cfg::KSTEP * kRowBytes) >> 4
                                    : static_cast<uint32_t>(Cfg::KSTEP * Cfg::kElem) >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int b, ks, tm_, tn;
      bool valid;
      for (uint32_t i = 0; detail::next_tile<CG>(p, tile_list, i, b, ks, tm_, tn, valid); ++i) {
        if (!valid) continue;
        if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&tempty[acc], acc_phase ^ 1u);
        else ptx::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb0 = ks * p.kb_per_split, kb = kb0, kb_end = min(p.num_kb, kb0 + p.kb_per_split); kb < kb_end; ++kb) {
          if constexpr (CG == 2) ptx::mbar_wait_acq_cluster(&full[stage], phase);
          else ptx::mbar_wait(&full[stage], phase);
          if (GENERIC && !all_tma && p.dbg != 5) ptx::fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05.mma
          ptx::tc_fence_after();
          if (kb == kb0 && lane == 0) detail::trace(p, i, TR_MMA_FIRST, t0);
          const uint64_t ad = adesc0 + static_cast<uint64_t>((stage * Cfg::A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + static_cast<uint64_t>((stage * Cfg::B_BYTES) >> 4);
          // K16 steps wholly past K (the last k-block of a ragged K, e.g. conv1's
          // 49 taps) multiply zero-filled operands: skip them
          const int ksteps = min(Cfg::NSTEP, (p.K - kb * BK + Cfg::KSTEP - 1) / Cfg::KSTEP);
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < Cfg::NSTEP; ++kk) {
              // dbg 6: loads only (no MMA) -> load floor; dbg 7: neither -> ring handshake floor
              if ((kk > 0 && kk >= ksteps) || p.dbg == 6 || p.dbg == 7) break;
              const uint64_t adesc = ad + static_cast<uint64_t>(kk * a_kstep);
              const uint64_t bdesc = bd + static_cast<uint64_t>(kk * b_kstep);
              const uint32_t accum = (kb != kb0 || kk != 0);
              if constexpr (CG == 2) {
                if (TF32) ptx::mma_tf32_2sm(d_tmem, adesc, bdesc, idesc, accum);
                else ptx::mma_f16_2sm(d_tmem, adesc, bdesc, idesc, accum);
              } else {
                if (TF32) ptx::mma_tf32(d_tmem, adesc, bdesc, idesc, accum);
                else ptx::mma_f16(d_tmem, adesc, bdesc, idesc, accum);
              }
            }
            // frees this ring slot (in both CTAs of the pair)
            if constexpr (CG == 2) ptx::mma_commit_2sm(&empty[stage], 0x3);
            else ptx::mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == ring) { stage = 0; phase ^= 1u; }
        }
        if (ptx::elect_one()) {
          if constexpr (CG == 2) ptx::mma_commit_2sm(&tfull[acc], 0x3);
          else ptx::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (lane == 0) detail::trace(p, i, TR_MMA_LAST, t0);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  }

  if (p.trace != nullptr && lane == 0)  // ns: warp reached the final barrier (tile 2 + warp, slot 15)
    p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + 2 + warp) * kTraceEvents + 15] =
        static_cast<long long>(ptx::globaltimer());
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer done with its TMEM before the pair frees it
  else __syncthreads();
  if (p.trace != nullptr && threadIdx.x == 0)  // ns: all roles done (tile 0's slot 15)
    p.trace[static_cast<int64_t>(blockIdx.x) * kTraceTiles * kTraceEvents + 15] =
        static_cast<long long>(ptx::globaltimer());
  if (warp == R::kMmaWarp) {
    if (p.trace != nullptr && lane == 0)  // ns: MMA warp past the barrier (tile 1's slot 14)
      p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + 1) * kTraceEvents + 14] =
          static_cast<long long>(ptx::globaltimer());
    ptx::tc_fence_after();
    if (!(skip & 4)) {
      if constexpr (CG == 2) ptx::tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
      else ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
    if (p.trace != nullptr && lane == 0)  // ns: TMEM released (tile 1's slot 15)
      p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + 1) * kTraceEvents + 15] =
          static_cast<long long>(ptx::globaltimer());
  }
}

}  // namespace tmb
