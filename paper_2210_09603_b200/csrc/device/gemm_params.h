// Parameter block of the fused task-mapped GEMM kernel (host + device).
//
// The kernel realises the spec's matmul_template with its
// two fusion splice points: operand *loaders* are the prologue
// splice (a direct/strided load, a cast, or the im2col gather of
// conv2d_im2col_dag, proj/src/compute_ir.cpp:532-557), and the *epilogue op
// list* plus the output *address map* are the epilogue splice (bijective
// chains, fusion spec SPEC.md:379-387).  Everything here is plain data so it
// can be built by the C++ planner and passed by value as a __grid_constant__.
#pragma once
#include <cstdint>

#include "taskmap.cuh"

namespace tmb {

enum DType : int32_t { DT_F32 = 0, DT_BF16 = 1, DT_F16 = 2 };

// Element address of GEMM coordinate (row, col, batch):
//   (row / P) * s_hi + (row % P) * s_lo + col * s_col + batch * s_batch + offset
// This is the canonical form every affine-bijective epilogue remap in the
// reference's builders reduces to (row-major, transpose, NCHW re-index of the
// im2col GEMM, reshape splits), cf. compute_ir.cpp:582-592.
struct Addr {
  int64_t P;  // >= 1
  int64_t s_hi, s_lo, s_col, s_batch, offset;
};

enum EpiKind : int32_t {
  EPI_ADD_C = 1, EPI_SUB_C, EPI_RSUB_C, EPI_MUL_C, EPI_DIV_C, EPI_RDIV_C, EPI_MAX_C, EPI_MIN_C,
  EPI_ADD_T = 16, EPI_SUB_T, EPI_RSUB_T, EPI_MUL_T, EPI_DIV_T, EPI_RDIV_T, EPI_MAX_T, EPI_MIN_T,
  EPI_RELU = 32, EPI_GELU_TANH, EPI_EXP, EPI_SQRT, EPI_NEG, EPI_ROUND_BF16
};

// How a side operand varies over the output tile (decides where the
// epilogue keeps it): per-column vectors (bias, BN scale/shift) are staged in
// shared memory once per tile, per-row scalars live in a register, general
// matrices (residuals) are prefetched one 16-column chunk ahead.
enum SideKind : int32_t { SIDE_NONE = 0, SIDE_COL = 1, SIDE_ROW = 2, SIDE_MAT = 3 };

// One epilogue op; *_T kinds read a side tensor at `a` (dtype `dtype`).
struct EpiOp {
  int32_t kind;
  int32_t dtype;
  float c;
  int32_t side;  // SideKind
  int32_t slot;  // SIDE_MAT: prefetch slot (< kMaxMatOps)
  int32_t pad_;
  const void* ptr;
  Addr a;
};

constexpr int kMaxSmem = 232448;  // 227 KB opt-in dynamic shared memory per CTA on sm_100
constexpr int kMaxEpiOps = 8;
constexpr int kMaxMatOps = 2;
constexpr int kTraceTiles = 64;
constexpr int kTraceEvents = 16;  // 0-7 role events (TraceEv); tile 0: 14/15 = setup done / exit (ns)

// Output staging of the epilogue: each epilogue warp owns one smem buffer of
// 32 rows x out_stage_row_bytes (a 64- or 128-byte swizzled row segment per
// lane), written to global memory by one TMA store per column group.  64-byte
// rows for BN = 256 single-CTA tiles, whose pipeline needs the shared memory.
// The two epilogue warp groups split every tile's columns in halves (compact
// kernel), so BN/2 must be a whole number of store groups: 64-byte rows
// (32 bf16 columns) for BN = 64 and 192.
constexpr int out_stage_row_bytes(int bn, int cg) {
  return ((bn == 256 && cg == 1) || bn == 64 || bn == 96 || bn == 192) ? 64 : 128;
}
// Row-band conv kernel (conv_rowband.cuh) output staging: 128-byte (64-column)
// swizzled row segments, one TMA store per warp per 64 columns (its epilogue
// groups alternate whole tiles instead of splitting columns).
constexpr int kRbOutRow = 128;
// trace events per tile
enum TraceEv : int32_t {
  TR_PROD_FIRST = 0,  // producer: first k-block slot acquired
  TR_PROD_LAST,       // producer: last TMA of the tile issued
  TR_MMA_FIRST,       // MMA: first k-block data ready
  TR_MMA_LAST,        // MMA: last MMA issued / commit
  TR_EPI_READY,       // epilogue: column operands staged
  TR_EPI_ACC,         // epilogue: accumulator available
  TR_EPI_DONE,        // epilogue: tile stored
  TR_CTA_START        // (tile 0 only) CTA start, globaltimer ns
};

enum LoaderKind : int32_t {
  LD_TMA_K = 0,         // TMA tile load, K contiguous (K-major)
  LD_TMA_MN = 1,        // TMA tile load, M/N contiguous (MN-major), B only, 16-bit
  LD_GATHER = 2,        // predicated LSU gather of a strided operand (+ cast)
  LD_IM2COL_GATHER = 3, // predicated im2col gather from any-strided X (A only)
  LD_IM2COL_TMA = 4,    // TMA im2col mode on channels-last X (A only)
  LD_FILTER_GATHER = 5, // conv filter W[F,C,Kh,Kw] with any strides (B only)
  LD_IM2COL_TMA8 = 6,   // small-C conv (C <= 8, 16-byte padded channels-last X): one
                        // TMA im2col box {8 ch x 128 px} per tap, 8 taps per k-block,
                        // no-swizzle K-major smem layout; K order (tap, c < 8)
  LD_IM2COL_G8 = 7,     // same layout and K order as LD_IM2COL_TMA8, gathered by the
                        // 128 loader threads: one 16-byte load per (pixel, tap), the
                        // channels >= C masked to zero (no per-box TMA cost: 49 taps)
  LD_ROWBAND = 8,       // no im2col tile at all: staged input rows read by the MMA through
                        // overlapping no-swizzle descriptors (tm_rowband_kernel)
  LD_HALO = 9           // same idea for C % 64 == 0: a staged channel-group-major input band
                        // read by every tap at its own offset (tm_halo_kernel)
};

// An elementwise prologue op applied to every operand element the gather
// loader reads (fuse_prologue: Fig. 11's A[99-i] -> C[99-i]*2.0,
// or a ReLU producer): the same constant-operand kinds as the epilogue
// (EPI_*_C, EPI_RELU, EPI_NEG, EPI_EXP, EPI_SQRT, EPI_GELU_TANH).
struct PreOp {
  int32_t kind;
  float c;
};
constexpr int kMaxPreOps = 4;

// A strided operand: element (row, k, batch) at
//   (row / P) * s_hi + (row % P) * s_lo + k * s_k + batch * s_batch + offset,
// optionally transformed by an arithmetic prologue (n_pre ops, in order).
struct Strided {
  const void* ptr;
  int32_t dtype;
  int32_t n_pre;
  int64_t P, s_hi, s_lo, s_k, s_batch, offset;
  PreOp pre[kMaxPreOps];
};

// Convolution geometry (reference conv2d_im2col_dag arguments) plus element
// strides of X[n,c,h,w] and W[f,c,kh,kw].  korder 0 = reference K order
// r = c*Kh*Kw + fh*Kw + fw (compute_ir.cpp:540-542); korder 1 = (fh, fw, c),
// the order TMA im2col produces (requires channels-last X and W).
struct ConvGeom {
  int32_t n, c, h, w, f, kh, kw, stride, pad, ho, wo, korder;
  int32_t cpad;  // channels per tap in K order 1 (= c, or 8 for LD_IM2COL_TMA8)
  int32_t pad2_;
  const void* x;
  const void* wt;
  int32_t x_dtype, w_dtype;
  int64_t sx[4];
  int64_t sw[4];
};

struct GemmParams {
  int32_t M, N, K, batch;
  int32_t num_kb;  // ceil(K / BK)
  int32_t tiles_m, tiles_n;
  int32_t a_loader, b_loader;
  int32_t mn_lbo_sbo_swap;  // debug knob for the MN-major descriptor
  Strided a, b;
  ConvGeom conv;
  tm::DevMapping tile_map;  // CTA -> (batch, tile_m, tile_n) task mapping
  // split-K (SPEC.md:277 split_k): work unit = (batch, k-split, tile_m, tile_n);
  // tile_map coordinate 0 enumerates batch * split_k + ks.  Each unit covers
  // k-blocks [ks*kb_per_split, min(num_kb, (ks+1)*kb_per_split)); partial
  // tiles go to `workspace` (fp32) and the last unit to arrive on the tile's
  // counter sums them in split order (deterministic) and runs the epilogue.
  int32_t split_k;
  int32_t kb_per_split;
  float* workspace;
  int32_t* counters;
  // one-round grids (every work unit resident): the tile's split_k units wait for
  // each other's partials and each reduces its own 32-row blocks (lg % split_k ==
  // ks) instead of the last arriver reducing the whole tile; counters grow
  // monotonically (arrival a waits for (a / split_k + 1) * split_k)
  int32_t sk_spin;
  int32_t sk_pad_;
  int32_t fast_math;  // approximate transcendentals (bf16 outputs)
  int32_t ab_f16;     // 16-bit MMA operands are fp16 (kind::f16 a/b format 0), else bf16 (format 1)
  int32_t out_tma;    // row-major output: stage each 32x16 chunk in smem, TMA-store it
  // Canonical epilogue v = act(acc * S[col] + T[col]) (+ R[row, col]), which every
  // chain of the BASELINE configs compiles to (bias, scale, BN-fold, ReLU/GELU,
  // residual): S/T are staged per tile as column vectors; ops that do not fit run
  // through the generic op interpreter instead.
  int32_t canon;
  int32_t canon_act;       // 0 none, 1 relu, 2 gelu_tanh
  int32_t canon_s_op;      // op index providing S (-1: constant canon_s)
  int32_t canon_t_op;      // op index providing T (-1: constant canon_t)
  int32_t canon_res_slot;  // SIDE_MAT prefetch slot added after the activation (-1: none)
  int32_t canon_res_op;    // op index of that residual (-1: none)
  int32_t canon_res_pre;   // 1: the residual is added before the activation (act(acc*S+T+R))
  float canon_s, canon_t;
  // optional per-tile role timeline (clock64 relative to CTA start), layout
  // [cta][kTraceTiles][kTraceEvents]; null = tracing off
  long long* trace;
  int32_t dbg;  // diagnostics (TMB_DBG): 1 = skip all roles after setup
  int32_t dbg_skip;
  // per-worker task list precomputed at bind time ([workers][tile_map.tasks] of
  // {tm | tn << 16, (b * split_k + ks) << 1 | valid}); null = decode on device
  const uint32_t* tile_tab;  // diagnostics with dbg 1 (TMB_SKIP bits): 1 tile list, 2 barrier init, 4 TMEM
  // canonical epilogue with a bf16 TMA-stored output (and bf16 contiguous
  // residual): drained by the lean drain_fast path in either kernel
  int32_t epi_fast;
  // weight-stationary B: one column tile, one batch, no split-K and a ring
  // depth that is a multiple of num_kb, so k-block kb always lands in the same
  // ring slot: B is loaded in the first ring pass only and stays resident
  int32_t b_resident;
  int32_t ring;  // ring slots in use (0 = all STAGES)
  // MN-major B as one 4-D box {64 n, BK k, BN/64 n-blocks} per slot instead of
  // BN/64 boxes (TMA issue is ~600 clk per box per warp): needs N % 64 == 0
  int32_t b_mn4d;
  // lean drain writes bf16 rows straight from registers (16-byte stores) instead
  // of smem staging + TMA store: row-major output, 16-byte aligned rows, N % 8 == 0
  int32_t out_direct;
  // Row-band implicit GEMM (tm_rowband_kernel, conv_rowband.cuh): small-C convs
  // whose input pixels are padded to cpad channels with stride * cpad == 8, so
  // consecutive output pixels' windows start 16 bytes apart in a staged input row
  // and every tcgen05.mma reads its A operand straight out of the staged rows.
  int32_t rb_T;        // output rows per band
  int32_t rb_rows;     // staged input rows per TMA box (4 boxes per band >= stride * (T - 1) + kh rows)
  int32_t rb_rowb;     // bytes per staged input row (whole 16- or 128-byte chunks)
  int32_t rb_off0;     // byte offset of output pixel 0's window inside a staged row
  int32_t rb_T0;       // output rows of a CTA's first band (short: the MMA starts sooner)
  int32_t rb_rows0;    // staged input rows per box of the first band
  int32_t rb_steps;    // K16 MMA steps per filter row (= 8 * cpad / 16)
  int32_t rb_g0;       // chunk coordinate of a staged row's first chunk (<= 0: left padding)
  int32_t rb_total;    // output rows N * Ho
  int32_t rb_cpad;     // channels per staged pixel
  int32_t rb_fix;      // zero channels [C, cpad) of every staged pixel (padding lanes)
  int32_t rb_bbytes;   // bytes of the packed filter image
  int32_t rb_pad3_;
  const void* rb_bimg; // packed filter smem image [kh][steps][F/8][2][8 rows][16 B]
  // Halo implicit GEMM (tm_halo_kernel, conv_halo.cuh): stride-1 convs on
  // channels-last X with C % 64 == 0.  A tile is R output rows of P = Wo + 2 pad
  // "virtual" pixels (the halo columns compute garbage that is never stored) on
  // the TMEM lanes; its staged input band [C/8][R + kh - 1 rows][P][8 ch] is read
  // by every tap's MMA at offset (fh * P + fw) * 16 bytes.
  int32_t hb_R;        // output rows per tile
  int32_t hb_P;        // staged pixels per row (Wo + 2 * pad)
  int32_t hb_rows;     // staged rows per band (R + kh - 1)
  int32_t hb_G;        // bytes between channel groups in a band (rows * P * 16)
  int32_t hb_band;     // bytes per band buffer (C/8 groups + read slack, 1 KB aligned)
  int32_t hb_kb;       // k-blocks per tile: kh * kw * C / 64
  int32_t hb_tpi;      // tiles per image: ceil(Ho / R)
  int32_t hb_ftiles;   // F / BN column tiles
  int32_t hb_total;    // N * tpi * ftiles tiles
  int32_t hb_stages;   // filter ring depth
  int32_t hb_mc;       // CTAs per cluster sharing (TMA-multicasting) each filter stage: 1 or 2
  int32_t hb_split;    // hb_mc == 2: each CTA loads half a stage -- 1: half the taps, 0: half the rows
  int32_t hb_nbands;   // band buffers: 2, or 1 when no CTA has a second tile
  int32_t n_ops;
  int32_t has_mat;  // any SIDE_MAT op
  int32_t out_dtype;
  EpiOp ops[kMaxEpiOps];
  void* out;
  Addr out_a;
};

}  // namespace tmb
