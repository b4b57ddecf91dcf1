// Row-band implicit-GEMM convolution for small-C inputs (the ResNet-50 stem
// conv1: C = 3, 7x7, stride 2), sm_100a.
//
// The reference computes the conv as Y = Wf * Col with the im2col node
// Col[r, s] = X[n, c, oh*stride - pad + fh, ow*stride - pad + fw] (zero outside
// the image; proj/src/compute_ir.cpp:532-557).  The K3 kernel materialises Col
// tiles in shared memory (TMA im2col boxes or LSU gathers); for C <= 8 that is
// one 8- or 16-byte piece per (pixel, tap), which TMA issues slowly and LSU
// gathers latency-bound (round-1/2 traces: conv1 at ~6% of roofline).
//
// Here Col is never built.  Input pixels are stored padded to cpad channels
// (8-byte pixels: cpad = 4, or 16-byte: cpad = 8) and the K order is
// (fh, fw' in [0, 8), c in [0, cpad)) with fw' = fw + shift.  When
// stride * cpad == 8, the 8-tap window of output pixel ow starts exactly 16 bytes
// after the window of ow - 1 inside a staged input row, so for filter row fh and
// K16 step t the UMMA A operand (128 output pixels x 16 K) is the staged row
// ih = oh*stride - pad + fh read as a no-swizzle K-major matrix with
//   start = row + 32 t,  SBO = 128 B (8 pixels),  LBO = 16 B (next 8 K),
// i.e. overlapping core matrices addressed by the descriptor alone.  One CTA
// tile = one output row (Wo <= 128 pixels on the TMEM lanes; lanes past Wo are
// computed and clipped by the TMA store).  Padding is free: rows outside the
// image and pixels left/right of it are TMA out-of-bounds zero fill, and the
// filter image (packed once at bind) is zero at padded taps / channels.
//
// Schedule (a task mapping over output rows, spatial(G) * repeat(R/G)): CTA w
// owns the contiguous output rows [w R / G, (w+1) R / G) and walks them in bands
// of <= T rows of one image; a band stages stride*(T-1)+kh input rows with one
// 4-D TMA box (double-buffered), so consecutive rows' shared input rows are read
// once.  Warp roles: 0 TMA producer (+ pad-lane fix-up), 1 MMA issuer / TMEM
// owner, 2-9 epilogue (two groups alternating tiles, canonical BN-fold + act,
// the lean drain of gemm_sm100.cuh).
#pragma once
#include "gemm_sm100.cuh"

namespace tmb {

constexpr int kRbThreads = 416;  // 13 warps
constexpr int kRbEpiWarps = 8;
// A band is staged as kRbLoadWarps boxes of rb_rows input rows each, issued by
// different warps (warp 0 and 10-12): TMA copies issued by one warp are serviced
// one after another, so one box per band left the SM latency-bound on HBM.
constexpr int kRbLoadWarps = 4;

__host__ __device__ constexpr int rb_nacc(int bn) { return bn <= 128 ? 4 : 2; }


// smem carve-up shared by host (sizing) and device
struct RbLayout {
  int band, bimg, outbuf, colbuf, bars, total;
  __host__ __device__ static int align(int x) { return (x + 1023) & ~1023; }
  __host__ __device__ RbLayout(int rows, int rowb, int bbytes, int bn) {
    band = align(rows * rowb);
    bimg = 2 * band;
    outbuf = bimg + align(bbytes);
    colbuf = outbuf + kRbEpiWarps * 32 * kRbOutRow;
    bars = colbuf + 2 * bn * 4;
    total = bars + 256;
  }
};

namespace detail {

__device__ __forceinline__ void rb_range(const GemmParams& p, int& r0, int& r1) {
  const int64_t R = p.rb_total, G = gridDim.x;
  r0 = static_cast<int>(R * blockIdx.x / G);
  r1 = static_cast<int>(R * (blockIdx.x + 1) / G);
}

// band starting at output row r (global row index n*Ho + oh): rows [r, end);
// a CTA's first band (r == r0) is short so its MMAs start early
__device__ __forceinline__ int rb_band_end(const GemmParams& p, int r, int r0, int r1) {
  const int img_end = (r / p.conv.ho + 1) * p.conv.ho;
  return min(min(r + (r == r0 ? p.rb_T0 : p.rb_T), r1), img_end);
}

// Channels [C, cpad) of every staged pixel are padding: zero them (the filter
// is zero there too, but the caller's pad lanes may hold NaN/Inf).  A band is a
// flat array of 16-byte granules (1 or 2 pixels each): one masked 16-byte
// read-modify-write per granule, spread over `nthreads` threads.
__device__ __forceinline__ void rb_zero_pad_lanes(const GemmParams& p, uint8_t* band, int rows, int tid,
                                                  int nthreads) {
  uint32_t m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {  // 16-bit lanes 2j, 2j+1 hold channels (2j) % cpad, (2j+1) % cpad
    const int c0 = (2 * j) % p.rb_cpad, c1 = (2 * j + 1) % p.rb_cpad;
    m[j] = (c0 < p.conv.c ? 0x0000FFFFu : 0u) | (c1 < p.conv.c ? 0xFFFF0000u : 0u);
  }
  uint4* gr = reinterpret_cast<uint4*>(band);
  const int total = rows * (p.rb_rowb >> 4);
#pragma unroll 4
  for (int i = tid; i < total; i += nthreads) {
    uint4 v = gr[i];
    v.x &= m[0]; v.y &= m[1]; v.z &= m[2]; v.w &= m[3];
    gr[i] = v;
  }
}

// optional timeline (TMB_TRACE): clock64 since setup, [cta][tile][event]
// events: 0 MMA start (accumulator free), 1 MMA issued, 2 epilogue has the
// accumulator, 3 epilogue stored, 4 band ready at the MMA (band's first tile),
// 5 band copy issued (band's first tile), 6 band landed (band's first tile)
__device__ __forceinline__ void rb_trace(const GemmParams& p, int tile, int ev, long long t0) {
  if (p.trace != nullptr && tile < kTraceTiles)
    p.trace[(static_cast<int64_t>(blockIdx.x) * kTraceTiles + tile) * kTraceEvents + ev] = clock64() - t0;
}

}  // namespace detail

// KH / STEPS > 0: compile-time filter rows and K16 steps per row (fully unrolled
// MMA issue); 0: runtime loops
template <int BN, int KH, int STEPS>
__global__ void __launch_bounds__(kRbThreads, 1)
    tm_rowband_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmX,
                      const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmC) {
  constexpr int NACC = rb_nacc(BN);
  constexpr uint32_t TMEM_COLS = NACC * BN <= 256 ? 256 : 512;
  constexpr int OUT_ROW = kRbOutRow;
  extern __shared__ __align__(1024) uint8_t smem[];
  const RbLayout L(kRbLoadWarps * p.rb_rows, p.rb_rowb, p.rb_bbytes, BN);
  uint8_t* band[2] = {smem, smem + L.band};
  uint8_t* bimg = smem + L.bimg;
  uint8_t* outbuf = smem + L.outbuf;
  float* colbuf = reinterpret_cast<float*>(smem + L.colbuf);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* bfull = bars;        // [2] band staged (TMA bytes)
  uint64_t* bready = bars + 2;   // [2] band fixed up (pad lanes zeroed), when rb_fix
  uint64_t* bempty = bars + 4;   // [2] band's MMAs done
  uint64_t* bbar = bars + 6;     // filter image landed
  uint64_t* tfull = bars + 7;    // [NACC]
  uint64_t* tempty = bars + 7 + NACC;  // [NACC]
  uint64_t* bready0 = bars + 7 + 2 * NACC;  // band 0 fixed up (by the 8 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmX);
    ptx::tma_prefetch_desc(&tmX0);
    ptx::tma_prefetch_desc(&tmC);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bready[i], kRbLoadWarps);
      ptx::mbar_init(&bempty[i], 1);
    }
    ptx::mbar_init(bbar, 1);
    ptx::mbar_init(bready0, kRbEpiWarps);
    for (int a = 0; a < NACC; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);  // the 4 warps of the draining group
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();

  int r0, r1;
  detail::rb_range(p, r0, r1);
  const long long t0 = clock64();
  const ConvGeom& g = p.conv;

  if (warp == 0 || warp >= 10) {
    // =============== producers: filter image + input bands (box q each) ===============
    const int q = warp == 0 ? 0 : warp - 9;
    if (q == 0 && lane == 0) {
      ptx::mbar_arrive_expect_tx(bbar, static_cast<uint32_t>(p.rb_bbytes));
      ptx::bulk_load(bimg, p.rb_bimg, static_cast<uint32_t>(p.rb_bbytes), bbar);
    }
    auto issue = [&](int bi, int r) {
      const int buf = bi & 1;
      const int rbox = bi == 0 ? p.rb_rows0 : p.rb_rows;
      if (bi >= 2) ptx::mbar_wait(&bempty[buf], ((bi >> 1) - 1) & 1);
      if (lane == 0) {
        const int n = r / g.ho, oh = r - n * g.ho;
        if (q == 0) {
          detail::rb_trace(p, r - r0, 5, t0);
          ptx::mbar_arrive_expect_tx(&bfull[buf], static_cast<uint32_t>(kRbLoadWarps * rbox * p.rb_rowb));
        }
        ptx::tma_load_4d(band[buf] + q * rbox * p.rb_rowb, bi == 0 ? &tmX0 : &tmX, &bfull[buf], 0, p.rb_g0,
                         oh * g.stride - g.pad + q * rbox, n);
      }
      __syncwarp();
    };
    if (r0 < r1) issue(0, r0);
    int bi = 0;
    for (int r = r0; r < r1; ++bi) {
      const int e = detail::rb_band_end(p, r, r0, r1);
      if (e < r1) issue(bi + 1, e);  // next band's copy overlaps this band's fix-up / MMAs
      if (p.rb_fix && bi > 0) {
        // channels [C, cpad) of every staged pixel are padding: zero them (the
        // filter is zero there too, but the caller's pad lanes may hold NaN/Inf)
        const int buf = bi & 1;
        ptx::mbar_wait(&bfull[buf], (bi >> 1) & 1);
        detail::rb_zero_pad_lanes(p, band[buf] + q * p.rb_rows * p.rb_rowb, p.rb_rows, lane, 32);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bready[buf]);
      }
      r = e;
    }
    // producer tail: every band's MMAs have completed before the CTA can exit
    if (bi >= 1) ptx::mbar_wait(&bempty[(bi - 1) & 1], ((bi - 1) >> 1) & 1);
    if (bi >= 2) ptx::mbar_wait(&bempty[(bi - 2) & 1], ((bi - 2) >> 1) & 1);
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    const uint32_t idesc = ptx::make_idesc(128, BN, p.ab_f16 ? 0u : 1u, false, false);
    const uint64_t a0 = ptx::smem_desc_noswz(ptx::smem_u32(band[0]) + p.rb_off0, 16, 128);
    const uint64_t b0 = ptx::smem_desc_noswz(ptx::smem_u32(bimg), 128, 256);
    const uint32_t band_off = static_cast<uint32_t>(L.band) >> 4;
    const uint32_t row_step = static_cast<uint32_t>(p.rb_rowb) >> 4;
    const uint32_t bstep = static_cast<uint32_t>(BN * 32) >> 4;  // one K16 step of the filter image
    ptx::mbar_wait(bbar, 0);
    int bi = 0, i = 0;
    for (int r = r0; r < r1; ++bi) {
      const int e = detail::rb_band_end(p, r, r0, r1);
      const int buf = bi & 1;
      if (!p.rb_fix) ptx::mbar_wait(&bfull[buf], (bi >> 1) & 1);
      else if (bi == 0) ptx::mbar_wait(bready0, 0);
      else ptx::mbar_wait(&bready[buf], ((bi >> 1) - (buf == 0 ? 1 : 0)) & 1);  // band 0 used bready0
      ptx::tc_fence_after();
      if (lane == 0) detail::rb_trace(p, r - r0, 4, t0);
      for (int rr = r; rr < e; ++rr, ++i) {
        const int acc = i % NACC;
        ptx::mbar_wait(&tempty[acc], ((i / NACC) & 1) ^ 1);
        ptx::tc_fence_after();
        if (lane == 0) detail::rb_trace(p, i, 0, t0);
        const uint32_t d = tmem_base + acc * BN;
        const uint32_t row0 = buf * band_off + static_cast<uint32_t>((rr - r) * g.stride) * row_step;
        if (ptx::elect_one()) {
          const uint64_t ar = a0 + row0;
          if constexpr (KH > 0) {
            // fully unrolled (compile-time filter rows / K16 steps): the issue loop is a
            // straight run of UTCHMMAs with independent descriptor adds -- at N = 64 an
            // MMA's tensor work is ~30 clk, so issue overhead is what bounds the tile
#pragma unroll
            for (int fh = 0; fh < KH; ++fh)
#pragma unroll
              for (int t = 0; t < STEPS; ++t)
                ptx::mma_f16(d, ar + static_cast<uint64_t>(fh) * row_step + static_cast<uint64_t>(2 * t),
                             b0 + static_cast<uint64_t>((fh * STEPS + t) * bstep), idesc, (fh | t) != 0);
          } else {
            uint32_t kstep = 0;
            for (int fh = 0; fh < g.kh; ++fh) {
              const uint64_t arf = ar + static_cast<uint32_t>(fh) * row_step;
              for (int t = 0; t < p.rb_steps; ++t, ++kstep)
                ptx::mma_f16(d, arf + static_cast<uint64_t>(2 * t), b0 + static_cast<uint64_t>(kstep * bstep), idesc,
                             kstep != 0);
            }
          }
          ptx::mma_commit(&tfull[acc]);
          detail::rb_trace(p, i, 1, t0);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma_commit(&bempty[buf]);  // band buffer reusable once these MMAs finish
      __syncwarp();
      r = e;
    }
  } else if (warp < 2 + kRbEpiWarps) {
    // ============================== epilogue ==============================
    const int e = warp - 2;         // 0..7
    const int grp = e >> 2;         // tiles i with i % 2 == grp
    const int lg = warp & 3;        // TMEM lane group (rows lg*32 .. +32)
    const int et = threadIdx.x - 64;  // 0..255
    if (p.rb_fix && r0 < r1) {  // band 0's pad lanes, while the MMA has nothing else to do
      ptx::mbar_wait(&bfull[0], 0);
      detail::rb_zero_pad_lanes(p, band[0], kRbLoadWarps * p.rb_rows0, et, kRbEpiWarps * 32);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bready0);
    }
    // canonical S / T for all F columns (one tile spans every output channel)
    for (int c = et; c < BN; c += kRbEpiWarps * 32) {
      float s = p.canon_s, t = p.canon_t;
      if (c < p.N && p.canon_s_op >= 0) {
        const EpiOp& op = p.ops[p.canon_s_op];
        s = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, 0) + c * op.a.s_col, op.dtype);
      }
      if (c < p.N && p.canon_t_op >= 0) {
        const EpiOp& op = p.ops[p.canon_t_op];
        t = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, 0) + c * op.a.s_col, op.dtype);
      }
      colbuf[c] = s;
      colbuf[BN + c] = t;
    }
    ptx::named_bar_sync(1, kRbEpiWarps * 32);
    uint8_t* obuf = outbuf + e * (32 * OUT_ROW);
    const int ncols = min(BN, p.N);
    for (int i = grp, r = r0 + grp; r < r1; i += 2, r += 2) {
      const int acc = i % NACC;
      ptx::mbar_wait(&tfull[acc], (i / NACC) & 1);
      ptx::tc_fence_after();
      if (lane == 0 && lg == 0) detail::rb_trace(p, i, 2, t0);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN;
      switch (p.canon_act) {
#define TMB_RB(A)                                                                                             \
  case A:                                                                                                     \
    detail::drain_fast<BN, 1, OUT_ROW, A, false>(&tmC, taddr, colbuf, obuf, ncols, 0, lg * 32, r, lane, nullptr, \
                                                 &tempty[acc]);                                               \
    break;
        TMB_RB(0) TMB_RB(1) TMB_RB(2)
#undef TMB_RB
        default: __trap();
      }
      if (lane == 0 && lg == 0) detail::rb_trace(p, i, 3, t0);
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tmb
