// Halo implicit-GEMM convolution for stride-1 convs on channels-last inputs
// with C % 64 == 0 (the ResNet-50 3x3 layers), sm_100a.
//
// The K3 kernel stages one im2col tile per (tap, 64-channel block) k-block: a 3x3
// conv streams every input pixel through shared memory nine times, and narrow
// tiles are bounded by that traffic (the ring round trip).  Here
// the im2col operand is never materialised.  A tile is R consecutive output rows
// of one image, each as P = Wo + 2 pad "virtual" pixels (the 2 pad halo columns
// compute values that are never stored), R * P <= 128 rows on the TMEM lanes.
// The tile's input band -- R + kh - 1 rows of P pixels, zero outside the image
// (TMA out-of-bounds fill) -- is staged once, channel-group-major:
//   band[g][row][px][8 channels]          (one 5-D TMA box, g = channel / 8)
// so lane r = j * P + ow (output row j, column ow; ow >= Wo are the dead "virtual"
// pixels) reads, for tap (fh, fw), staged pixel (j + fh) * P + ow + fw -- input
// column ow + fw - pad -- i.e. byte (r + fh * P + fw) * 16 of its channel group.  For k-block (tap, cb) and K16 step t the UMMA A operand is a
// no-swizzle K-major matrix with
//   start = band + (8 cb + 2 t) * G + (fh * P + fw) * 16,  SBO = 128 B,  LBO = G
// (G = bytes per channel group of the band): every tap reads the same staged
// band through its own descriptor offset.  The filter (OHWI = K-major with K order
// (tap, c)) streams through a ring of NB-k-block stages, one 3-D TMA box each.
// Epilogue: canonical BN-fold + activation, direct 16-byte stores of the valid
// lanes (consecutive pixels of a channels-last output row are contiguous).
//
// Schedule: tiles (image, output-row block, F block) spread over a persistent grid
// in contiguous ranges (spatial(G) * repeat(T/G)); bands double-buffered; warps 0
// producer (bands + filter ring), 1 MMA issuer / TMEM owner, 2-9 epilogue (two
// groups alternating tiles).
#pragma once
#include "conv_rowband.cuh"  // rb_trace, drain helpers

namespace tmb {

constexpr int kHbThreads = 320;  // 10 warps
constexpr int kHbEpiWarps = 8;
constexpr int kHbMaxKb = 128;    // k-blocks per tile (kh * kw * C / 64)

// smem carve-up shared by host (sizing) and device
struct HbLayout {
  int band, ring, colbuf, kbtab, bars, total;
  __host__ __device__ static int align(int x) { return (x + 1023) & ~1023; }
  // nbands: 2 (the next tile's band loads while this one's MMAs run) or 1 when no CTA
  // has a second tile (the freed band deepens the filter ring)
  __host__ __device__ HbLayout(int band_bytes, int stage_bytes, int stages, int bn, int nbands = 2) {
    band = align(band_bytes);
    ring = nbands * band;
    colbuf = ring + stages * stage_bytes;
    kbtab = colbuf + 4 * bn * 4;  // S / T per epilogue group
    bars = kbtab + kHbMaxKb * 4;
    total = bars + 512;
  }
};

namespace detail {

// This CTA's work items [t0, t1).  hb_mc == 1: tiles.  hb_mc == 2: units of the CTA
// pair (cluster) -- unit u = (spatial pair j, column block f); both CTAs walk the same
// units, so they consume the same filter stages in the same order (each loads half of
// every stage and multicasts it to both).
__device__ __forceinline__ void hb_range(const GemmParams& p, int& t0, int& t1) {
  int64_t T = p.hb_total, G = gridDim.x, b = blockIdx.x;
  if (p.hb_mc == 2) {
    const int64_t S = p.hb_total / p.hb_ftiles;
    T = (S + 1) / 2 * p.hb_ftiles;
    G /= 2;
    b /= 2;
  }
  t0 = static_cast<int>(T * b / G);
  t1 = static_cast<int>(T * (b + 1) / G);
}

// tile t -> (image n, first output row oh0, rows in this tile, column tile f)
// hb_mc == 2: work item t is a pair unit; this CTA (cluster rank r) takes spatial tile
// 2j + r.  With an odd spatial count the last unit's rank-1 tile is a duplicate of
// rank 0's (it still walks the shared filter stages) and stores nothing (rows = 0).
__device__ __forceinline__ void hb_tile(const GemmParams& p, int t, int& n, int& oh0, int& rows, int& f) {
  f = t % p.hb_ftiles;
  int s = t / p.hb_ftiles;
  bool dup = false;
  if (p.hb_mc == 2) {
    s = 2 * s + static_cast<int>(blockIdx.x & 1u);
    dup = s >= p.hb_total / p.hb_ftiles;
    if (dup) --s;
  }
  n = s / p.hb_tpi;
  oh0 = (s - n * p.hb_tpi) * p.hb_R;
  rows = dup ? 0 : min(p.hb_R, p.conv.ho - oh0);
}

}  // namespace detail

// NBT: k-blocks per filter stage (compile time: the MMA burst is unrolled)
template <int BN, int NBT>
__global__ void __launch_bounds__(kHbThreads, 1)
    tm_halo_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmW) {
  constexpr int NACC = 2;
  constexpr uint32_t TMEM_COLS = NACC * BN <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NB = NBT;  // k-blocks per filter stage (host: p.rb_steps)
  const int stage_bytes = NB * BN * 128;
  const HbLayout L(p.hb_band, stage_bytes, p.hb_stages, BN, p.hb_nbands);
  uint8_t* band[2] = {smem, smem + (p.hb_nbands == 2 ? L.band : 0)};
  uint8_t* ring = smem + L.ring;
  float* colbuf = reinterpret_cast<float*>(smem + L.colbuf);
  uint32_t* kbtab = reinterpret_cast<uint32_t*>(smem + L.kbtab);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* bfull = bars;              // [2][8] band chunk (64 channels) staged
  uint64_t* bempty = bars + 16;        // [2] band's MMAs done
  uint64_t* tfull = bars + 18;         // [2] accumulator ready
  uint64_t* tempty = bars + 20;        // [2] accumulator drained
  uint64_t* sfull = bars + 22;         // [<=8] filter stage landed
  uint64_t* sempty = bars + 30;        // [<=8] filter stage consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 38);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ConvGeom& g = p.conv;
  const int cblocks = g.c / 64;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmX);
    ptx::tma_prefetch_desc(&tmW);
    for (int i = 0; i < 16; ++i) ptx::mbar_init(&bfull[i], 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bempty[i], 1);
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4);
    }
    for (int s = 0; s < p.hb_stages; ++s) {
      ptx::mbar_init(&sfull[s], 1);
      ptx::mbar_init(&sempty[s], p.hb_mc);  // both CTAs' MMAs release a shared stage
    }
    ptx::fence_mbar_init();
  }
  // per k-block A offset (16-byte units): tap (fh, fw) shift + channel-block groups
  const int taps = g.kh * g.kw;
  for (int kb = threadIdx.x; kb < p.hb_kb; kb += blockDim.x) {  // K order (64-channel block, tap)
    const int cb = kb / taps, tap = kb - cb * taps;
    const int fh = tap / g.kw, fw = tap - fh * g.kw;
    kbtab[kb] = static_cast<uint32_t>(((fh * p.hb_P + fw) * 16 + 8 * cb * p.hb_G) >> 4);
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  if (p.hb_mc == 2) ptx::cluster_sync();  // the peer's barriers exist before any multicast lands
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();

  int t0, t1;
  detail::hb_range(p, t0, t1);
  const long long clk0 = clock64();

  if (warp == 0) {
    // ======================= producer: bands + filter ring =======================
    // the band arrives in 64-channel chunks (8 channel groups, one 5-D box and one
    // barrier each), so the MMAs of chunk 0 start while the rest is in flight
    const uint32_t chunk_tx = static_cast<uint32_t>(p.hb_G * 8);
    int stage = 0;
    uint32_t sphase = 0;
    for (int t = t0; t < t1; ++t) {
      const int i = t - t0, bb = i & 1;
      int n, oh0, rows, f;
      detail::hb_tile(p, t, n, oh0, rows, f);
      if (i >= 2) ptx::mbar_wait_poll(&bempty[bb], ((i >> 1) - 1) & 1);
      if (lane == 0) {
        detail::rb_trace(p, i, 5, clk0);
        for (int cb = 0; cb < cblocks; ++cb) {
          ptx::mbar_arrive_expect_tx(&bfull[bb * 8 + cb], chunk_tx);
          // box {8 ch, P px, rows, 8 groups, 1 image} at (0, -pad, oh0 - pad, 8 cb, n)
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(ptx::smem_u32(band[bb] + 8 * cb * p.hb_G)),
              "l"(reinterpret_cast<uint64_t>(&tmX)), "r"(ptx::smem_u32(&bfull[bb * 8 + cb])), "r"(0), "r"(-g.pad),
              "r"(oh0 - g.pad), "r"(8 * cb), "r"(n)
              : "memory");
        }
      }
      __syncwarp();
      // filter stages of this tile's column block: NB taps of one 64-channel block each
      for (int cb = 0; cb < cblocks; ++cb)
        for (int tap0 = 0; tap0 < taps; tap0 += NB) {
          ptx::mbar_wait_poll(&sempty[stage], sphase ^ 1u);
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&sfull[stage], static_cast<uint32_t>(stage_bytes));
            if (p.hb_mc == 2) {
              // this CTA's half of the stage (half the taps, or half the filter rows),
              // multicast into both CTAs of the pair at the same offset
              const int r = static_cast<int>(blockIdx.x & 1u);
              ptx::tma_load_4d_mc(ring + stage * stage_bytes + r * (stage_bytes / 2), &tmW, &sfull[stage], 0,
                                  f * BN + (p.hb_split ? 0 : r * (BN / 2)), cb, tap0 + (p.hb_split ? r * (NB / 2) : 0),
                                  0x3);
            } else {
              ptx::tma_load_4d(ring + stage * stage_bytes, &tmW, &sfull[stage], 0, f * BN, cb, tap0);
            }
          }
          __syncwarp();
          if (++stage == p.hb_stages) { stage = 0; sphase ^= 1u; }
        }
    }
    // producer tail: the last bands' and stages' MMAs have completed
    const int nt = t1 - t0;
    if (nt >= 1) ptx::mbar_wait(&bempty[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
    if (nt >= 2) ptx::mbar_wait(&bempty[(nt - 2) & 1], ((nt - 2) >> 1) & 1);
    if (p.hb_mc == 2) {
      // and the peer's releases of the last stages have landed here (no remote
      // arrival may target this CTA after it exits)
      const int used = nt * cblocks * ((taps + NB - 1) / NB);
      for (int u = max(0, used - p.hb_stages); u < used; ++u)
        ptx::mbar_wait(&sempty[u % p.hb_stages], (u / p.hb_stages) & 1);
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    const uint32_t idesc = ptx::make_idesc(128, BN, p.ab_f16 ? 0u : 1u, false, false);
    const uint32_t G16 = static_cast<uint32_t>(p.hb_G);
    const uint64_t a0 = ptx::smem_desc_noswz(ptx::smem_u32(band[0]), G16, 128);
    const uint64_t b0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
    const uint32_t band_step = static_cast<uint32_t>(L.band) >> 4;
    const uint32_t g2 = (2u * G16) >> 4;  // K16 step: two channel groups
    int stage = 0, stage_l = 0;
    uint32_t sphase = 0, sphase_l = 0;
    for (int t = t0; t < t1; ++t) {
      const int i = t - t0, bb = i & 1, acc = i & 1;
      ptx::mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) detail::rb_trace(p, i, 0, clk0);
      const uint32_t d = tmem_base + acc * BN;
      const uint64_t ab = a0 + bb * band_step;
      if constexpr (NBT >= 4) {
        // Stages of 4 k-blocks (16 MMAs): the whole warp walks the tile (warp-uniform
        // control flow, descriptors in uniform registers) and one elected lane issues
        // each stage's burst and commit.  Smaller stages keep the single-lane walk
        // below: the per-stage reconvergence costs more than the uniform issue saves
        // (measured, 1 B200: l1.c2 NB=4 21.3 -> 20.4 us uniform; l2.c2 NB=2 16.2 ->
        // 17.1 us and l3.c2 NB=1 16.1 -> 18.5 us if made uniform).
        constexpr uint32_t bsub = static_cast<uint32_t>(BN * 128) >> 4;  // next tap in a stage
        int kb = 0;
        for (int cb = 0; cb < cblocks; ++cb) {
          ptx::mbar_wait(&bfull[bb * 8 + cb], (i >> 1) & 1);  // this 64-channel chunk of the band
          for (int tap0 = 0; tap0 < taps; tap0 += NBT) {
            ptx::mbar_wait(&sfull[stage], sphase);
            ptx::tc_fence_after();
            const uint64_t bs = b0 + static_cast<uint64_t>((stage * stage_bytes) >> 4);
            const int kbn = min(NBT, taps - tap0);
            uint32_t off[NBT];
#pragma unroll
            for (int s2 = 0; s2 < NBT; ++s2) off[s2] = kbtab[kb + min(s2, kbn - 1)];
            if (ptx::elect_one()) {
#pragma unroll
              for (int s2 = 0; s2 < NBT; ++s2) {
                if (s2 < kbn) {
                  const uint64_t ak = ab + off[s2];
                  const uint64_t bk = bs + static_cast<uint64_t>(s2 * bsub);
#pragma unroll
                  for (int q = 0; q < 4; ++q)
                    ptx::mma_f16(d, ak + static_cast<uint64_t>(q * g2), bk + static_cast<uint64_t>(2 * q), idesc,
                                 (kb + s2 + q) != 0);
                }
              }
              // stage reusable once these MMAs finish (in both CTAs of a pair)
              if (p.hb_mc == 2) ptx::mma_commit_mc(&sempty[stage], 0x3);
              else ptx::mma_commit(&sempty[stage]);
            }
            __syncwarp();
            if (++stage == p.hb_stages) { stage = 0; sphase ^= 1u; }
            kb += kbn;
          }
        }
      } else {
        // One elected lane issues the tile: per filter stage, its NB k-blocks' A
        // offsets (precomputed in smem) are read first, then the stage's 4 NB MMAs go
        // out as one straight-line burst (looped issue measured ~100+ clk per MMA;
        // unrolled bursts run near the pacing floor)
        if (ptx::elect_one()) {
          constexpr uint32_t bsub = static_cast<uint32_t>(BN * 128) >> 4;  // next tap in a stage
          int kb = 0;
          for (int cb = 0; cb < cblocks; ++cb) {
            ptx::mbar_wait(&bfull[bb * 8 + cb], (i >> 1) & 1);  // this 64-channel chunk of the band
            for (int tap0 = 0; tap0 < taps; tap0 += NBT) {
              ptx::mbar_wait(&sfull[stage], sphase);
              ptx::tc_fence_after();
              const uint64_t bs = b0 + static_cast<uint64_t>((stage * stage_bytes) >> 4);
              const int kbn = min(NBT, taps - tap0);
              uint32_t off[NBT];
#pragma unroll
              for (int s2 = 0; s2 < NBT; ++s2) off[s2] = kbtab[kb + min(s2, kbn - 1)];
#pragma unroll
              for (int s2 = 0; s2 < NBT; ++s2) {
                if (s2 < kbn) {
                  const uint64_t ak = ab + off[s2];
                  const uint64_t bk = bs + static_cast<uint64_t>(s2 * bsub);
#pragma unroll
                  for (int q = 0; q < 4; ++q)
                    ptx::mma_f16(d, ak + static_cast<uint64_t>(q * g2), bk + static_cast<uint64_t>(2 * q), idesc,
                                 (kb + s2 + q) != 0);
                }
              }
              // stage reusable once these MMAs finish (in both CTAs of a pair)
              if (p.hb_mc == 2) ptx::mma_commit_mc(&sempty[stage], 0x3);
              else ptx::mma_commit(&sempty[stage]);
              if (++stage == p.hb_stages) { stage = 0; sphase ^= 1u; }
              kb += kbn;
            }
          }
        }
        __syncwarp();
        {  // every lane tracks the ring position the elected lane reached
          const int nst = cblocks * ((taps + NBT - 1) / NBT);
          for (int j = 0; j < nst; ++j)
            if (++stage_l == p.hb_stages) { stage_l = 0; sphase_l ^= 1u; }
          stage = stage_l;
          sphase = sphase_l;
        }
      }
      if (ptx::elect_one()) {
        ptx::mma_commit(&tfull[acc]);
        ptx::mma_commit(&bempty[bb]);
        detail::rb_trace(p, i, 1, clk0);
      }
      __syncwarp();
    }
  } else {
    // ============================== epilogue ==============================
    const int e = warp - 2;           // 0..7
    const int grp = e >> 2;           // tiles i with i % 2 == grp
    const int lg = warp & 3;          // TMEM lane group (rows lg*32 .. +32)
    const int r = lg * 32 + lane;     // this lane's tile row
    const int jrow = r / p.hb_P, ow = r - jrow * p.hb_P;  // virtual pixel = output column
    const bool col_ok = ow < g.wo;  // the last 2 pad virtual pixels of each row are not outputs
    int staged_f = -1;
    for (int t = t0 + grp; t < t1; t += 2) {
      const int i = t - t0, acc = i & 1;
      int n, oh0, rows, f;
      detail::hb_tile(p, t, n, oh0, rows, f);
      if (f != staged_f) {  // this group's S / T for column block f
        ptx::named_bar_sync(1 + grp, 128);
        const int gt = lg * 32 + lane;
        for (int c = gt; c < BN; c += 128) {
          const int col = f * BN + c;
          float s = p.canon_s, tt = p.canon_t;
          if (col < p.N && p.canon_s_op >= 0) {
            const EpiOp& op = p.ops[p.canon_s_op];
            s = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, 0) + col * op.a.s_col, op.dtype);
          }
          if (col < p.N && p.canon_t_op >= 0) {
            const EpiOp& op = p.ops[p.canon_t_op];
            tt = detail::load_side(op.ptr, detail::addr_rowpart(op.a, 0, 0) + col * op.a.s_col, op.dtype);
          }
          colbuf[grp * 2 * BN + c] = s;
          colbuf[grp * 2 * BN + BN + c] = tt;
        }
        ptx::named_bar_sync(1 + grp, 128);
        staged_f = f;
      }
      ptx::mbar_wait(&tfull[acc], (i >> 1) & 1);
      ptx::tc_fence_after();
      if (lane == 0 && lg == 0) detail::rb_trace(p, i, 2, clk0);
      const bool ok = col_ok && jrow < rows;
      __nv_bfloat16* orow = nullptr;
      if (ok) {
        const int64_t m = (static_cast<int64_t>(n) * g.ho + oh0 + jrow) * g.wo + ow;
        orow = static_cast<__nv_bfloat16*>(p.out) + detail::addr_rowpart(p.out_a, m, 0) + static_cast<int64_t>(f) * BN;
      }
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t rr[32];
        ptx::tmem_ld32(taddr + c, rr);
        ptx::tmem_wait_ld();
        if (c + 32 >= BN) {  // last TMEM read of this accumulator
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 sv = *reinterpret_cast<const float4*>(colbuf + grp * 2 * BN + c + 4 * q);
          const float4 tv = *reinterpret_cast<const float4*>(colbuf + grp * 2 * BN + BN + c + 4 * q);
          float x[4] = {fmaf(__uint_as_float(rr[4 * q]), sv.x, tv.x), fmaf(__uint_as_float(rr[4 * q + 1]), sv.y, tv.y),
                        fmaf(__uint_as_float(rr[4 * q + 2]), sv.z, tv.z), fmaf(__uint_as_float(rr[4 * q + 3]), sv.w, tv.w)};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (p.canon_act == 1) x[k] = fmaxf(x[k], 0.f);
            else if (p.canon_act == 2) x[k] = detail::gelu_tanh_fast(x[k]);
          }
          w[2 * q] = detail::pack_bf16x2(x[0], x[1]);
          w[2 * q + 1] = detail::pack_bf16x2(x[2], x[3]);
        }
        if (ok && f * BN + c < p.N) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            *reinterpret_cast<uint4*>(orow + c + 8 * k) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        }
      }
      if (lane == 0 && lg == 0) detail::rb_trace(p, i, 3, clk0);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (p.hb_mc == 2) ptx::cluster_sync();  // both producers' tails done: no arrival in flight
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tmb
