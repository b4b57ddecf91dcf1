// TMA load-throughput micro-benchmark (diagnostic, not part of the library).
// One CTA per SM; one thread streams TMA loads into an S-stage smem ring, one
// thread consumes (waits full, frees the slot).  Reports bytes/clk/SM and
// chip GB/s for: tiled 2-D boxes, im2col boxes (NHWC conv activations) and
// tiled 4-D spatial boxes over the same NHWC tensor.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tmabench scripts/tmabench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(done) : "r"(su32(b)), "r"(par) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void tma2d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma3d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma4d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_i2c(void* d, const CUtensorMap* m, uint64_t* b, int c, int w, int h, int n,
                                        uint16_t ow, uint16_t oh) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh) : "memory");
}

struct Args {
  int mode, stages, box_bytes, boxes_per_stage, iters;
  int N, H, W, C;          // NHWC tensor (modes 1, 2)
  int rows, kcols;         // 2-D matrix (mode 0)
  int bw, bh;              // spatial box (mode 2)
  int split;               // 0: 1 producer + 1 consumer per chain; 1: 2 producers (even/odd stages); 2: 2 consumers
};

__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ CUtensorMap tm, Args a, long long* cyc, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  __shared__ uint64_t fullv[8][16], emptyv[8][16];
  const int stage_bytes = a.box_bytes * a.boxes_per_stage;
  const int P = blockDim.x / 64, pw = (threadIdx.x >> 5) % P;  // producer/consumer pair index
  uint64_t* full = fullv[pw];
  uint64_t* empty = emptyv[pw];
  uint8_t* sm = smraw + pw * a.stages * stage_bytes;
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < P) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  const int wid = threadIdx.x >> 5;
  const bool lane0 = (threadIdx.x & 31) == 0;
  const int lane = threadIdx.x & 31;
  // split 3: two producer lanes (0 and 1) of warp 0, one consumer (warp 2)
  const bool prod = a.split == 3 ? (wid == 0 && lane < 2) : lane0 && (a.split == 1 ? wid < 2 : (a.split == 2 ? wid == 0 : wid < P));
  const bool cons = lane0 && (a.split == 1 || a.split == 3 ? wid == 2 : (a.split == 2 ? (wid == 2 || wid == 3) : wid >= P));
  const int role_par = a.split == 3 ? lane : a.split == 1 ? wid : (a.split == 2 ? wid - 2 : -1);  // which parity of stage index this thread handles
  if (a.split) { full = fullv[0]; empty = emptyv[0]; sm = smraw; }
  if (prod) {
    int s = 0; uint32_t ph = 0;
    uint32_t x = (blockIdx.x * 8 + pw) * 2654435761u;
    for (int i = 0; i < a.iters; ++i) {
      if ((a.split == 1 || a.split == 3) && (i & 1) != role_par) { if (++s == a.stages) { s = 0; ph ^= 1; } continue; }
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect(&full[s], stage_bytes);
      for (int j = 0; j < a.boxes_per_stage; ++j) {
        uint8_t* dst = sm + s * stage_bytes + j * a.box_bytes;
        x = x * 1664525u + 1013904223u;
        if (a.mode == 6) {
          const size_t off = (size_t)((blockIdx.x * 7 + i * a.boxes_per_stage + j) % 700) * a.box_bytes;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(dst)), "l"(gsrc + off), "r"(a.box_bytes), "r"(su32(&full[s])) : "memory");
        } else if (a.mode == 5) {
          const int kc = a.box_bytes / (a.bw * 128);
          const int kb = (i * a.boxes_per_stage + j) % (a.kcols / (64 * kc));
          const int rb = (blockIdx.x + 148 * ((i * a.boxes_per_stage + j) / (a.kcols / (64 * kc)))) % (a.rows / a.bw);
          tma3d(dst, &tm, &full[s], 0, rb * a.bw, kb * kc);
        } else if (a.mode == 3) {
          const int kb = (i * a.boxes_per_stage + j) % (a.kcols / 64);
          const int rb = (blockIdx.x + 148 * ((i * a.boxes_per_stage + j) / (a.kcols / 64))) % (a.rows / (a.box_bytes / 128));
          tma2d(dst, &tm, &full[s], kb * 64, rb * (a.box_bytes / 128));
        } else if (a.mode == 0 || a.mode == 4) {
          const int kb = (x >> 8) % (a.kcols / 64);
          const int rb = (x >> 20) % (a.rows / (a.box_bytes / 128));
          tma2d(dst, &tm, &full[s], kb * 64, rb * (a.box_bytes / 128));
        } else if (a.mode == 1) {
          const int pix = ((x >> 4) % (a.N * a.H * a.W / 128)) * 128;
          const int n = pix / (a.H * a.W), r = pix % (a.H * a.W);
          const int tap = (x >> 24) % 9, cb = (x >> 12) % (a.C / 64);
          tma_i2c(dst, &tm, &full[s], cb * 64, r % a.W - 1, r / a.W - 1, n, tap % 3, tap / 3);
        } else {
          const int n = (x >> 4) % a.N, tap = (x >> 24) % 9, cb = (x >> 12) % (a.C / 64);
          const int tw = (x >> 16) % ((a.W + a.bw - 1) / a.bw), th = (x >> 20) % ((a.H + a.bh - 1) / a.bh);
          tma4d(dst, &tm, &full[s], cb * 64, tw * a.bw - 1 + tap % 3, th * a.bh - 1 + tap / 3, n);
        }
      }
      if (++s == a.stages) { s = 0; ph ^= 1; }
    }
  } else if (cons) {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < a.iters; ++i) {
      if (a.split == 2 && (i & 1) != role_par) { if (++s == a.stages) { s = 0; ph ^= 1; } continue; }
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == a.stages) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;  // (each producer moves a.iters stages)
}

typedef CUresult (*EncT)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncI)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                         CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int promo = argc > 3 ? atoi(argv[3]) : 2, swz = argc > 4 ? atoi(argv[4]) : 3;
  int grid = argc > 1 ? atoi(argv[1]) : 148;
  void* fT = nullptr; void* fI = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fT, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fI, cudaEnableDefault, &q));
  EncT encT = (EncT)fT; EncI encI = (EncI)fI;
  // NHWC activations of ResNet l3.c2 (batch 32, 14x14, 256 ch) and a 2-D matrix of the same order of size
  const int N = 32, H = 14, W = 14, C = 256;
  const size_t act_bytes = (size_t)N * H * W * C * 2;
  const int rows = 8192, kcols = 768;
  void *act, *mat;
  CK(cudaMalloc(&act, act_bytes)); CK(cudaMalloc(&mat, (size_t)rows * kcols * 2));
  cudaMemset(act, 0, act_bytes); cudaMemset(mat, 0, (size_t)rows * kcols * 2);
  long long* cyc; CK(cudaMalloc(&cyc, grid * 8));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  struct Case { const char* name; int mode, box_rows, boxes, stages, bw, bh; };
  Case sweep[] = {
      {"im2col 128px x1", 1, 128, 1, 4, 0, 0}, {"tiled 2D 64x128B x1", 0, 64, 1, 4, 0, 0},
      {"bulk1D 16KB", 6, 128, 1, 6, 0, 0}, {"bulk1D 64KB", 6, 512, 1, 3, 0, 0}, {"bulk1D 4KB", 6, 32, 1, 12, 0, 0},
      {"3D 128r x 2kc (32KB)", 5, 128, 1, 4, 128, 2}, {"3D 128r x 4kc (64KB)", 5, 128, 1, 3, 128, 4},
      {"3D 256r x 2kc (64KB)", 5, 256, 1, 3, 256, 2}, {"3D 64r x 4kc (32KB)", 5, 64, 1, 4, 64, 4},
      {"3D 128r x 1kc (16KB)", 5, 128, 1, 6, 128, 1},
      {"seqK 2D 128x128B", 3, 128, 1, 6, 0, 0}, {"seqK 2D 128x128B x2", 3, 128, 2, 4, 0, 0},
      {"seqK 2D 256x128B", 3, 256, 1, 4, 0, 0},
      {"contig 2D 128x128B", 4, 128, 1, 6, 0, 0}, {"contig 2D 128x128B x2", 4, 128, 2, 4, 0, 0},
      {"tiled 2D 128x128B", 0, 128, 1, 1, 0, 0}, {"tiled 2D 128x128B", 0, 128, 1, 2, 0, 0},
      {"tiled 2D 128x128B", 0, 128, 1, 4, 0, 0}, {"tiled 2D 128x128B", 0, 128, 1, 12, 0, 0},
      {"tiled 2D 128x128B x2", 0, 128, 2, 1, 0, 0}, {"tiled 2D 128x128B x4", 0, 128, 4, 1, 0, 0},
      {"tiled 2D 128x128B x8", 0, 128, 8, 1, 0, 0}, {"tiled 2D 128x128B x4", 0, 128, 4, 3, 0, 0},
      {"tiled 2D 32x128B x8", 0, 32, 8, 4, 0, 0},
      {"im2col 128px x4", 1, 128, 4, 3, 0, 0}, {"im2col 128px x1", 1, 128, 1, 1, 0, 0},
  };
  Case cases[] = {
      {"tiled 2D 128x128B", 0, 128, 1, 8, 0, 0},   {"tiled 2D 256x128B", 0, 256, 1, 6, 0, 0},
      {"tiled 2D 128x128B x3", 0, 128, 3, 4, 0, 0}, {"tiled 2D 64x128B", 0, 64, 1, 12, 0, 0},
      {"im2col 128px x128B", 1, 128, 1, 8, 0, 0},  {"im2col 128px x128B x2", 1, 128, 2, 4, 0, 0},
      {"im2col 64px x128B", 1, 64, 1, 12, 0, 0},   {"im2col 256px x128B", 1, 256, 1, 6, 0, 0},
      {"tiled 4D 16x8px x128B", 2, 128, 1, 8, 16, 8}, {"tiled 4D 8x16px x128B", 2, 128, 1, 8, 8, 16},
      {"tiled 4D 14x8px(pad16) x128B", 2, 128, 1, 8, 16, 8},
  };
  const bool do_sweep = argc > 2;
  const int ncase = do_sweep ? sizeof(sweep) / sizeof(Case) : sizeof(cases) / sizeof(Case);
  for (int ci = 0; ci < ncase; ++ci) {
    const Case& c = do_sweep ? sweep[ci] : cases[ci];
    CUtensorMap tm;
    Args a{};
    a.mode = c.mode; a.stages = c.stages; a.box_bytes = c.box_rows * 128; a.boxes_per_stage = c.boxes;
    a.iters = 2000; a.N = N; a.H = H; a.W = W; a.C = C; a.rows = rows; a.kcols = kcols; a.bw = c.bw; a.bh = c.bh;
    if (c.mode == 5) {
      a.box_bytes = c.box_rows * 128 * c.bh;  // rows x 128 B x kchunks
      cuuint64_t d[3] = {64, (cuuint64_t)rows, (cuuint64_t)kcols / 64}, s[2] = {(cuuint64_t)kcols * 2, 128};
      cuuint32_t b[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.bh}, e[3] = {1, 1, 1};
      CK(encT(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, mat, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    } else if (c.mode == 6) {
      tm = CUtensorMap{};
    } else if (c.mode == 0 || c.mode == 3 || c.mode == 4) {
      if (c.mode == 4) { a.kcols = 64; a.rows = rows * kcols / 64; }
      cuuint64_t d[2] = {(cuuint64_t)a.kcols, (cuuint64_t)a.rows}, s[1] = {(cuuint64_t)a.kcols * 2};
      cuuint32_t b[2] = {64, (cuuint32_t)c.box_rows}, e[2] = {1, 1};
      CK(encT(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
              (CUtensorMapSwizzle)swz, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    } else if (c.mode == 1) {
      cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t s[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
      int lo[2] = {-1, -1}, hi[2] = {-1, -1};
      cuuint32_t e[4] = {1, 1, 1, 1};
      CK(encI(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, act, d, s, lo, hi, 64, c.box_rows, e,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    } else {
      cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t s[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
      cuuint32_t b[4] = {64, (cuuint32_t)c.bw, (cuuint32_t)c.bh, 1}, e[4] = {1, 1, 1, 1};
      CK(encT(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, act, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    }
    const int P = argc > 5 ? atoi(argv[5]) : 1;
    a.split = argc > 6 ? atoi(argv[6]) : 0;
    if (a.split && (P != 2 || (a.stages & 1))) continue;
    const int smem = (a.split ? 1 : P) * a.stages * a.box_bytes * a.boxes_per_stage;
    if (smem > 200 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<grid, 64 * P, smem>>>(tm, a, cyc, (const uint8_t*)mat);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long h[148 * 2]; cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; double avg = 0;
      for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i]; }
      avg /= grid;
      const double bytes = (double)(a.split ? 1 : P) * a.iters * a.box_bytes * a.boxes_per_stage;
      if (rep) printf("%-30s stages %2d  %7.1f B/clk/SM  %8.0f GB/s chip  (%.3f ms, %.0f clk/box)\n", c.name, a.stages,
                      bytes / avg, bytes * grid / (ms * 1e6), ms, avg / ((a.split ? 1 : P) * a.iters * a.boxes_per_stage));
    }
  }
  return 0;
}
