// Ring + TMA micro-benchmark (diagnostic, not part of the library): the GEMM
// mainloop's protocol with real copies.  L loader warps (lane 0 each) issue the
// two 16 KB SWIZZLE_128B boxes (A, B) of every ring slot -- box j of slot q from
// warp (2q + j) % L, the kernel's assignment -- from an L2-resident bf16 matrix;
// warp L (MMA) waits full[s], issues `nmma` kind::f16 MMAs (128x128x16) and
// commits empty[s].  Reports clk per slot vs L, ring depth and MMA count.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2210_09603_b200/csrc/device \
//        -o ringtma scripts/ringtma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "ptx.cuh"

using namespace tmb;
constexpr int kBox = 16384;

__global__ void __launch_bounds__(32 * 9, 1) k(const __grid_constant__ CUtensorMap tm, int slots, int ring, int L,
                                               int nmma, int rows_total, long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == L) ptx::tmem_alloc<256>(&tslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { ptx::mbar_init(&full[i], 2); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (warp < L) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int q = 0; q < slots; ++q) {
        const bool da = (2 * q) % L == warp, db = (2 * q + 1) % L == warp;
        if (da || db) {
          ptx::mbar_wait_poll(&empty[stage], phase ^ 1u);
          // different 128-row bands per CTA and slot (L2-resident matrix)
          const int r0 = ((blockIdx.x * 977 + q * 2) * 128) % rows_total;
          if (da) {
            ptx::mbar_arrive_expect_tx(&full[stage], kBox);
            ptx::tma_load_2d(sm + stage * 2 * kBox, &tm, &full[stage], 0, r0);
          }
          if (db) {
            ptx::mbar_arrive_expect_tx(&full[stage], kBox);
            ptx::tma_load_2d(sm + stage * 2 * kBox + kBox, &tm, &full[stage], 0, (r0 + 128) % rows_total);
          }
        }
        if (++stage == ring) { stage = 0; phase ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == L) {
    const uint32_t idesc = ptx::make_idesc(128, 128, 1u, false, false);
    int stage = 0; uint32_t phase = 0;
    for (int q = 0; q < slots; ++q) {
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(sm + stage * 2 * kBox), 16, 1024);
      const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sm + stage * 2 * kBox + kBox), 16, 1024);
      if (ptx::elect_one()) {
        for (int kk = 0; kk < nmma; ++kk)
          ptx::mma_f16(tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc, q | kk);
        ptx::mma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == ring) { stage = 0; phase ^= 1u; }
    }
    for (int j = 0; j < ring && j < slots; ++j) {
      const int q = slots - 1 - j;
      ptx::mbar_wait(&empty[q % ring], (q / ring) & 1u);
    }
  }
  long long t1 = clock64();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == L) ptx::tmem_dealloc<256>(tmem);
  if (threadIdx.x == 32 * L) out[blockIdx.x] = t1 - t0;
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 32768;  // 32768 x 64 bf16 = 4 MB: L2-resident
  void* buf; cudaMalloc(&buf, (size_t)rows * 128);
  cudaMemset(buf, 0, (size_t)rows * 128);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows}, strides[1] = {128};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeTiled>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 6 * 2 * kBox + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int slots = 512;
  for (int nmma : {0, 4})
    for (int ring : {4, 6})
      for (int L : {1, 2, 3, 4, 6, 8}) {
        for (int rep = 0; rep < 2; ++rep) {
          k<<<148, 32 * (L + 1), smem>>>(tm, slots, ring, L, nmma, rows, d);
          cudaDeviceSynchronize();
        }
        long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
        printf("mma/slot=%d ring=%d loader warps=%d: %6.1f clk per slot (%.1f B/clk/SM), err=%s\n", nmma, ring, L,
               avg / slots, 2.0 * kBox / (avg / slots), cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
