// Ring handshake micro-benchmark (diagnostic, not part of the library): the GEMM
// mainloop's protocol without copies.  Warp 0 (loader) polls empty[s] and arrives
// on full[s]; warp 1 (MMA) waits full[s], issues `nmma` kind::f16 MMAs (M=128,
// N=128, K=16) from one elected lane of the warp-uniform loop, and commits
// empty[s].  Reports clk per ring slot for ring depths 2..8, MMA counts 0/4/8,
// suspending vs polling MMA-side wait.  One CTA per SM.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2210_09603_b200/csrc/device \
//        -o ringbench scripts/ringbench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "ptx.cuh"

using namespace tmb;

template <int NMMA, bool POLL>
__global__ void __launch_bounds__(64, 1) k(int slots, int ring, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x / 32;
  if (warp == 1) ptx::tmem_alloc<256>(&tslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (warp == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int q = 0; q < slots; ++q) {
      ptx::mbar_wait_poll(&empty[stage], phase ^ 1u);
      if (ptx::lane_id() == 0) ptx::mbar_arrive(&full[stage]);
      __syncwarp();
      if (++stage == ring) { stage = 0; phase ^= 1u; }
    }
  } else {
    const uint32_t idesc = ptx::make_idesc(128, 128, 1u, false, false);
    const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(sm), 16, 1024);
    const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(sm + 8 * 16384), 16, 1024);
    int stage = 0; uint32_t phase = 0;
    for (int q = 0; q < slots; ++q) {
      if (POLL) ptx::mbar_wait_poll(&full[stage], phase); else ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint64_t ad = ad0 + static_cast<uint64_t>((stage * 16384) >> 4);
      const uint64_t bd = bd0 + static_cast<uint64_t>((stage * 4096) >> 4);
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < NMMA; ++kk)
          ptx::mma_f16(tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc, q | kk);
        ptx::mma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == ring) { stage = 0; phase ^= 1u; }
    }
    // drain: the last commits
    for (int j = 0; j < ring && j < slots; ++j) {
      const int q = slots - 1 - j;
      ptx::mbar_wait(&empty[q % ring], (q / ring) & 1u);
    }
  }
  long long t1 = clock64();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<256>(tmem);
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int NMMA, bool POLL>
void run(int ring) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 8 * 16384 + 8 * 4096 + 1024;
  cudaFuncSetAttribute(k<NMMA, POLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int slots = 1024;
  for (int rep = 0; rep < 2; ++rep) {
    k<NMMA, POLL><<<148, 64, smem>>>(slots, ring, d);
    cudaDeviceSynchronize();
  }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("mma/slot=%d %s ring=%d: %6.1f clk per slot (MMA floor %d), err=%s\n", NMMA, POLL ? "poll   " : "suspend", ring,
         avg / slots, NMMA * 64, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int r : {2, 4, 5, 8}) { run<0, false>(r); run<0, true>(r); }
  for (int r : {2, 4, 5, 8}) { run<4, false>(r); run<4, true>(r); }
  for (int r : {4, 8}) { run<8, false>(r); run<8, true>(r); }
  return 0;
}
