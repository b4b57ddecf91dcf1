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

template <int NMMA, bool POLL, int N = 128>
__global__ void __launch_bounds__(64, 1) k(int slots, int ring, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x / 32;
  if (warp == 1) ptx::tmem_alloc<512>(&tslot);
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
    const uint32_t idesc = ptx::make_idesc(128, N, 1u, false, false);
    const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(sm), 16, 1024);
    const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(sm + 4 * 16384), 16, 1024);
    int stage = 0; uint32_t phase = 0;
    for (int q = 0; q < slots; ++q) {
      if (POLL) ptx::mbar_wait_poll(&full[stage], phase); else ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint64_t ad = ad0 + static_cast<uint64_t>(((stage & 3) * 16384) >> 4);
      const uint64_t bd = bd0 + static_cast<uint64_t>(((stage & 1) * 32768) >> 4);
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < NMMA; ++kk)
          ptx::mma_f16(tmem, ad + static_cast<uint64_t>((kk & 3) * 2), bd + static_cast<uint64_t>((kk & 3) * 2), idesc, q | kk);
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
  if (warp == 1) ptx::tmem_dealloc<512>(tmem);
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int NMMA, bool POLL, int N = 128>
void run(int ring) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 4 * 16384 + 2 * 32768 + 1024;
  cudaFuncSetAttribute(k<NMMA, POLL, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int slots = 1024;
  for (int rep = 0; rep < 2; ++rep) {
    k<NMMA, POLL, N><<<148, 64, smem>>>(slots, ring, d);
    cudaDeviceSynchronize();
  }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("N=%d mma/slot=%d %s ring=%d: %6.1f clk per slot, %5.1f per MMA (floor %d), err=%s\n", N, NMMA, POLL ? "poll   " : "suspend", ring,
         avg / slots, avg / slots / (NMMA ? NMMA : 1), N / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<4, false>(4); run<8, false>(4); run<16, false>(4); run<32, false>(4);
  run<4, false, 256>(4); run<8, false, 256>(4); run<16, false, 256>(4);
  run<4, false, 64>(4); run<16, false, 64>(4);
  return 0;
}
