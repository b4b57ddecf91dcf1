// tcgen05.commit -> mbarrier latency micro-benchmark (diagnostic, not part of the
// library): one CTA per SM; warp 0 issues k MMAs (M=128, N=n, K=16, smem operands,
// TMEM accumulator) then a commit, and waits (poll or suspend) for the barrier;
// reports clk per (MMAs + commit + wait) round trip, averaged over 256 rounds.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o commitbench scripts/commitbench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__global__ void __launch_bounds__(128, 1) k(int n_mma, int n, int suspend, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t ad = desc_sw128(su32(sm)), bd = desc_sw128(su32(sm + 16384));
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    uint32_t ph = 0;
    t0 = clock64();
    for (int r = 0; r < 256; ++r) {
      uint32_t e;
      asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0,1,0,p;}" : "=r"(e));
      if (e) {
#pragma unroll 1
        for (int i = 0; i < n_mma; ++i)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                       ::"r"(tmem + (i % nacc) * n), "l"(ad), "l"(bd), "r"(idesc), "r"((int)(i >= nacc)));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      }
      __syncwarp();
      uint32_t done = 0;
      do {
        if (suspend)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(su32(&bar)), "r"(ph), "r"(0x989680u));
        else
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(su32(&bar)), "r"(ph));
      } while (!done);
      ph ^= 1;
    }
    t1 = clock64();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int nacc : {1, 2, 4})
    for (int n : {64, 128, 256})
      for (int m : {16, 32}) {
        const int susp = 0;
        if (nacc * n > 512) continue;
        for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 65536>>>(m, n, susp, nacc, d);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148 * 256.0;
        printf("nacc=%d N=%3d mmas=%d: %.0f clk per round, %.1f per MMA (floor %d) %s\n", nacc, n, m, avg, avg / m,
               128 * n / 256, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
