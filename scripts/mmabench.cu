// tcgen05.mma issue-rate micro-benchmark (diagnostic, not part of the library):
// one CTA per SM, one elected thread issues back-to-back kind::f16 MMAs
// (M=128, N in {64,128,256}, K=16, smem operands, fp32 accumulate in TMEM),
// optionally with a commit + mbarrier wait every `group` instructions.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mmabench scripts/mmabench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int N>
__global__ void __launch_bounds__(128, 1) k(int iters, int group, long long* out) {
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
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint64_t ad = desc_sw128(su32(sm)), bd = desc_sw128(su32(sm + 16384));
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t e;
      asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0,1,0,p;}" : "=r"(e));
      if (e) {
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                     ::"r"(tmem), "l"(ad + (uint64_t)(2 * (i & 3))), "l"(bd + (uint64_t)(2 * (i & 3))), "r"(idesc), "r"(1));
        if (group > 0 && (i + 1) % group == 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      }
      __syncwarp();
      if (group > 0 && (i + 1) % group == 0) {
        uint32_t done = 0;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(su32(&bar)), "r"(ph));
        } while (!done);
        ph ^= 1;
      }
    }
    uint32_t e;
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0,1,0,p;}" : "=r"(e));
    if (e) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    __syncwarp();
    uint32_t done = 0;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(su32(&bar)), "r"(ph));
    } while (!done);
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int N>
void run(int group) {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k<N><<<148, 128, 65536>>>(iters, group, d);
    cudaDeviceSynchronize();
  }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("N=%3d group=%3d: %.1f clk per MMA (floor %d), err=%s\n", N, group, avg / iters, 128 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int g : {0, 4, 8, 16}) { run<64>(g); run<128>(g); run<256>(g); }
  return 0;
}
