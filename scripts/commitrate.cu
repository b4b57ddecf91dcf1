// tcgen05.commit throughput micro-benchmark (diagnostic, not part of the library).
// One CTA per SM; one elected lane issues `groups` groups of `per` unrolled
// kind::f16 MMAs (M=128, N, K=16, smem operands) and, every `cevery` groups, a
// commit onto ring barrier (g / cevery) % 8 -- the shape of the GEMM mainloop's
// per-k-block commit -- without waiting (a second warp consumes the barriers in
// order, like the loaders).  Reports clk per MMA: if commits had a throughput
// limit above the MMA time of a group, clk/MMA would fall as `cevery` grows.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o commitrate scripts/commitrate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
               ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(1));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(done) : "r"(su32(bar)), "r"(ph));
  } while (!done);
}

template <int N, int PER, int NACC>
__global__ void __launch_bounds__(64, 1) k(int groups, int cevery, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[8];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const int ncommit = groups / cevery;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint64_t ad = desc_sw128(su32(sm)), bd = desc_sw128(su32(sm + 65536));
    for (int g = 0; g < groups; ++g) {
      uint32_t e;
      asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0,1,0,p;}" : "=r"(e));
      if (e) {
        const uint64_t a = ad + (uint64_t)((g & 3) * 1024), b = bd + (uint64_t)((g & 3) * 1024);
#pragma unroll
        for (int j = 0; j < PER; ++j) mma(tmem + (j % NACC) * N, a + 2 * j, b + 2 * j, idesc);
        if ((g + 1) % cevery == 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(su32(&bar[((g + 1) / cevery - 1) & 7])));
      }
      __syncwarp();
      // keep at most 6 commits outstanding (ring of 8 barriers), like a 6-stage ring
      const int c = (g + 1) / cevery - 1;
      if ((g + 1) % cevery == 0 && c >= 6) {
        const int w = c - 6;
        wait_bar(&bar[w & 7], (w >> 3) & 1);
      }
    }
    for (int w = ncommit - 6 < 0 ? 0 : ncommit - 6; w < ncommit; ++w) wait_bar(&bar[w & 7], (w >> 3) & 1);
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int N, int PER, int NACC>
void run(int cevery) {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<N, PER, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int groups = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    k<N, PER, NACC><<<148, 64, 160 * 1024>>>(groups, cevery, d);
    cudaDeviceSynchronize();
  }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("N=%3d acc=%d mma/group=%d commit every %d groups: %6.1f clk per MMA, %7.1f per group (floor %d/MMA), err=%s\n",
         N, NACC, PER, cevery, avg / (groups * PER), avg / groups, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, 4, 1>(1); run<64, 4, 2>(1); run<64, 4, 4>(1);
  run<128, 4, 1>(1); run<128, 4, 2>(1); run<128, 4, 4>(1);
  run<256, 4, 1>(1); run<256, 4, 2>(1);
  run<128, 8, 2>(1); run<128, 8, 4>(1); run<64, 8, 4>(1); run<64, 8, 8>(1);
  run<128, 4, 2>(2); run<64, 4, 4>(2);
  return 0;
}
