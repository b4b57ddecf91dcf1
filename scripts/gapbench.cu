// Kernel-to-kernel gap micro-benchmark (diagnostic, not part of the library).
// Launches variants of an empty persistent kernel back to back inside a CUDA
// graph and reports ms per launch: plain, + 200 KB dynamic smem, + TMEM
// alloc/dealloc, + 1.6 KB of parameters, + 416 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gapbench scripts/gapbench.cu
#include <cuda_runtime.h>

#include <cstdio>

struct Big {
  char b[1600];
};

template <bool TMEM>
__global__ void k_empty(Big p, unsigned long long* t) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned slot;
  if (p.b[1] == 1) {  // PDL variant
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (TMEM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&slot))));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
  }
  if (threadIdx.x == 0 && p.b[0] == 1) t[blockIdx.x] = sm[0];
}

int main() {
  unsigned long long* t;
  cudaMalloc(&t, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  Big p{};
  const int smem_big = 200 * 1024;
  cudaFuncSetAttribute(k_empty<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  cudaFuncSetAttribute(k_empty<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  struct V {
    const char* name;
    bool tmem;
    int smem, threads;
    bool pdl;
  } vs[] = {{"empty 128 thr", false, 0, 128, false},
            {"empty 416 thr", false, 0, 416, false},
            {"+200KB smem", false, smem_big, 416, false},
            {"+TMEM alloc", true, smem_big, 416, false},
            {"TMEM no smem", true, 0, 416, false},
            {"PDL empty 128", false, 0, 128, true},
            {"PDL +200KB+TMEM", true, smem_big, 416, true},
            {"PDL 200KB+TMEM 384", true, smem_big, 384, true}};
  for (auto& v : vs) {
    const int n = 50;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    p.b[1] = v.pdl ? 1 : 0;
    for (int i = 0; i < n; ++i) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(v.threads);
      cfg.dynamicSmemBytes = v.smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = v.pdl ? 1 : 0;
      if (v.tmem) cudaLaunchKernelEx(&cfg, k_empty<true>, p, t);
      else cudaLaunchKernelEx(&cfg, k_empty<false>, p, t);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-16s %.2f us/launch (%s)\n", v.name, ms * 1e3f / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
