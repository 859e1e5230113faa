// Grid-barrier latency on B200: 148 persistent CTAs x N barriers, several
// arrival / polling flavours.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void bar_kernel(unsigned* cnt, int n, float* sink) {
  __shared__ float s[256];
  s[threadIdx.x] = threadIdx.x;
  for (int i = 1; i <= n; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)i * gridDim.x;
      if (MODE == 0) {  // fence + atomicAdd, acquire polling
        __threadfence();
        atomicAdd(cnt, 1u);
        while (ld_acquire(cnt) < target) {}
      } else if (MODE == 1) {  // red.release, relaxed polling + fence
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        while (ld_relaxed(cnt) < target) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (MODE == 2) {  // atom.add.release returns old; relaxed polling
        unsigned old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        if (old + 1 < target) while (ld_relaxed(cnt) < target) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {  // polling with nanosleep
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        while (ld_relaxed(cnt) < target) __nanosleep(64);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (s[threadIdx.x] == -1.f) sink[0] = 1.f;
}

int main() {
  unsigned* cnt;
  float* sink;
  cudaMalloc(&cnt, 4);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n = 2000;
  auto run = [&](auto kern, const char* name, int threads) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cnt, 0, 4);
      cudaEventRecord(a);
      kern<<<sms, threads>>>(cnt, n, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%-40s threads=%d : %.3f us / barrier\n", name, threads, ms * 1e3 / n);
    }
  };
  run(bar_kernel<0>, "fence+atomicAdd, ld.acquire poll", 256);
  run(bar_kernel<1>, "red.release, ld.relaxed poll + fence", 256);
  run(bar_kernel<2>, "atom.release (skip poll if last)", 256);
  run(bar_kernel<3>, "red.release, poll + nanosleep(64)", 256);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
