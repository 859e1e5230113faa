// H2D expert-copy probe: per-copy overhead of cudaMemcpyAsync for 17.3 MB
// experts, multi-stream copies, and SM-driven zero-copy pulls.
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>

__global__ void pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  const size_t eb = 17301504;  // Qwen expert bytes
  const int n = 48;
  char* h;
  cudaHostAlloc(&h, eb * n, cudaHostAllocDefault);
  for (size_t i = 0; i < eb * n; i += 4096) h[i] = 1;
  char* d;
  cudaMalloc(&d, eb * n);
  cudaStream_t st[4];
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ns : {1, 2, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, st[0]);
      for (int i = 0; i < ns; ++i) cudaStreamWaitEvent(st[i], e0, 0);
      for (int i = 0; i < n; ++i) cudaMemcpyAsync(d + i * eb, h + i * eb, eb, cudaMemcpyHostToDevice, st[i % ns]);
      for (int i = 1; i < ns; ++i) { cudaEvent_t ev; cudaEventCreate(&ev); cudaEventRecord(ev, st[i]); cudaStreamWaitEvent(st[0], ev, 0); }
      cudaEventRecord(e1, st[0]);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("memcpy streams=%d : %.1f GB/s  (%.1f us per expert)\n", ns, eb * n / (ms / 1e3) / 1e9, ms * 1e3 / n);
    }
  }
  // single large copy for reference
  cudaEventRecord(e0, st[0]);
  cudaMemcpyAsync(d, h, eb * n, cudaMemcpyHostToDevice, st[0]);
  cudaEventRecord(e1, st[0]);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("memcpy one %zu MB : %.1f GB/s\n", eb * n >> 20, eb * n / (ms / 1e3) / 1e9);
  // zero-copy pull kernels
  char* hp;
  cudaHostGetDevicePointer(&hp, h, 0);
  for (int blocks : {16, 32, 64, 148, 296}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, st[0]);
      for (int i = 0; i < n; ++i) pull<<<blocks, 512, 0, st[0]>>>((const uint4*)(hp + i * eb), (uint4*)(d + i * eb), eb / 16);
      cudaEventRecord(e1, st[0]);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("pull kernel blocks=%d : %.1f GB/s (%.1f us per expert)\n", blocks, eb * n / (ms / 1e3) / 1e9, ms * 1e3 / n);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
