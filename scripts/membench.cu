// Streaming-read microbenchmark on B200: what does it take to reach HBM
// bandwidth with (a) cp.async.bulk + mbarrier pipelines and (b) LDG.128?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

// one thread per CTA issues; all threads wait + do a trivial read of the stage
__global__ void tma_stream(const char* src, size_t bytes, int stages, int stage_bytes, int copies_per_stage, float* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full[16];
  const size_t nitems = bytes / stage_bytes;
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const size_t first = blockIdx.x, step = gridDim.x;
  float acc = 0.f;
  const uint32_t cb = stage_bytes / copies_per_stage;
  if (threadIdx.x == 0) {
    size_t it = first;
    for (int s = 0; s < stages && it < nitems; ++s, it += step) {
      mbar_expect_tx(&full[s], stage_bytes);
      for (int c = 0; c < copies_per_stage; ++c) bulk(sm + (size_t)s * stage_bytes + c * cb, src + it * stage_bytes + c * cb, cb, &full[s]);
    }
  }
  uint32_t ph = 0;
  int s = 0;
  size_t issue = first + (size_t)stages * step;
  for (size_t it = first; it < nitems; it += step) {
    mbar_wait(&full[s], (ph >> s) & 1);
    ph ^= 1u << s;
    acc += reinterpret_cast<const float*>(sm + (size_t)s * stage_bytes)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && issue < nitems) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[s], stage_bytes);
      for (int c = 0; c < copies_per_stage; ++c) bulk(sm + (size_t)s * stage_bytes + c * cb, src + issue * stage_bytes + c * cb, cb, &full[s]);
    }
    issue += step;
    s = s + 1 == stages ? 0 : s + 1;
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int U>
__global__ void ldg_stream(const uint4* src, size_t n, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x ^ v[u].w);
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  char* buf;
  float* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 3.0 * bytes / (ms / 1e3) / 1e9;
  };
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int cfgs[][4] = {{3, 65536, 1, 1}, {3, 65536, 16, 1}, {6, 32768, 1, 1}, {12, 16384, 1, 1}, {4, 49152, 1, 1},
                   {2, 65536, 1, 2}, {3, 32768, 1, 2}, {6, 16384, 1, 2}, {4, 16384, 1, 3}, {6, 8192, 1, 4},
                   {3, 65536, 4, 1}, {8, 24576, 1, 1}, {2, 32768, 1, 3}, {3, 16384, 1, 4}, {13, 16384, 1, 1}, {26, 8192, 1, 1}};
  for (auto& c : cfgs) {
    int stages = c[0], sb = c[1], cps = c[2], per_sm = c[3];
    if ((size_t)stages * sb * per_sm > 220 * 1024) continue;
    double gbs = timeit([&] { tma_stream<<<sms * per_sm, 128, (size_t)stages * sb>>>(buf, bytes, stages, sb, cps, sink); });
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(le)); continue; }
    printf("tma stages=%2d stage=%6d copies/stage=%2d ctas/sm=%d : %7.1f GB/s\n", stages, sb, cps, per_sm, gbs);
  }
  for (int threads : {256, 512, 1024}) {
    for (int bpsm : {1, 2, 4}) {
      double g4 = timeit([&] { ldg_stream<4><<<sms * bpsm, threads>>>((const uint4*)buf, bytes / 16, sink); });
      double g8 = timeit([&] { ldg_stream<8><<<sms * bpsm, threads>>>((const uint4*)buf, bytes / 16, sink); });
      printf("ldg threads=%4d blocks/sm=%d : U4 %7.1f GB/s  U8 %7.1f GB/s\n", threads, bpsm, g4, g8);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
