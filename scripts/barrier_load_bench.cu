// Grid-barrier latency on B200 under concurrent bulk-copy HBM streaming from
// the same SMs (the persistent decode pass's situation), as a function of the
// bytes each SM keeps in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_load_bench barrier_load_bench.cu
// One CTA per SM: lane 0 of warp 1 streams `tile`-byte cp.async.bulk copies
// keeping `nfl` of them in flight (ring of 8 stages); thread 0 runs N grid
// barriers (red.release + relaxed poll + fence.acq_rel, the decode pass's
// flavour) and, separately, N bare relaxed round trips.  Prints ns per
// barrier and the streamed GB/s over the same window.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

__global__ void __launch_bounds__(64, 1) k(unsigned* cnt, int n, const char* src, size_t src_bytes, int tile, int nfl,
                                           int mode, volatile int* stop, unsigned long long* out,
                                           unsigned long long* bytes, unsigned* data, unsigned* bad) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    if (nfl == 0 || lane) return;
    size_t off = (size_t)blockIdx.x * tile;
    uint32_t it = 0;
    unsigned long long done = 0;
    while (!*stop) {
      const int R = tile >= 65536 ? 3 : (tile == 32768 ? 6 : 8);
      const int s = it % R;
      if (it >= (uint32_t)nfl) {  // wait for the copy issued nfl items ago
        const int so = (it - nfl) % R;
        const uint32_t par = ((it - nfl) / R) & 1u;
        uint32_t ok = 0;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(ok) : "r"(su32(&full[so])), "r"(par) : "memory");
        done += tile;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"((unsigned)tile) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(smem + (size_t)s * tile)), "l"(src + off), "r"((unsigned)tile), "r"(su32(&full[s])) : "memory");
      off += (size_t)gridDim.x * tile;
      if (off + tile > src_bytes) off = (size_t)blockIdx.x * tile;
      ++it;
    }
    atomicAdd(bytes, done);
    return;
  }
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gtimer();
  while (gtimer() - t0 < 50000) {}
  unsigned long long tb = 0;
  unsigned nbad = 0;
  for (int i = 1; i <= n; ++i) {
    const unsigned target = (unsigned)i * gridDim.x;
    if (i == 2) tb = gtimer();
    // this CTA's "phase output": 4 words on distinct lines
    for (int w = 0; w < 4; ++w) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(data + (blockIdx.x * 4 + w) * 32), "r"((unsigned)i) : "memory");
    if (mode == 0) {  // the decode pass: red.release + relaxed poll + fence.acq_rel
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) __nanosleep(64);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    } else if (mode == 1) {  // no ordering at all (not a valid barrier): the raw round trip
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
    } else if (mode == 2) {  // red.release, relaxed poll, no acquire fence
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
    } else if (mode == 3) {  // relaxed red, ld.acquire poll
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    } else if (mode == 4) {  // fence.release (PTX 8.6) + relaxed red, relaxed poll + fence.acquire
      asm volatile("fence.release.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
      asm volatile("fence.acquire.gpu;" ::: "memory");
    } else if (mode == 5) {  // fence.release alone + relaxed barrier
      asm volatile("fence.release.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
    } else if (mode == 6) {  // relaxed barrier + fence.acquire alone
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
      asm volatile("fence.acquire.gpu;" ::: "memory");
    } else if (mode == 7) {  // __threadfence() + relaxed barrier
      __threadfence();
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while (ld_relaxed(cnt) < target) {}
    } else if (mode == 8) {  // fence.acq_rel.cluster + relaxed red, acquire poll
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    } else if (mode == 9) {  // read back own stores from L2, dependent relaxed red, acquire poll
      unsigned acc = 0;
      for (int w = 0; w < 4; ++w) acc += ld_relaxed(data + (blockIdx.x * 4 + w) * 32);
      const unsigned inc = 1u + (acc == 0xffffffffu ? 1u : 0u);  // data dependency on the read-backs
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(cnt), "r"(inc) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    } else if (mode == 10) {  // red.release.cta + acquire poll
      asm volatile("red.release.cta.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    } else if (mode == 11) {  // no release at all, acquire poll (the negative control)
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    }
    // check the other CTAs' outputs of this round
    for (int w = 0; w < 4; ++w) {
      const unsigned o = (blockIdx.x * 37 + w * 53 + i) % gridDim.x;
      if (ld_relaxed(data + (o * 4 + w) * 32) < (unsigned)i) ++nbad;
    }
  }
  atomicAdd(bad, nbad);
  if (blockIdx.x == 0) {
    out[0] = (gtimer() - tb) / (n - 1);
    out[1] = gtimer() - t0;
    __threadfence_system();
  }
}

int main() {
  unsigned* cnt;
  char* src;
  unsigned long long* bytes;
  const size_t SB = (size_t)4 << 30;
  cudaMalloc(&cnt, 4); cudaMalloc(&src, SB); cudaMemset(src, 1, SB); cudaMalloc(&bytes, 8);
  unsigned *data, *bad; cudaMalloc(&data, 148 * 4 * 128); cudaMalloc(&bad, 4);
  int* h_stop; unsigned long long* h_out;
  cudaHostAlloc(&h_stop, 4, cudaHostAllocMapped); cudaHostAlloc(&h_out, 16, cudaHostAllocMapped);
  int* stop; unsigned long long* out;
  cudaHostGetDevicePointer((void**)&stop, h_stop, 0); cudaHostGetDevicePointer((void**)&out, h_out, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 * 1 + 0);
  const int tiles[] = {65536, 65536, 65536};
  const int nfls[] = {0, 1, 3, 9, 9, 9};
  for (int mode = 0; mode < 12; ++mode)
    for (int ti = 0; ti < 1; ++ti)
      for (int fi = 0; fi < 3; ++fi) {
        const int tile = tiles[ti], nfl = nfls[fi];
                const int smem = tile * (tile == 65536 ? 3 : (tile == 32768 ? 6 : 8));
        if (nfl > (tile == 65536 ? 3 : (tile == 32768 ? 6 : 8))) continue;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaMemset(cnt, 0, 4); cudaMemset(bytes, 0, 8); cudaMemset(data, 0, 148 * 4 * 128); cudaMemset(bad, 0, 4);
        h_out[0] = 0; h_out[1] = 0;
        *(volatile int*)h_stop = 0;
        cudaDeviceSynchronize();
        // the ring index wraps at 8 stages: with 64 KB tiles only 3 fit, so nfl <= 3 and stages s % 8 < 3 ... use tile*8 smem
        k<<<148, 64, smem>>>(cnt, 2000, src, SB, tile, nfl, mode, stop, out, bytes, data, bad);
        volatile unsigned long long* hp = h_out;
        while (hp[0] == 0) {}
        unsigned long long ns = hp[0], win = hp[1];
        *(volatile int*)h_stop = 1;
        cudaDeviceSynchronize();
        unsigned long long b = 0;
        cudaMemcpy(&b, bytes, 8, cudaMemcpyDeviceToHost);
        unsigned nb = 0;
        cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost);
        printf("mode %2d inflight %d x 64 KB: %7llu ns/barrier, stale reads %u  %s\n", mode, nfl, ns, nb,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
