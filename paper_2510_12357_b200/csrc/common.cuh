// Shared device helpers for the MoBiLE sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/mobile.h"

namespace mobile {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- error state
void set_error(const char* fmt, ...);
int sm_count();
int set_smem_once(const void* func, size_t smem);
int cuda_status(cudaError_t e, const char* where);
#define MOBILE_CHECK_LAUNCH(name) \
  do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return ::mobile::cuda_status(_e, name); } while (0)

// ---------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// ---------------------------------------------------------------- ordering keys
// Monotone map float -> uint32 (larger float -> larger key).  -0.0 is
// canonicalised to +0.0 so the two tie (numpy compares them equal and the
// stable argsort then orders by index, toymoe.py:87).
__device__ __forceinline__ uint32_t order_key_f32(float v) {
  uint32_t b = __float_as_uint(v == 0.0f ? 0.0f : v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t order_key_f64(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v == 0.0 ? 0.0 : v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
// (value desc, index asc) packed: max key wins; ties -> lower index.
__device__ __forceinline__ unsigned long long topk_key(float v, int idx) {
  return ((unsigned long long)order_key_f32(v) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)idx);
}
__device__ __forceinline__ int topk_key_index(unsigned long long k) {
  return (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// Vector of weights: 16 bytes = 8 bf16 or 4 f32, widened to f32.
template <typename W> struct WVec;
template <> struct WVec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static float elem(const uint4& u, int q) {  // q compile-time after unrolling
    const uint32_t w = q < 2 ? u.x : q < 4 ? u.y : q < 6 ? u.z : u.w;
    return (q & 1) ? bf16hi(w) : bf16lo(w);
  }
  __device__ __forceinline__ static void widen(const uint4& u, float* f) {
    f[0] = bf16lo(u.x); f[1] = bf16hi(u.x); f[2] = bf16lo(u.y); f[3] = bf16hi(u.y);
    f[4] = bf16lo(u.z); f[5] = bf16hi(u.z); f[6] = bf16lo(u.w); f[7] = bf16hi(u.w);
  }
};
template <> struct WVec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static float elem(const uint4& u, int q) {
    return __uint_as_float(q == 0 ? u.x : q == 1 ? u.y : q == 2 ? u.z : u.w);
  }
  __device__ __forceinline__ static void widen(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: every decode-path kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, lets its successor be
// scheduled early (launch_dependents) and waits for its predecessor's results
// (griddepcontrol.wait) only right before it reads them.  Reads of static
// data (weights) may be issued before the wait; global writes never are.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster_x,
               const char* name, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) return cuda_status(e, name);
  return MOBILE_OK;
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }
__device__ __forceinline__ float sigmoid_f(float g) { return 1.0f / (1.0f + expf(-g)); }

}  // namespace mobile
