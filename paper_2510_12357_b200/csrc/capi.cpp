// Error state and version for the C ABI (include/mobile.h).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/mobile.h"

namespace mobile {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
  return MOBILE_ERR_CUDA;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel (and only
// when the requested size grows), so launches stay legal inside CUDA-graph
// capture and cost nothing on the hot path.
int set_smem_once(const void* func, size_t smem) {
  if (smem <= 48 * 1024) return MOBILE_OK;
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[func];
  if (smem <= cur) return MOBILE_OK;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
  cur = smem;
  return MOBILE_OK;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MOBILE_PDL");
    v = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

}  // namespace mobile

extern "C" int mobile_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return mobile::cuda_status(e, "memcpy_async");
  return MOBILE_OK;
}

extern "C" int mobile_version(void) { return 1; }
extern "C" const char* mobile_last_error(void) { return mobile::g_err; }
