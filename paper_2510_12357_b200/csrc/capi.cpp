// Error state and version for the C ABI (include/mobile.h).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

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

}  // namespace mobile

extern "C" int mobile_version(void) { return 1; }
extern "C" const char* mobile_last_error(void) { return mobile::g_err; }
