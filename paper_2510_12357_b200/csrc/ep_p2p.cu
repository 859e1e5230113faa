// Expert-parallel token exchange over peer memory (NVLink P2P on an NVSwitch
// node; CUDA IPC maps every rank's mailbox into every other rank's process).
//
// The NCCL path (ep.py EPExchange) needs host round trips for the counts and
// four all-to-alls per layer.  Here the home rank's dispatch kernel stores
// each pair's activation row straight into the owner's mailbox, the owner's
// return kernel stores the expert outputs straight back, and release/acquire
// flags at system scope (one per (source, direction), tagged with the
// exchange's epoch) replace the collectives -- no host sync, no counts
// all-to-all, every transfer overlaps with nothing but its own kernel.
//
// Mailbox of one rank (G sources, cap rows per source, d features):
//   in_rows  [G][cap][d] f32   rows dispatched to this rank by source g
//   in_ids   [G][cap]    i32   owner-local expert id of each row
//   in_count [G]         i32
//   in_flag  [G]         u32   epoch of the source's last completed dispatch
//   back_rows[G][cap][d] f32   expert outputs returned to this rank by owner g
//   back_flag[G]         u32
// Semantics are those of ep.py: pairs go to their owner in
// pair order (stable), each output row returns to its pair on the home rank,
// where the combine runs in selection order -- bit-identical to one GPU.
#include <cstring>

#include "common.cuh"

namespace mobile {
namespace ep {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kPlanThreads = 1024;
constexpr unsigned long long kWaitNs = 10000000000ull;  // 10 s: a lost peer traps instead of hanging

struct Box {  // byte offsets inside a mailbox
  size_t in_rows, in_ids, in_count, in_flag, back_rows, back_flag, total;
};

__host__ __device__ inline Box layout(int G, int cap, int d) {
  Box b{};
  const size_t rows = (size_t)G * cap * d * sizeof(float);
  size_t o = 0;
  b.in_rows = o;   o += (rows + 255) / 256 * 256;
  b.in_ids = o;    o += ((size_t)G * cap * 4 + 255) / 256 * 256;
  b.in_count = o;  o += 256;
  b.in_flag = o;   o += 256;
  b.back_rows = o; o += (rows + 255) / 256 * 256;
  b.back_flag = o; o += 256;
  b.total = o;
  return b;
}

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 1. destinations and stable positions: pair p (token p / k_max, slot p % k_max)
//    -> dest_pos[p] = owner * cap + (#earlier pairs to the same owner), or -1.
__global__ void __launch_bounds__(kPlanThreads) ep_plan_kernel(const int* __restrict__ idx, const int* __restrict__ k_tok,
                                                               int P, int k_max, const int* __restrict__ owner, int G,
                                                               int cap, int* __restrict__ dest_pos, int* __restrict__ counts,
                                                               int* __restrict__ flags) {
  __shared__ int wsum[kPlanThreads / 32][8];
  __shared__ int run[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();
  if (tid < 8) run[tid] = 0;
  __syncthreads();
  for (int p0 = 0; p0 < P; p0 += kPlanThreads) {
    const int p = p0 + tid;
    int dst = -1;
    if (p < P) {
      const int t = p / k_max, j = p - t * k_max;
      const int e = idx[p];
      if (j < k_tok[t] && e >= 0) dst = owner[e];
    }
    int below[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const unsigned m = __ballot_sync(0xffffffffu, g < G && dst == g);
      below[g] = __popc(m & ((1u << lane) - 1u));
      if (lane == 0) wsum[warp][g] = __popc(m);
    }
    __syncthreads();
    if (dst >= 0) {
      int pos = run[dst] + below[dst];
      for (int w = 0; w < warp; ++w) pos += wsum[w][dst];
      if (pos >= cap) { atomicOr(flags, 1); dest_pos[p] = -1; }
      else dest_pos[p] = dst * cap + pos;
    } else if (p < P) {
      dest_pos[p] = -1;
    }
    __syncthreads();
    if (tid < G) {
      int s = 0;
      for (int w = 0; w < kPlanThreads / 32; ++w) s += wsum[w][tid];
      run[tid] += s;
    }
    __syncthreads();
  }
  if (tid < G) counts[tid] = min(run[tid], cap);
}

// 2. rows -> the owners' mailboxes (peer stores), one CTA per pair
__global__ void ep_send_kernel(const float* __restrict__ rows, const int* __restrict__ idx, const int* __restrict__ dest_pos,
                               int P, int k_max, int d, const int* __restrict__ local_id, void* const* __restrict__ peers,
                               int rank, int G, int cap, int rows_bf16) {
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.x;
  if (p >= P) return;
  const int dp = dest_pos[p];
  if (dp < 0) return;
  const int g = dp / cap, pos = dp - g * cap;
  const Box b = layout(G, cap, d);
  char* box = reinterpret_cast<char*>(peers[g]);
  const float* src = rows + (size_t)(p / k_max) * d;
  if (rows_bf16) {  // the owner's tensor-core experts consume bf16 rows: half the link bytes
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(box + b.in_rows) + ((size_t)rank * cap + pos) * d;
    for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2)
      *reinterpret_cast<__nv_bfloat162*>(dst + i) = __floats2bfloat162_rn(src[i], src[i + 1]);
    if (threadIdx.x == 0) reinterpret_cast<int*>(box + b.in_ids)[(size_t)rank * cap + pos] = local_id[idx[p]];
    __threadfence_system();
    return;
  }
  float* dst = reinterpret_cast<float*>(box + b.in_rows) + ((size_t)rank * cap + pos) * d;
  if ((d & 3) == 0) {
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x)
      reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
  }
  if (threadIdx.x == 0) reinterpret_cast<int*>(box + b.in_ids)[(size_t)rank * cap + pos] = local_id[idx[p]];
  __threadfence_system();
}

// 3. counts, then the epoch flag, into every owner's mailbox
__global__ void ep_post_kernel(const int* __restrict__ counts, void* const* __restrict__ peers, int rank, int G, int cap,
                               int d, unsigned epoch, const unsigned* epoch_dev) {
  pdl_trigger();
  pdl_wait();
  if (epoch_dev) epoch += *epoch_dev;
  const int g = threadIdx.x;
  if (g >= G) return;
  const Box b = layout(G, cap, d);
  char* box = reinterpret_cast<char*>(peers[g]);
  reinterpret_cast<int*>(box + b.in_count)[rank] = counts[g];
  __threadfence_system();
  st_release_sys_u32(reinterpret_cast<unsigned*>(box + b.in_flag) + rank, epoch);
}

// 4. wait until every source posted this epoch; owner side also derives the
//    per-row validity (k_tok = 1 for rows below the source's count)
__global__ void ep_wait_kernel(void* mailbox, int G, int cap, int d, int which, unsigned epoch, int* k_tok_out,
                               int* flags, const unsigned* epoch_dev) {
  pdl_trigger();
  pdl_wait();
  if (epoch_dev) epoch += *epoch_dev;
  const Box b = layout(G, cap, d);
  char* box = reinterpret_cast<char*>(mailbox);
  const unsigned* fl = reinterpret_cast<const unsigned*>(box + (which == 0 ? b.in_flag : b.back_flag));
  __shared__ int counts[64];
  if (threadIdx.x < G) {
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys_u32(fl + threadIdx.x) != epoch) {
      __nanosleep(100);
      if (gtimer() - t0 > kWaitNs) {
        atomicOr(flags, 2);
        __trap();
      }
    }
    counts[threadIdx.x] = which == 0 ? reinterpret_cast<const volatile int*>(box + b.in_count)[threadIdx.x] : 0;
  }
  __syncthreads();
  if (which == 0 && k_tok_out)
    for (int i = threadIdx.x; i < G * cap; i += blockDim.x) k_tok_out[i] = (i % cap) < counts[i / cap] ? 1 : 0;
}

// 5. owner: expert outputs of source s's rows -> s's back mailbox, one CTA per row
__global__ void ep_return_kernel(const float* __restrict__ out_rows, const void* mailbox, void* const* __restrict__ peers,
                                 int rank, int G, int cap, int d) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int s = r / cap, i = r - s * cap;
  const Box b = layout(G, cap, d);
  const int n = reinterpret_cast<const volatile int*>(reinterpret_cast<const char*>(mailbox) + b.in_count)[s];
  if (i >= n) return;
  float* dst = reinterpret_cast<float*>(reinterpret_cast<char*>(peers[s]) + b.back_rows) + ((size_t)rank * cap + i) * d;
  const float* src = out_rows + (size_t)r * d;
  if ((d & 3) == 0) {
    for (int q = threadIdx.x; q < d / 4; q += blockDim.x)
      reinterpret_cast<float4*>(dst)[q] = reinterpret_cast<const float4*>(src)[q];
  } else {
    for (int q = threadIdx.x; q < d; q += blockDim.x) dst[q] = src[q];
  }
  __threadfence_system();
}

__global__ void ep_post_back_kernel(void* const* __restrict__ peers, int rank, int G, int cap, int d, unsigned epoch,
                                    const unsigned* epoch_dev) {
  pdl_trigger();
  pdl_wait();
  if (epoch_dev) epoch += *epoch_dev;
  const int s = threadIdx.x;
  if (s >= G) return;
  const Box b = layout(G, cap, d);
  __threadfence_system();
  st_release_sys_u32(reinterpret_cast<unsigned*>(reinterpret_cast<char*>(peers[s]) + b.back_flag) + rank, epoch);
}

// graph-replayable exchanges: the epoch lives in device memory, advanced by
// one kernel at the start of every exchange (ranks advance in lockstep: every
// rank runs every exchange)
__global__ void ep_advance_kernel(unsigned* epoch_dev) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) *epoch_dev += 1u;
}

// 6. home: Y[p] = the owner's output row of pair p (zero for unselected slots)
__global__ void ep_collect_kernel(const void* mailbox, const int* __restrict__ dest_pos, int P, int G, int cap, int d,
                                  float* __restrict__ Y) {
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.x;
  const int dp = dest_pos[p];
  const Box b = layout(G, cap, d);
  float* dst = Y + (size_t)p * d;
  if (dp < 0) {
    for (int q = threadIdx.x; q < d; q += blockDim.x) dst[q] = 0.f;
    return;
  }
  const float* src = reinterpret_cast<const float*>(reinterpret_cast<const char*>(mailbox) + b.back_rows) + (size_t)dp * d;
  for (int q = threadIdx.x; q < d; q += blockDim.x) dst[q] = __ldcv(src + q);
}

}  // namespace ep
}  // namespace mobile

using namespace mobile;
using namespace mobile::ep;

extern "C" size_t mobile_ep_mailbox_bytes(int G, int cap, int d) { return layout(G, cap, d).total; }

extern "C" int mobile_ep_mailbox_create(int G, int cap, int d, void** mailbox) {
  if (G < 1 || G > 8 || cap < 1 || d < 1 || !mailbox) { set_error("ep mailbox: bad shape G=%d cap=%d d=%d (G <= 8)", G, cap, d); return MOBILE_ERR_INVALID; }
  const size_t n = layout(G, cap, d).total;
  void* p = nullptr;
  if (cudaMalloc(&p, n) != cudaSuccess) { set_error("ep mailbox: cudaMalloc(%zu) failed", n); return MOBILE_ERR_CUDA; }
  if (cudaMemset(p, 0, n) != cudaSuccess) { cudaFree(p); set_error("ep mailbox: memset failed"); return MOBILE_ERR_CUDA; }
  *mailbox = p;
  return MOBILE_OK;
}

extern "C" int mobile_ep_mailbox_destroy(void* mailbox) {
  if (mailbox) cudaFree(mailbox);
  return MOBILE_OK;
}

extern "C" int mobile_ep_ipc_handle(void* mailbox, void* handle64) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, mailbox) != cudaSuccess) { set_error("ep: cudaIpcGetMemHandle failed"); return MOBILE_ERR_CUDA; }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle64, &h, 64);
  return MOBILE_OK;
}

extern "C" int mobile_ep_ipc_open(const void* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    set_error("ep: cudaIpcOpenMemHandle failed");
    return MOBILE_ERR_CUDA;
  }
  return MOBILE_OK;
}

extern "C" int mobile_ep_ipc_close(void* ptr) {
  cudaIpcCloseMemHandle(ptr);
  return MOBILE_OK;
}

extern "C" int mobile_ep_dispatch(const float* rows, const int* idx, const int* k_tok, int T, int k_max, int d,
                                  const int* owner, const int* local_id, void* const* peers_dev, int G, int rank, int cap,
                                  unsigned epoch, const unsigned* epoch_dev, int rows_bf16, int* dest_pos, int* counts,
                                  int* flags, void* stream) {
  if (T < 0 || k_max < 1 || d < 1 || G < 1 || G > 8 || rank < 0 || rank >= G || cap < 1) {
    set_error("ep_dispatch: bad arguments");
    return MOBILE_ERR_INVALID;
  }
  if (rows_bf16 && (d & 1)) { set_error("ep_dispatch: bf16 rows need an even d"); return MOBILE_ERR_UNSUPPORTED; }
  cudaStream_t s = (cudaStream_t)stream;
  const int P = T * k_max;
  if (int st = launch_pdl(ep_plan_kernel, dim3(1), dim3(kPlanThreads), 0, s, 1, "ep_plan", idx, k_tok, P, k_max, owner, G,
                          cap, dest_pos, counts, flags)) return st;
  if (P > 0)
    if (int st = launch_pdl(ep_send_kernel, dim3(P), dim3(128), 0, s, 1, "ep_send", rows, idx, dest_pos, P, k_max, d,
                            local_id, peers_dev, rank, G, cap, rows_bf16)) return st;
  return launch_pdl(ep_post_kernel, dim3(1), dim3(32), 0, s, 1, "ep_post", counts, peers_dev, rank, G, cap, d, epoch,
                    epoch_dev);
}

extern "C" int mobile_ep_wait(void* mailbox, int G, int cap, int d, int which, unsigned epoch, const unsigned* epoch_dev,
                              int* k_tok_out, int* flags, void* stream) {
  if (G < 1 || G > 8 || (which != 0 && which != 1)) { set_error("ep_wait: bad arguments"); return MOBILE_ERR_INVALID; }
  return launch_pdl(ep_wait_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, 1, "ep_wait", mailbox, G, cap, d, which,
                    epoch, k_tok_out, flags, epoch_dev);
}

extern "C" int mobile_ep_return(const float* out_rows, const void* mailbox, void* const* peers_dev, int G, int rank, int cap,
                                int d, unsigned epoch, const unsigned* epoch_dev, void* stream) {
  if (G < 1 || G > 8 || rank < 0 || rank >= G) { set_error("ep_return: bad arguments"); return MOBILE_ERR_INVALID; }
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = launch_pdl(ep_return_kernel, dim3(G * cap), dim3(128), 0, s, 1, "ep_return", out_rows, mailbox, peers_dev,
                          rank, G, cap, d)) return st;
  return launch_pdl(ep_post_back_kernel, dim3(1), dim3(32), 0, s, 1, "ep_post_back", peers_dev, rank, G, cap, d, epoch,
                    epoch_dev);
}

extern "C" int mobile_ep_advance(unsigned* epoch_dev, void* stream) {
  if (!epoch_dev) { set_error("ep_advance: null epoch"); return MOBILE_ERR_INVALID; }
  return launch_pdl(ep_advance_kernel, dim3(1), dim3(32), 0, (cudaStream_t)stream, 1, "ep_advance", epoch_dev);
}

extern "C" int mobile_ep_collect(const void* mailbox, const int* dest_pos, int P, int G, int cap, int d, float* Y,
                                 void* stream) {
  if (P <= 0) return MOBILE_OK;
  return launch_pdl(ep_collect_kernel, dim3(P), dim3(128), 0, (cudaStream_t)stream, 1, "ep_collect", mailbox, dest_pos, P,
                    G, cap, d, Y);
}
