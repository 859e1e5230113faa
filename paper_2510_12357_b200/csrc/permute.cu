// Deterministic token permute (counting sort of (token, slot) pairs by expert)
// and the weighted combine.  Replaces the implicit per-position loop of
// toymoe.py:193-204 and the accumulation/residual of toymoe.py:192, 204, 207.
#include "common.cuh"

namespace mobile {

constexpr int kPermThreads = 1024;
constexpr int kPermWarps = kPermThreads / 32;
constexpr int kPermMaxE = 256;

// One CTA.  Pass 1 counts pairs per expert; an exclusive scan gives offsets;
// pass 2 places pairs chunk by chunk: within a warp `match.any` ranks equal
// experts by lane, across warps a per-warp count table ranks by warp, across
// chunks a running base.  The order inside every expert list is therefore
// pair order (token-major, then selection slot): stable and deterministic.
__global__ void __launch_bounds__(kPermThreads) permute_kernel(const int* __restrict__ idx,
                                                               const int* __restrict__ k_tok, int T,
                                                               int k_max, int E, int* offsets,
                                                               int* sorted_pairs, int* active) {
  __shared__ int cnt[kPermMaxE];
  __shared__ int base[kPermMaxE];
  __shared__ int wcnt[kPermWarps][kPermMaxE];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();
  const int P = T * k_max;
  for (int e = tid; e < E; e += kPermThreads) cnt[e] = 0;
  for (int i = tid; i < kPermWarps * E; i += kPermThreads) wcnt[i / E][i % E] = 0;
  __syncthreads();
  for (int p = tid; p < P; p += kPermThreads) {
    const int t = p / k_max, j = p - t * k_max;
    const int kt = k_tok ? k_tok[t] : k_max;
    const int e = j < kt ? idx[p] : -1;
    if (e >= 0 && e < E) atomicAdd(&cnt[e], 1);  // integer count: order-free
  }
  __syncthreads();
  if (tid == 0) {
    int run = 0, na = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = run;
      base[e] = run;
      run += cnt[e];
      if (cnt[e] > 0) active[1 + na++] = e;
    }
    offsets[E] = run;
    active[0] = na;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int c = 0; c < P; c += kPermThreads) {
    const int p = c + tid;
    int e = -1;
    if (p < P) {
      const int t = p / k_max, j = p - t * k_max;
      const int kt = k_tok ? k_tok[t] : k_max;
      e = j < kt ? idx[p] : -1;
      if (e >= E) e = -1;
    }
    const unsigned m = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(m & lt);
    if (e >= 0 && rank == 0) wcnt[warp][e] = __popc(m);
    __syncthreads();
    if (e >= 0) {
      int pos = base[e] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][e];
      sorted_pairs[pos] = p;
    }
    __syncthreads();
    for (int e2 = tid; e2 < E; e2 += kPermThreads) {
      int s = 0;
      for (int w = 0; w < kPermWarps; ++w) { s += wcnt[w][e2]; wcnt[w][e2] = 0; }
      base[e2] += s;
    }
    __syncthreads();
  }
}

// x_out[t] = x[t] + (sum_j g[t,j] * Y[t*k+j]  (selection order)
//                    + sum_s gate_s(t) * Ys[t][s])          toymoe.py:204, 207
// and, if ln_out, ln_out[t] = LN(x_out[t]) -- the next layer's attention input
// (toymoe.py:178), fused here because this CTA already holds the whole row.
__global__ void __launch_bounds__(1024) combine_kernel(const float* __restrict__ x, const float* __restrict__ Y,
                                                      const float* __restrict__ gates, const int* __restrict__ k_tok,
                                                      int k_max, int d, const float* __restrict__ Ys, int n_shared,
                                                      const float* __restrict__ shared_logits, int T,
                                                      float* __restrict__ x_out, float* __restrict__ ln_out) {
  __shared__ float red[32];
  __shared__ float sg[16];    // gates (selection order) then shared-expert gates
  const int t = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  const int kt = k_tok ? k_tok[t] : k_max;
  if (threadIdx.x < kt && threadIdx.x < 8) sg[threadIdx.x] = gates[(size_t)t * k_max + threadIdx.x];  // later gates: global
  if (threadIdx.x < n_shared)
    sg[8 + threadIdx.x] = shared_logits ? sigmoid_f(shared_logits[(size_t)t * n_shared + threadIdx.x]) : 1.0f;
  __syncthreads();
  float sum = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    // issue every independent load first, then accumulate in selection order
    float yv[8], ys[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) yv[j] = j < kt ? Y[((size_t)t * k_max + j) * d + i] : 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s) ys[s] = s < n_shared ? Ys[((size_t)t * n_shared + s) * d + i] : 0.f;
    const float xv = x[(size_t)t * d + i];
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) if (j < kt) m = fmaf(sg[j], yv[j], m);
    for (int j = 8; j < kt; ++j) m = fmaf(gates[(size_t)t * k_max + j], Y[((size_t)t * k_max + j) * d + i], m);
#pragma unroll
    for (int s = 0; s < 8; ++s) if (s < n_shared) m += sg[8 + s] * ys[s];
    const float v = xv + m;
    x_out[(size_t)t * d + i] = v;
    sum += v;
  }
  if (!ln_out) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  float mean = 0.f;
  for (int w = 0; w < nw; ++w) mean += red[w];
  mean /= (float)d;
  __syncthreads();
  float q = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float c = x_out[(size_t)t * d + i] - mean;
    q += c * c;
  }
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  float var = 0.f;
  for (int w = 0; w < nw; ++w) var += red[w];
  const float inv = 1.0f / sqrtf(var / (float)d + 1e-5f);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    ln_out[(size_t)t * d + i] = (x_out[(size_t)t * d + i] - mean) * inv;
}

// float4 variant (d % 4 == 0): the same per-element arithmetic and order,
// 256 threads so several tokens' CTAs share an SM (prefill / batched decode)
constexpr int kComb4Threads = 256;
__global__ void __launch_bounds__(kComb4Threads) combine4_kernel(
    const float4* __restrict__ x, const float4* __restrict__ Y, const float* __restrict__ gates,
    const int* __restrict__ k_tok, int k_max, int d4, const float4* __restrict__ Ys, int n_shared,
    const float* __restrict__ shared_logits, float4* __restrict__ x_out, float4* __restrict__ ln_out) {
  __shared__ float red[kComb4Threads / 32];
  __shared__ float sg[16];
  const int t = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  const int kt = k_tok ? k_tok[t] : k_max;
  if (threadIdx.x < kt && threadIdx.x < 8) sg[threadIdx.x] = gates[(size_t)t * k_max + threadIdx.x];
  if (threadIdx.x < n_shared)
    sg[8 + threadIdx.x] = shared_logits ? sigmoid_f(shared_logits[(size_t)t * n_shared + threadIdx.x]) : 1.0f;
  __syncthreads();
  float sum = 0.f;
  for (int i = threadIdx.x; i < d4; i += kComb4Threads) {
    float4 yv[8], ys[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) if (j < kt) yv[j] = Y[((size_t)t * k_max + j) * d4 + i];
#pragma unroll
    for (int s = 0; s < 8; ++s) if (s < n_shared) ys[s] = Ys[((size_t)t * n_shared + s) * d4 + i];
    const float4 xv = x[(size_t)t * d4 + i];
    float m[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < kt) {
        m[0] = fmaf(sg[j], yv[j].x, m[0]); m[1] = fmaf(sg[j], yv[j].y, m[1]);
        m[2] = fmaf(sg[j], yv[j].z, m[2]); m[3] = fmaf(sg[j], yv[j].w, m[3]);
      }
    }
    for (int j = 8; j < kt; ++j) {
      const float g = gates[(size_t)t * k_max + j];
      const float4 y = Y[((size_t)t * k_max + j) * d4 + i];
      m[0] = fmaf(g, y.x, m[0]); m[1] = fmaf(g, y.y, m[1]); m[2] = fmaf(g, y.z, m[2]); m[3] = fmaf(g, y.w, m[3]);
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s < n_shared) {
        const float g = sg[8 + s];
        m[0] += g * ys[s].x; m[1] += g * ys[s].y; m[2] += g * ys[s].z; m[3] += g * ys[s].w;
      }
    }
    const float4 v = make_float4(xv.x + m[0], xv.y + m[1], xv.z + m[2], xv.w + m[3]);
    x_out[(size_t)t * d4 + i] = v;
    sum += (v.x + v.y) + (v.z + v.w);
  }
  if (!ln_out) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kComb4Threads / 32;
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  float mean = 0.f;
#pragma unroll
  for (int w = 0; w < nw; ++w) mean += red[w];
  mean /= (float)(4 * d4);
  __syncthreads();
  float q = 0.f;
  for (int i = threadIdx.x; i < d4; i += kComb4Threads) {
    const float4 v = x_out[(size_t)t * d4 + i];
    const float a = v.x - mean, b = v.y - mean, c = v.z - mean, e = v.w - mean;
    q += (a * a + b * b) + (c * c + e * e);
  }
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  float var = 0.f;
#pragma unroll
  for (int w = 0; w < nw; ++w) var += red[w];
  const float inv = 1.0f / sqrtf(var / (float)(4 * d4) + 1e-5f);
  for (int i = threadIdx.x; i < d4; i += kComb4Threads) {
    const float4 v = x_out[(size_t)t * d4 + i];
    ln_out[(size_t)t * d4 + i] = make_float4((v.x - mean) * inv, (v.y - mean) * inv, (v.z - mean) * inv, (v.w - mean) * inv);
  }
}

}  // namespace mobile

using namespace mobile;

extern "C" int mobile_permute(const int* idx, const int* k_tok, int T, int k_max, int E, int* offsets,
                              int* sorted_pairs, int* active, void* stream) {
  if (T < 0 || k_max <= 0 || E <= 0) { set_error("permute: bad shape T=%d k=%d E=%d", T, k_max, E); return MOBILE_ERR_INVALID; }
  if (E > kPermMaxE) { set_error("permute: E=%d exceeds %d", E, kPermMaxE); return MOBILE_ERR_UNSUPPORTED; }
  return launch_pdl(permute_kernel, dim3(1), dim3(kPermThreads), 0, (cudaStream_t)stream, 1, "permute", idx, k_tok,
                    T, k_max, E, offsets, sorted_pairs, active);
}

extern "C" int mobile_combine(const float* x, const float* Y, const float* gates, const int* k_tok,
                              int T, int k_max, int d, const float* Y_shared, int n_shared,
                              const float* shared_logits, float* x_out, float* ln_out, void* stream) {
  if (T < 0 || d <= 0 || k_max <= 0 || n_shared < 0) { set_error("combine: bad shape"); return MOBILE_ERR_INVALID; }
  if (T == 0) return MOBILE_OK;
  if (n_shared > 8) { set_error("combine: at most 8 shared experts"); return MOBILE_ERR_UNSUPPORTED; }
  const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(x_out) |
                    reinterpret_cast<uintptr_t>(ln_out) | reinterpret_cast<uintptr_t>(Y_shared)) & 15) == 0;
  if (d % 4 == 0 && al)
    return launch_pdl(combine4_kernel, dim3(T), dim3(kComb4Threads), 0, (cudaStream_t)stream, 1, "combine",
                      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(Y), gates, k_tok, k_max, d / 4,
                      reinterpret_cast<const float4*>(Y_shared), Y_shared ? n_shared : 0, shared_logits,
                      reinterpret_cast<float4*>(x_out), reinterpret_cast<float4*>(ln_out));
  const int threads = d >= 1024 ? 1024 : ((d + 31) / 32) * 32;
  return launch_pdl(combine_kernel, dim3(T), dim3(threads), 0, (cudaStream_t)stream, 1, "combine", x, Y, gates,
                    k_tok, k_max, d, Y_shared, Y_shared ? n_shared : 0, shared_logits, T, x_out, ln_out);
}

namespace mobile {
// SM count of the current device (grids are sized in multiples of it)
int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}
}  // namespace mobile

extern "C" int mobile_num_sms(void) { return mobile::sm_count(); }
