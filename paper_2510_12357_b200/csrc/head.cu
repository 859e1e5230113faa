// Output head + confidence: the reference's "importance score".
// Replaces toymoe.py:209-210 (probs = softmax(LN(x[-1]) @ head * 24)) plus
// toymoe.py:273 (confidence = max(probs)) and policy.py:69-79 (max p <= gamma
// falls back; strict > accepts).
//
// The head is the largest single weight on the decode path (V x d: 622 MB at
// the Qwen shape), so this is an HBM-streaming GEMV: CTAs own contiguous
// vocabulary slices, each warp streams 2 rows at a time with 16-byte
// no-allocate loads, and keeps an online (max, sum-exp, first-argmax) per
// token.  Per-CTA partials are merged by the last CTA to finish (atomic
// ticket) in CTA order, so the result is deterministic.  conf = 1 / Z where
// Z = sum exp(l - max) (the max element of softmax is exp(0)/Z).
#include "common.cuh"

namespace mobile {

constexpr int kHeadThreads = 256;
constexpr int kHeadWarps = kHeadThreads / 32;
constexpr int kHeadTT = 4;  // tokens per launch pass

struct HeadPartial {
  float m;
  float s;
  int arg;
  int pad;
};

struct HeadArgs {
  const float* x;
  const void* w;
  int T, d, V;
  float scale, gamma;
  float* logits_out;
  float* conf_out;
  int* argmax_out;
  uint8_t* fallback_out;
  HeadPartial* partials;  // (T, gridDim.x)
  unsigned int* ticket;   // one counter, left at 0
};

__device__ __forceinline__ void online_merge(float& m, float& s, int& arg, float m2, float s2, int arg2) {
  // merge (m2, s2, arg2) that comes AFTER (m, s, arg) in vocabulary order
  if (m2 > m) {
    s = s * expf(m - m2) + s2;
    m = m2;
    arg = arg2;
  } else {
    s = s + s2 * expf(m2 - m);
  }
}

template <typename W>
__global__ void __launch_bounds__(kHeadThreads) head_kernel(HeadArgs a) {
  extern __shared__ __align__(16) float sh[];
  float* h = sh;                                   // kHeadTT * d
  float* red = sh + (size_t)kHeadTT * a.d;         // warp partials: kHeadWarps * kHeadTT * 3
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t0 = blockIdx.y * kHeadTT;
  const int nt = min(kHeadTT, a.T - t0);

  // LN of the token rows (toymoe.py:209 _layer_norm(x[-1]))
  for (int t = 0; t < nt; ++t) {
    const float* xr = a.x + (size_t)(t0 + t) * a.d;
    float sum = 0.f;
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) { float v = xr[i]; h[(size_t)t * a.d + i] = v; sum += v; }
    sum = warp_sum(sum);
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    float mean = 0.f;
    for (int w = 0; w < kHeadWarps; ++w) mean += red[w];
    mean /= (float)a.d;
    __syncthreads();
    float q = 0.f;
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) { float c = h[(size_t)t * a.d + i] - mean; q += c * c; }
    q = warp_sum(q);
    if (lane == 0) red[warp] = q;
    __syncthreads();
    float var = 0.f;
    for (int w = 0; w < kHeadWarps; ++w) var += red[w];
    var /= (float)a.d;
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    __syncthreads();
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) h[(size_t)t * a.d + i] = (h[(size_t)t * a.d + i] - mean) * inv;
  }
  __syncthreads();

  // this CTA's vocabulary slice
  const int per = (a.V + gridDim.x - 1) / gridDim.x;
  const int v0 = blockIdx.x * per, v1 = min(a.V, v0 + per);
  const W* w = reinterpret_cast<const W*>(a.w);
  constexpr int Vn = WVec<W>::N;
  const int nvec = a.d / Vn;
  float m[kHeadTT], s[kHeadTT];
  int arg[kHeadTT];
#pragma unroll
  for (int t = 0; t < kHeadTT; ++t) { m[t] = -INFINITY; s[t] = 0.f; arg[t] = 0x7fffffff; }
  // warp handles rows v0 + warp*2 + {0,1}, stepping 2*kHeadWarps
  for (int r = v0 + warp * 2; r < v1; r += 2 * kHeadWarps) {
    const bool two = r + 1 < v1;
    float acc[2][kHeadTT];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int t = 0; t < kHeadTT; ++t) acc[i][t] = 0.f;
    const W* w0 = w + (size_t)r * a.d;
    const W* w1 = w0 + a.d;
    for (int vi = lane; vi < nvec; vi += 64) {
      const bool hi = vi + 32 < nvec;
      uint4 u[4];
      u[0] = ld_stream_u4(w0 + (size_t)vi * Vn);
      if (two) u[1] = ld_stream_u4(w1 + (size_t)vi * Vn);
      if (hi) {
        u[2] = ld_stream_u4(w0 + (size_t)(vi + 32) * Vn);
        if (two) u[3] = ld_stream_u4(w1 + (size_t)(vi + 32) * Vn);
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (hh == 1 && !hi) break;
        const int k0 = (vi + hh * 32) * Vn;
        float f0[Vn], f1[Vn];
        WVec<W>::widen(u[hh * 2], f0);
        if (two) WVec<W>::widen(u[hh * 2 + 1], f1);
#pragma unroll
        for (int t = 0; t < kHeadTT; ++t) {
          if (t < nt) {
            const float* hr = h + (size_t)t * a.d + k0;
#pragma unroll
            for (int q = 0; q < Vn; ++q) {
              acc[0][t] = fmaf(f0[q], hr[q], acc[0][t]);
              if (two) acc[1][t] = fmaf(f1[q], hr[q], acc[1][t]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (i == 1 && !two) break;
#pragma unroll
      for (int t = 0; t < kHeadTT; ++t) {
        if (t < nt) {
          float l = warp_sum(acc[i][t]) * a.scale;
          if (a.logits_out && lane == 0) a.logits_out[(size_t)(t0 + t) * a.V + r + i] = l;
          online_merge(m[t], s[t], arg[t], l, 1.0f, r + i);
        }
      }
    }
  }
  // block merge in warp order.  Warps interleave rows, so merge by (m, arg):
  // equal maxima keep the smaller vocabulary index.
  for (int t = 0; t < nt; ++t) {
    if (lane == 0) {
      red[(warp * kHeadTT + t) * 3 + 0] = m[t];
      red[(warp * kHeadTT + t) * 3 + 1] = s[t];
      red[(warp * kHeadTT + t) * 3 + 2] = __int_as_float(arg[t]);
    }
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    const int t = threadIdx.x;
    float M = -INFINITY, S = 0.f;
    int A = 0x7fffffff;
    for (int w2 = 0; w2 < kHeadWarps; ++w2) {
      float m2 = red[(w2 * kHeadTT + t) * 3 + 0], s2 = red[(w2 * kHeadTT + t) * 3 + 1];
      int a2 = __float_as_int(red[(w2 * kHeadTT + t) * 3 + 2]);
      if (s2 == 0.f) continue;
      if (m2 > M) { S = S * expf(M - m2) + s2; M = m2; A = a2; }
      else { S = S + s2 * expf(m2 - M); if (m2 == M && a2 < A) A = a2; }
    }
    a.partials[(size_t)(t0 + t) * gridDim.x + blockIdx.x] = HeadPartial{M, S, A, 0};
  }
  // last CTA of this token tile merges all partials in CTA order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(a.ticket + blockIdx.y, 1u);
    is_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (threadIdx.x < nt) {
    const int t = threadIdx.x;
    float M = -INFINITY, S = 0.f;
    int A = 0x7fffffff;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const volatile HeadPartial* vp = a.partials + (size_t)(t0 + t) * gridDim.x + b;
      const float pm = vp->m, ps = vp->s;
      const int pa = vp->arg;
      if (ps == 0.f) continue;
      if (pm > M) { S = S * expf(M - pm) + ps; M = pm; A = pa; }
      else { S = S + ps * expf(pm - M); if (pm == M && pa < A) A = pa; }
    }
    const float conf = 1.0f / S;
    a.conf_out[t0 + t] = conf;
    if (a.argmax_out) a.argmax_out[t0 + t] = A;
    if (a.fallback_out) a.fallback_out[t0 + t] = conf <= a.gamma ? 1 : 0;
  }
  if (threadIdx.x == 0) a.ticket[blockIdx.y] = 0u;  // leave the workspace reusable
}

static int head_grid_x(int V) {
  int g = sm_count() * 4;
  const int min_rows = 2 * kHeadWarps;
  if ((long long)g * min_rows > V) g = (V + min_rows - 1) / min_rows;
  return g < 1 ? 1 : g;
}

// ---------------------------------------------------------------- confidence of logits rows
// Large-batch decode: the head product runs as a tcgen05 GEMM (raw logits,
// T x V f32); this reduces each row to the head's outputs with the same
// arithmetic as head_kernel (l = raw * scale, conf = 1 / sum exp(l - max),
// first maximiser).  One CTA per row; merges in a fixed (thread, warp) order.
constexpr int kConfThreads = 512;

__device__ __forceinline__ void conf_merge(float& M, float& S, int& A, float m, float s, int a) {
  if (s == 0.f) return;
  if (m > M) { S = S * expf(M - m) + s; M = m; A = a; }
  else { S += s * expf(m - M); if (m == M && a < A) A = a; }
}

__global__ void __launch_bounds__(kConfThreads) logits_conf_kernel(const float* __restrict__ logits, int V,
                                                                   float scale, float gamma, float* conf_out,
                                                                   int* argmax_out, uint8_t* fallback_out) {
  __shared__ float rm[kConfThreads / 32], rs[kConfThreads / 32];
  __shared__ int ra[kConfThreads / 32];
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const float* row = logits + (size_t)t * V;
  float m = -INFINITY, s = 0.f;
  int arg = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += kConfThreads) online_merge(m, s, arg, row[i] * scale, 1.0f, i);
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, arg, o);
    conf_merge(m, s, arg, m2, s2, a2);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { rm[warp] = m; rs[warp] = s; ra[warp] = arg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    int A = 0x7fffffff;
    for (int w = 0; w < kConfThreads / 32; ++w) conf_merge(M, S, A, rm[w], rs[w], ra[w]);
    const float conf = 1.0f / S;
    conf_out[t] = conf;
    if (argmax_out) argmax_out[t] = A;
    if (fallback_out) fallback_out[t] = conf <= gamma ? 1 : 0;
  }
}

// ---------------------------------------------------------------- softmax rows
// probs = exp(l - max) / sum (toymoe.py:91-94); accumulation in Acc (double
// when either side is f64, so the fp64 API keeps |sum - 1| ~ 1e-16).
template <typename In, typename Out, typename Acc>
__global__ void softmax_rows_kernel(const In* __restrict__ logits, Out* __restrict__ probs, int V) {
  __shared__ Acc red[32];
  const In* row = logits + (size_t)blockIdx.x * V;
  Out* out = probs + (size_t)blockIdx.x * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Acc m = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmax(m, (Acc)row[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = -INFINITY;
  for (int w = 0; w < nw; ++w) m = fmax(m, red[w]);
  __syncthreads();
  Acc s = 0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += exp((Acc)row[i] - m);
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0;
  for (int w = 0; w < nw; ++w) s += red[w];
  for (int i = threadIdx.x; i < V; i += blockDim.x) out[i] = (Out)(exp((Acc)row[i] - m) / s);
}

// ---------------------------------------------------------------- probs check
template <typename F>
__global__ void probs_check_kernel(const F* __restrict__ p, int V, double* out) {
  __shared__ double rs[32], rm[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double s = 0.0, m = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) { double v = (double)p[i]; s += v; m = fmax(m, v); }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) { rs[warp] = s; rm[warp] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0, M = -INFINITY;
    for (int w = 0; w < nw; ++w) { S += rs[w]; M = fmax(M, rm[w]); }
    out[0] = S;
    out[1] = M;
  }
}

}  // namespace mobile

using namespace mobile;

extern "C" size_t mobile_head_ws_bytes(int T, int V) {
  const int g = head_grid_x(V);
  const int ty = (T + kHeadTT - 1) / kHeadTT;
  return 256 + sizeof(HeadPartial) * (size_t)ty * kHeadTT * g + sizeof(unsigned) * (size_t)ty;
}

extern "C" int mobile_head_confidence(const float* x, const void* w_head, int w_dtype, int T, int d,
                                      int V, float logit_scale, float gamma, float* logits_out,
                                      float* conf_out, int* argmax_out, uint8_t* fallback_out,
                                      void* workspace, void* stream) {
  if (T < 0 || d <= 0 || V <= 0) { set_error("head: bad shape T=%d d=%d V=%d", T, d, V); return MOBILE_ERR_INVALID; }
  if (T == 0) return MOBILE_OK;
  const int Vn = w_dtype == MOBILE_BF16 ? 8 : 4;
  if (d % Vn) { set_error("head: d=%d must be a multiple of %d", d, Vn); return MOBILE_ERR_UNSUPPORTED; }
  const int gx = head_grid_x(V);
  const int ty = (T + kHeadTT - 1) / kHeadTT;
  unsigned* ticket = reinterpret_cast<unsigned*>(workspace);
  HeadPartial* partials = reinterpret_cast<HeadPartial*>(reinterpret_cast<char*>(workspace) + 256);
  if (ty > 64) { set_error("head: T=%d too large for one launch", T); return MOBILE_ERR_UNSUPPORTED; }
  HeadArgs a{x, w_head, T, d, V, logit_scale, gamma, logits_out, conf_out, argmax_out, fallback_out, partials, ticket};
  const size_t smem = sizeof(float) * ((size_t)kHeadTT * d + kHeadWarps * kHeadTT * 3 + 8);
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid(gx, ty), block(kHeadThreads);
  if (w_dtype == MOBILE_BF16) {
    set_smem_once((const void*)head_kernel<__nv_bfloat16>, smem);
    head_kernel<__nv_bfloat16><<<grid, block, smem, s>>>(a);
  } else if (w_dtype == MOBILE_F32) {
    set_smem_once((const void*)head_kernel<float>, smem);
    head_kernel<float><<<grid, block, smem, s>>>(a);
  } else {
    set_error("head: unsupported weight dtype %d", w_dtype);
    return MOBILE_ERR_UNSUPPORTED;
  }
  MOBILE_CHECK_LAUNCH("head_confidence");
  return MOBILE_OK;
}

extern "C" int mobile_softmax_rows(const void* logits, int in_dtype, void* probs, int out_dtype, int T,
                                   int V, void* stream) {
  if (T < 0 || V <= 0) { set_error("softmax: bad shape"); return MOBILE_ERR_INVALID; }
  if (T == 0) return MOBILE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (in_dtype == MOBILE_F32 && out_dtype == MOBILE_F32)
    softmax_rows_kernel<float, float, float><<<T, 512, 0, s>>>((const float*)logits, (float*)probs, V);
  else if (in_dtype == MOBILE_F32 && out_dtype == MOBILE_F64)
    softmax_rows_kernel<float, double, double><<<T, 512, 0, s>>>((const float*)logits, (double*)probs, V);
  else if (in_dtype == MOBILE_F64 && out_dtype == MOBILE_F64)
    softmax_rows_kernel<double, double, double><<<T, 512, 0, s>>>((const double*)logits, (double*)probs, V);
  else { set_error("softmax: unsupported dtypes %d -> %d", in_dtype, out_dtype); return MOBILE_ERR_UNSUPPORTED; }
  MOBILE_CHECK_LAUNCH("softmax_rows");
  return MOBILE_OK;
}

extern "C" int mobile_probs_check(const void* probs, int dtype, int V, double* out, void* stream) {
  if (V <= 0) { set_error("probs: empty"); return MOBILE_ERR_INVALID; }
  if (dtype == MOBILE_F64) probs_check_kernel<double><<<1, 512, 0, (cudaStream_t)stream>>>((const double*)probs, V, out);
  else if (dtype == MOBILE_F32) probs_check_kernel<float><<<1, 512, 0, (cudaStream_t)stream>>>((const float*)probs, V, out);
  else { set_error("probs: unsupported dtype %d", dtype); return MOBILE_ERR_UNSUPPORTED; }
  MOBILE_CHECK_LAUNCH("probs_check");
  return MOBILE_OK;
}

extern "C" int mobile_logits_confidence(const float* logits, int T, int V, float logit_scale, float gamma,
                                        float* conf_out, int* argmax_out, uint8_t* fallback_out, void* stream) {
  if (T < 0 || V <= 0 || !logits || !conf_out) { set_error("logits_confidence: bad arguments T=%d V=%d", T, V); return MOBILE_ERR_INVALID; }
  if (T == 0) return MOBILE_OK;
  return launch_pdl(logits_conf_kernel, dim3(T), dim3(kConfThreads), 0, (cudaStream_t)stream, 1, "logits_confidence",
                    logits, V, logit_scale, gamma, conf_out, argmax_out, fallback_out);
}
