// Grouped expert FFN, weight-streaming form (decode / few tokens per expert).
// Replaces toymoe.py:202-204 (hidden = act(h2[pos] @ W_in[e]); y = hidden @ W_out[e]).
//
// At decode each expert sees 1..4 tokens, so the FFN is a set of GEMVs bound
// by HBM: every weight byte is read exactly once.  The work is cut into warp
// tasks of 8 output features of one expert (SwiGLU: 8 gate + 8 up rows, which
// the W13 layout stores contiguously as a 16-row group), spread over all SMs by
// a grid-stride over a device-side task count (the active-expert list written
// by mobile_permute), so no host sync is needed between routing and experts.
// Weight rows are streamed with 16-byte L1::no_allocate loads, R rows x 2
// vectors in flight per lane; activations (tiny, reused by every warp on the
// SM) come through the L1.  Each output is one warp's fixed-order dot product
// (deterministic, no atomics).
#include "common.cuh"

namespace mobile {

constexpr int kFfnThreads = 256;
constexpr int kFfnWarps = kFfnThreads / kWarp;

enum FfnMode { kGateUpSwiglu = 0, kGateUpRelu = 1, kDown = 2 };

struct FfnArgs {
  const float* x;          // activation rows (h2 rows for gate-up, U rows for down)
  int x_div;               // activation row = pair / x_div
  const int* offsets;      // (E+1)
  const int* sorted_pairs; // (P)
  const int* active;       // [n_active, ids...]
  int max_active;
  int K;                   // input dim
  int out_dim;             // output features per expert (I or d)
  const char* w_base;
  long long stride;        // bytes between consecutive slots
  const int* slot;
  float* out;              // (P, out_dim) f32
};

template <typename W, int TT, int R>
__device__ __forceinline__ void multirow_dot(const W* __restrict__ w, int K, const float* const* xr,
                                             int nt, float (&acc)[R][TT]) {
  constexpr int V = WVec<W>::N;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[r][t] = 0.f;
  const int nvec = K / V;
  for (int vi = lane; vi < nvec; vi += 64) {
    const bool two = vi + 32 < nvec;
    uint4 u0[R], u1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u0[r] = ld_stream_u4(w + (size_t)r * K + (size_t)vi * V);
    if (two) {
#pragma unroll
      for (int r = 0; r < R; ++r) u1[r] = ld_stream_u4(w + (size_t)r * K + (size_t)(vi + 32) * V);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
      const int k0 = (vi + h * 32) * V;
      float xv[TT][V];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          const float4* p = reinterpret_cast<const float4*>(xr[t] + k0);
#pragma unroll
          for (int q = 0; q < V / 4; ++q) {
            float4 f = __ldg(p + q);
            xv[t][4 * q + 0] = f.x; xv[t][4 * q + 1] = f.y; xv[t][4 * q + 2] = f.z; xv[t][4 * q + 3] = f.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < V; ++q) xv[t][q] = 0.f;
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float f[V];
        WVec<W>::widen(h == 0 ? u0[r] : u1[r], f);
#pragma unroll
        for (int t = 0; t < TT; ++t)
#pragma unroll
          for (int q = 0; q < V; ++q) acc[r][t] = fmaf(f[q], xv[t][q], acc[r][t]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[r][t] = warp_sum(acc[r][t]);
}

template <typename W, int TT, int MODE>
__global__ void __launch_bounds__(kFfnThreads) ffn_stream_kernel(FfnArgs a) {
  constexpr int F = 8;                               // output features per task
  constexpr int R = MODE == kGateUpSwiglu ? 2 * F : F;
  const int lane = threadIdx.x & 31;
  const int groups = a.out_dim / F;
  const int n_active = a.active[0];
  const int n_tasks = n_active * groups;
  const int wid = blockIdx.x * kFfnWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kFfnWarps;
  const size_t rows_per_expert = (size_t)(MODE == kGateUpSwiglu ? 2 : 1) * a.out_dim;
  for (int task = wid; task < n_tasks; task += nw) {
    const int e = a.active[1 + task / groups];
    const int g = task % groups;
    const int s = a.slot ? a.slot[e] : e;
    const W* w = reinterpret_cast<const W*>(a.w_base + (long long)s * a.stride) +
                 (size_t)g * R * a.K;
    (void)rows_per_expert;
    const int p0 = a.offsets[e], p1 = a.offsets[e + 1];
    for (int c = p0; c < p1; c += TT) {
      const int nt = min(TT, p1 - c);
      const float* xr[TT];
      int pair[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        pair[t] = t < nt ? a.sorted_pairs[c + t] : 0;
        xr[t] = a.x + (size_t)(pair[t] / a.x_div) * a.K;
      }
      float acc[R][TT];
      multirow_dot<W, TT, R>(w, a.K, xr, nt, acc);
      // epilogue: lane f (< 8) writes feature g*8+f of each token
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          float v = 0.f;
#pragma unroll
          for (int f = 0; f < F; ++f) {
            float o;
            if (MODE == kGateUpSwiglu) o = silu_f(acc[f][t]) * acc[F + f][t];
            else if (MODE == kGateUpRelu) o = fmaxf(acc[f][t], 0.f);
            else o = acc[f][t];
            v = lane == f ? o : v;
          }
          if (lane < F) a.out[(size_t)pair[t] * a.out_dim + (size_t)g * F + lane] = v;
        }
      }
    }
  }
}

static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename W, int MODE>
static int launch_ffn(const FfnArgs& a, int max_tok, cudaStream_t s) {
  const int groups = a.out_dim / 8;
  const long long tasks = (long long)a.max_active * groups;
  if (tasks == 0) return MOBILE_OK;
  long long blocks = (tasks + kFfnWarps - 1) / kFfnWarps;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  dim3 grid((unsigned)blocks), block(kFfnThreads);
  if (max_tok <= 1) ffn_stream_kernel<W, 1, MODE><<<grid, block, 0, s>>>(a);
  else if (max_tok == 2) ffn_stream_kernel<W, 2, MODE><<<grid, block, 0, s>>>(a);
  else ffn_stream_kernel<W, 4, MODE><<<grid, block, 0, s>>>(a);
  MOBILE_CHECK_LAUNCH("ffn_stream");
  return MOBILE_OK;
}

int ffn_dispatch(const FfnArgs& a, int w_dtype, int mode, int max_tok, cudaStream_t s) {
  if (w_dtype == MOBILE_BF16) {
    if (mode == kGateUpSwiglu) return launch_ffn<__nv_bfloat16, kGateUpSwiglu>(a, max_tok, s);
    if (mode == kGateUpRelu) return launch_ffn<__nv_bfloat16, kGateUpRelu>(a, max_tok, s);
    return launch_ffn<__nv_bfloat16, kDown>(a, max_tok, s);
  }
  if (w_dtype == MOBILE_F32) {
    if (mode == kGateUpSwiglu) return launch_ffn<float, kGateUpSwiglu>(a, max_tok, s);
    if (mode == kGateUpRelu) return launch_ffn<float, kGateUpRelu>(a, max_tok, s);
    return launch_ffn<float, kDown>(a, max_tok, s);
  }
  set_error("expert ffn: unsupported weight dtype %d", w_dtype);
  return MOBILE_ERR_UNSUPPORTED;
}

int sm_count() { return num_sms(); }

}  // namespace mobile

using namespace mobile;

static int check_ffn_shapes(int d, int I, int w_dtype) {
  const int V = w_dtype == MOBILE_BF16 ? 8 : 4;
  if (d <= 0 || I <= 0) { set_error("expert ffn: bad shape d=%d I=%d", d, I); return MOBILE_ERR_INVALID; }
  if (d % 8 || I % 8 || d % V || I % V) {
    set_error("expert ffn: d=%d and I=%d must be multiples of 8", d, I);
    return MOBILE_ERR_UNSUPPORTED;
  }
  return MOBILE_OK;
}

extern "C" int mobile_expert_gate_up(const float* h2, const int* offsets, const int* sorted_pairs,
                                     const int* active, int max_active, int max_tokens_per_expert,
                                     int tok_div, int d, int I, const void* w13_base,
                                     long long expert_stride, const int* slot, int w_dtype,
                                     int activation, float* U, void* stream) {
  int st = check_ffn_shapes(d, I, w_dtype);
  if (st) return st;
  if (tok_div <= 0) { set_error("expert ffn: tok_div must be > 0"); return MOBILE_ERR_INVALID; }
  FfnArgs a{h2, tok_div, offsets, sorted_pairs, active, max_active, d, I,
            (const char*)w13_base, expert_stride, slot, U};
  const int mode = activation == MOBILE_ACT_SWIGLU ? kGateUpSwiglu : kGateUpRelu;
  return ffn_dispatch(a, w_dtype, mode, max_tokens_per_expert, (cudaStream_t)stream);
}

extern "C" int mobile_expert_down(const float* U, const int* offsets, const int* sorted_pairs,
                                  const int* active, int max_active, int max_tokens_per_expert,
                                  int d, int I, const void* w2_base, long long expert_stride,
                                  const int* slot, int w_dtype, float* Y, void* stream) {
  int st = check_ffn_shapes(d, I, w_dtype);
  if (st) return st;
  FfnArgs a{U, 1, offsets, sorted_pairs, active, max_active, I, d,
            (const char*)w2_base, expert_stride, slot, Y};
  return ffn_dispatch(a, w_dtype, kDown, max_tokens_per_expert, (cudaStream_t)stream);
}

extern "C" int mobile_num_sms(void) { return sm_count(); }
