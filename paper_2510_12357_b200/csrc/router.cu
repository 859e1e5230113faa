// Fused router: LN -> router GEMV -> stable top-k -> replay -> gate softmax.
// Replaces toymoe.py:188-201 (and the top_k of policy.py:98-103).
//
// One thread-block cluster of CS CTAs per tile of TT tokens.  Every CTA
// layer-normalises the tile into shared memory (the d-row is re-read from L2,
// 8 KB at d=2048) and computes the logits of its E/CS slice of router rows;
// the slices are written into the leader CTA's shared memory over DSMEM, one
// cluster barrier, then the leader's warps run the top-k (one warp per token).
// Splitting the rows over a cluster keeps batch-1 decode (T=1) from being
// limited by a single SM's load bandwidth while keeping the reduction
// deterministic (each logit is one warp's fixed-order dot product).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mobile {

constexpr int kRouterThreads = 256;
constexpr int kRouterWarps = kRouterThreads / kWarp;
constexpr int kMaxE = 256;       // toymoe.py:40 _MAX_EXPERTS
constexpr int kMaxExtra = 8;

struct RouterArgs {
  const float* x;
  float* h2_out;
  const void* w;
  int T, d, E, n_extra, k_max;
  const int* k_tok;
  const float* replay;
  const uint8_t* replay_mask;
  int reuse_gates, gate_norm;
  float* logits_out;
  float* extra_out;
  int* idx_out;
  float* gates_out;
  int* flags;
  int* perm_offsets;   // fused permute (single token tile, T*k_max <= 32), else NULL
  int* perm_pairs;
  int* perm_active;
  // optional: L2 prefetch of each selected expert's first pf_bytes at
  // pf_base + e * pf_stride, issued as soon as the selection is known (the
  // routed gate-up launch that follows finds its first tiles in L2)
  const char* pf_base;
  long long pf_stride, pf_bytes;
};

// Deterministic stable permute of <= 32 (token, slot) pairs by one warp
// (the mobile_permute contract): bitonic sort of keys (expert << 6 | pair).
__device__ void warp_permute(const RouterArgs& a) {
  const int lane = threadIdx.x & 31;
  const int P = a.T * a.k_max;
  int key = 0x7fffffff;
  if (lane < P) {
    const int t = lane / a.k_max, j = lane - t * a.k_max;
    const int kt = a.k_tok ? a.k_tok[t] : a.k_max;
    const int e = j < kt ? a.idx_out[lane] : -1;
    if (e >= 0 && e < a.E) key = (e << 6) | lane;
  }
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int other = __shfl_xor_sync(0xffffffffu, key, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      key = (lower == up) ? min(key, other) : max(key, other);
    }
  }
  const bool valid = key != 0x7fffffff;
  const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
  const int e_me = valid ? (key >> 6) : 0x7fffffff;
  if (valid) a.perm_pairs[lane] = key & 63;
  const int e_prev = __shfl_up_sync(0xffffffffu, e_me, 1);
  const bool first = valid && (lane == 0 || e_prev != e_me);
  const unsigned fm = __ballot_sync(0xffffffffu, first);
  if (first) a.perm_active[1 + __popc(fm & ((1u << lane) - 1u))] = e_me;
  if (lane == 0) a.perm_active[0] = __popc(fm);
  // offsets[e] = #pairs with expert < e  (uniform trip count: every lane
  // takes part in every shuffle)
  for (int base = 0; base <= a.E; base += 32) {
    const int e = base + lane;
    int c = 0;
    for (int j = 0; j < 32; ++j) {
      const int ej = __shfl_sync(0xffffffffu, e_me, j);
      c += ej < e;
    }
    if (e <= a.E) a.perm_offsets[e] = c;
  }
  (void)nvalid;
}

// Block-wide LayerNorm statistics for TT rows held in smem (two-pass, like
// numpy: mean, then mean of squared deviations; toymoe.py:129-132).
template <int TT>
__device__ void tile_layer_norm(float* h, int rows, int d, float* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = 0; t < rows; ++t) {
    float* row = h + (size_t)t * d;
    float s = 0.f;
    for (int i = tid; i < d; i += blockDim.x) s += row[i];
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (warp == 0) {
      float v = lane < kRouterWarps ? red[lane] : 0.f;
      v = warp_sum(v);
      if (lane == 0) red[kRouterWarps] = v / (float)d;
    }
    __syncthreads();
    const float mean = red[kRouterWarps];
    float q = 0.f;
    for (int i = tid; i < d; i += blockDim.x) {
      float c = row[i] - mean;
      q += c * c;
    }
    q = warp_sum(q);
    __syncthreads();
    if (lane == 0) red[warp] = q;
    __syncthreads();
    if (warp == 0) {
      float v = lane < kRouterWarps ? red[lane] : 0.f;
      v = warp_sum(v);
      if (lane == 0) red[kRouterWarps + 1] = v / (float)d;
    }
    __syncthreads();
    const float inv = 1.0f / sqrtf(red[kRouterWarps + 1] + 1e-5f);
    for (int i = tid; i < d; i += blockDim.x) row[i] = (row[i] - mean) * inv;
    __syncthreads();
  }
}

// acc[t] = sum_k h[t][k] * w[k] for one weight row (warp-cooperative).
template <typename W, int TT>
__device__ __forceinline__ void warp_row_dot(const W* __restrict__ wrow, const float* h, int d,
                                             int rows, float* acc) {
  constexpr int V = WVec<W>::N;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < TT; ++t) acc[t] = 0.f;
  const int nvec = d / V;
  int vi = lane;
  for (; vi + 3 * 32 < nvec; vi += 4 * 32) {
    uint4 u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = ld_stream_u4(wrow + (size_t)(vi + j * 32) * V);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float f[V];
      WVec<W>::widen(u[j], f);
      const int k0 = (vi + j * 32) * V;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < rows) {
          const float* hr = h + (size_t)t * d + k0;
#pragma unroll
          for (int q = 0; q < V; ++q) acc[t] = fmaf(f[q], hr[q], acc[t]);
        }
      }
    }
  }
  for (; vi < nvec; vi += 32) {
    uint4 u = ld_stream_u4(wrow + (size_t)vi * V);
    float f[V];
    WVec<W>::widen(u, f);
    const int k0 = vi * V;
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      if (t < rows) {
        const float* hr = h + (size_t)t * d + k0;
#pragma unroll
        for (int q = 0; q < V; ++q) acc[t] = fmaf(f[q], hr[q], acc[t]);
      }
    }
  }
  // scalar tail (d not a multiple of V)
  for (int k = nvec * V + lane; k < d; k += 32) {
    float wv = (float)wrow[k];
#pragma unroll
    for (int t = 0; t < TT; ++t)
      if (t < rows) acc[t] = fmaf(wv, h[(size_t)t * d + k], acc[t]);
  }
#pragma unroll
  for (int t = 0; t < TT; ++t) acc[t] = warp_sum(acc[t]);
}

// Stable top-k over one row held as E values (own logits in smem).
// Writes idx/gates for token `tok`.  One warp.
__device__ void warp_route_token(const RouterArgs& a, int tok, const float* own) {
  const int lane = threadIdx.x & 31;
  const int E = a.E;
  int k = a.k_tok ? a.k_tok[tok] : a.k_max;
  if (k > E || k > a.k_max || k < 0) {
    if (lane == 0) atomicOr(a.flags, 2);
    k = min(min(k, E), a.k_max);
    if (k < 0) k = 0;
  }
  const bool replay = a.replay != nullptr && a.replay_mask != nullptr && a.replay_mask[tok] != 0;
  const float* sel_src = replay ? a.replay + (size_t)tok * E : own;
  const float* gate_src = (replay && a.reuse_gates) ? a.replay + (size_t)tok * E : own;

  // keys held in registers: lane owns e = lane + 32*i
  constexpr int kPer = kMaxE / 32;
  unsigned long long key[kPer];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    if (e < E) {
      float v = sel_src[e];
      bad |= !isfinite(v);
      key[i] = topk_key(v, e);
    } else {
      key[i] = 0ull;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags, 1);

  int* idx_row = a.idx_out + (size_t)tok * a.k_max;
  float* gate_row = a.gates_out + (size_t)tok * a.k_max;
  int sel_local = -1;  // lane j keeps the j-th selected index (k <= 32 fast path)
  for (int j = 0; j < k; ++j) {
    unsigned long long best = 0ull;
#pragma unroll
    for (int i = 0; i < kPer; ++i) best = key[i] > best ? key[i] : best;
    best = warp_max_u64(best);
    const int e = topk_key_index(best);
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (key[i] == best) key[i] = 0ull;
    if (lane == 0) idx_row[j] = e;
    if (lane == (j & 31)) sel_local = e;
  }
  for (int j = k + lane; j < a.k_max; j += 32) {
    idx_row[j] = -1;
    gate_row[j] = 0.f;
  }
  __syncwarp();
  // gate softmax in selection order (toymoe.py:201 / HF softmax-all extension)
  if (a.gate_norm == MOBILE_GATE_SELECTED_SOFTMAX) {
    if (k <= 32) {
      float gl = lane < k ? gate_src[sel_local] : -INFINITY;
      float m = warp_max(gl);
      float ex = lane < k ? expf(gl - m) : 0.f;
      // sequential sum in selection order (numpy sums short vectors serially)
      float s = 0.f;
      for (int j = 0; j < k; ++j) s += __shfl_sync(0xffffffffu, ex, j);
      if (lane < k) gate_row[lane] = ex / s;
    } else if (lane == 0) {
      float m = -INFINITY;
      for (int j = 0; j < k; ++j) m = fmaxf(m, gate_src[idx_row[j]]);
      float s = 0.f;
      for (int j = 0; j < k; ++j) s += expf(gate_src[idx_row[j]] - m);
      for (int j = 0; j < k; ++j) gate_row[j] = expf(gate_src[idx_row[j]] - m) / s;
    }
  } else {
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, gate_src[e]);
    m = warp_max(m);
    float z = 0.f;
    for (int e = lane; e < E; e += 32) z += expf(gate_src[e] - m);
    z = warp_sum(z);
    for (int j = lane; j < k; j += 32) gate_row[j] = expf(gate_src[idx_row[j]] - m) / z;
  }
}

template <typename W, int TT>
__global__ void __launch_bounds__(kRouterThreads) router_kernel(RouterArgs a) {
  extern __shared__ __align__(16) float smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int Etot = a.E + a.n_extra;
  const int t0 = blockIdx.y * TT;
  const int rows = min(TT, a.T - t0);
  float* h = smem;                                  // TT * d
  float* logits = smem + (size_t)TT * a.d;          // TT * Etot (leader's copy is used)
  float* red = logits + (size_t)TT * Etot;          // reduction scratch
  // every CTA of the cluster must have started before DSMEM is touched; the
  // relaxed arrive here overlaps that handshake with the LayerNorm below.
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  pdl_trigger();
  {  // the router rows are static: pull this CTA's slice into L2 while the previous kernel drains
    const int per0 = (Etot + CS - 1) / CS;
    const int eb = rank * per0, ee = min(Etot, eb + per0);
    if (threadIdx.x == 0 && ee > eb) {
      const char* src = reinterpret_cast<const char*>(a.w) + (size_t)eb * a.d * sizeof(W);
      const unsigned bytes = (unsigned)((size_t)(ee - eb) * a.d * sizeof(W));
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (bytes & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  }
  pdl_wait();  // x is the previous kernel's output

  // 1. stage + layer-normalise the token tile
  for (int t = 0; t < rows; ++t) {
    const float4* src = reinterpret_cast<const float4*>(a.x + (size_t)(t0 + t) * a.d);
    float4* dst = reinterpret_cast<float4*>(h + (size_t)t * a.d);
    if ((a.d & 3) == 0) {
      for (int i = threadIdx.x; i < a.d / 4; i += blockDim.x) dst[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < a.d; i += blockDim.x) h[(size_t)t * a.d + i] = a.x[(size_t)(t0 + t) * a.d + i];
    }
  }
  __syncthreads();
  tile_layer_norm<TT>(h, rows, a.d, red);
  if (rank == 0 && a.h2_out) {
    for (int t = 0; t < rows; ++t)
      for (int i = threadIdx.x; i < a.d; i += blockDim.x) a.h2_out[(size_t)(t0 + t) * a.d + i] = h[(size_t)t * a.d + i];
  }

  // 2. this CTA's slice of router rows -> leader smem (DSMEM)
  const int per = (Etot + CS - 1) / CS;
  const int e_begin = rank * per, e_end = min(Etot, e_begin + per);
  float* leader_logits = cluster.map_shared_rank(logits, 0);
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  const W* w = reinterpret_cast<const W*>(a.w);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = e_begin + warp; e < e_end; e += kRouterWarps) {
    float acc[TT];
    warp_row_dot<W, TT>(w + (size_t)e * a.d, h, a.d, rows, acc);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < rows) {
          leader_logits[(size_t)t * Etot + e] = acc[t];
          if (e < a.E) a.logits_out[(size_t)(t0 + t) * a.E + e] = acc[t];
          else if (a.extra_out) a.extra_out[(size_t)(t0 + t) * a.n_extra + (e - a.E)] = acc[t];
        }
      }
    }
  }
  cluster.sync();
  if (rank != 0) return;

  // 3. top-k + replay + gates, one warp per token
  for (int t = warp; t < rows; t += kRouterWarps) {
    // compact own logits (first E of the Etot row) are contiguous already
    warp_route_token(a, t0 + t, logits + (size_t)t * Etot);
  }
  if (a.perm_offsets) {  // 4. fused permute (decode): every token of the launch is in this tile
    __syncthreads();
    if (warp == 0) warp_permute(a);
  }
  if (a.pf_base) {  // 5. the selected experts' weights toward L2 (HBM is idle during routing)
    __syncthreads();
    constexpr long long kChunk = 64 * 1024;
    for (int q = warp; q < rows * a.k_max; q += kRouterWarps) {
      const int t = q / a.k_max, j = q - t * a.k_max;
      const int kt = a.k_tok ? a.k_tok[t0 + t] : a.k_max;
      if (j >= kt) continue;
      const int e = a.idx_out[(size_t)(t0 + t) * a.k_max + j];
      const char* src = a.pf_base + (long long)e * a.pf_stride;
      for (long long off = (long long)lane * kChunk; off < a.pf_bytes; off += 32 * kChunk) {
        const unsigned n = (unsigned)min(kChunk, a.pf_bytes - off);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"(n) : "memory");
      }
    }
  }
}

constexpr int kRouterClusterMaxT = 256;  // measured: clusters win up to batch 256, lose at 512-token prefill

template <typename W, int TT>
static int launch_router(const RouterArgs& a, cudaStream_t stream) {
  const int Etot = a.E + a.n_extra;
  // small T: a cluster of up to 8 CTAs splits the router rows of each token
  // tile (latency); large T (prefill, big batches): the token tiles alone fill
  // the GPU, so one CTA per tile computes every row (no cluster co-scheduling)
  const int cs = a.T > kRouterClusterMaxT ? 1 : min(8, max(1, (Etot + 7) / 8));
  const size_t smem = sizeof(float) * ((size_t)TT * a.d + (size_t)TT * Etot + 64);
  auto kern = router_kernel<W, TT>;
  if (int st = set_smem_once((const void*)kern, smem)) return st;
  return launch_pdl(kern, dim3(cs, (a.T + TT - 1) / TT, 1), dim3(kRouterThreads), smem, stream, cs,
                    "router launch", a);
}

template <typename W>
static int launch_router_tt(const RouterArgs& a, int TT, cudaStream_t s) {
  switch (TT) {
    case 1: return launch_router<W, 1>(a, s);
    case 2: return launch_router<W, 2>(a, s);
    default: return launch_router<W, 4>(a, s);
  }
}

// ---------------------------------------------------------------- topk rows
// One warp per row; keys staged in shared memory; f32 or f64 input.
template <typename F>
__global__ void topk_rows_kernel(const F* __restrict__ rows, int R, int E, int k, int* idx_out,
                                 int* flags) {
  extern __shared__ unsigned long long keys[];  // warps_per_block * E
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int r = blockIdx.x * wpb + warp;
  if (r >= R) return;
  unsigned long long* kr = keys + (size_t)warp * E;
  const F* row = rows + (size_t)r * E;
  bool bad = false;
  for (int e = lane; e < E; e += 32) {
    F v = row[e];
    bad |= !isfinite((double)v);
    if constexpr (sizeof(F) == 8) kr[e] = order_key_f64((double)v);
    else kr[e] = (unsigned long long)order_key_f32((float)v);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1);
  __syncwarp();
  // live keys are >= 1 (a key of 0 is only possible for an all-ones -NaN,
  // which is flagged above); a taken entry is set to 0 and never wins again.
  for (int e = lane; e < E; e += 32) kr[e] = kr[e] == 0ull ? 1ull : kr[e];
  __syncwarp();
  for (int j = 0; j < k; ++j) {
    unsigned long long bk = 0ull;
    int bi = E;
    for (int e = lane; e < E; e += 32) {
      unsigned long long v = kr[e];
      if (v > bk) { bk = v; bi = e; }  // e ascends per lane: first max kept
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    if (lane == 0) {
      idx_out[(size_t)r * k + j] = bi;
      kr[bi] = 0ull;
    }
    __syncwarp();
  }
}

}  // namespace mobile

using namespace mobile;

extern "C" int mobile_permute(const int* idx, const int* k_tok, int T, int k_max, int E, int* offsets,
                              int* sorted_pairs, int* active, void* stream);

extern "C" int mobile_router_topk(const float* x, float* h2_out, const void* w_router, int w_dtype,
                                  int T, int d, int E, int n_extra, int k_max, const int* k_tok,
                                  const float* replay, const uint8_t* replay_mask, int reuse_gates,
                                  int gate_norm, float* logits_out, float* extra_out, int* idx_out,
                                  float* gates_out, int* flags, int* perm_offsets, int* perm_pairs,
                                  int* perm_active, void* stream) {
  return mobile_router_topk_pf(x, h2_out, w_router, w_dtype, T, d, E, n_extra, k_max, k_tok, replay, replay_mask,
                               reuse_gates, gate_norm, logits_out, extra_out, idx_out, gates_out, flags,
                               perm_offsets, perm_pairs, perm_active, nullptr, 0, 0, stream);
}

extern "C" int mobile_router_topk_pf(const float* x, float* h2_out, const void* w_router, int w_dtype,
                                     int T, int d, int E, int n_extra, int k_max, const int* k_tok,
                                     const float* replay, const uint8_t* replay_mask, int reuse_gates,
                                     int gate_norm, float* logits_out, float* extra_out, int* idx_out,
                                     float* gates_out, int* flags, int* perm_offsets, int* perm_pairs,
                                     int* perm_active, const void* pf_base, long long pf_stride,
                                     long long pf_bytes, void* stream) {
  if (T < 0 || d <= 0 || E <= 0 || k_max <= 0) { set_error("router: bad shape T=%d d=%d E=%d k=%d", T, d, E, k_max); return MOBILE_ERR_INVALID; }
  if (E > kMaxE) { set_error("router: E=%d exceeds kernel limit %d", E, kMaxE); return MOBILE_ERR_UNSUPPORTED; }
  if (n_extra < 0 || n_extra > kMaxExtra) { set_error("router: n_extra=%d unsupported", n_extra); return MOBILE_ERR_UNSUPPORTED; }
  if (k_max > E) { set_error("k (%d) exceeds number of experts (%d)", k_max, E); return MOBILE_ERR_K_EXCEEDS; }
  if (T == 0) return MOBILE_OK;
  if (d % 4 != 0 || (w_dtype == MOBILE_BF16 && d % 8 != 0)) { set_error("router: d=%d must be a multiple of 8", d); return MOBILE_ERR_UNSUPPORTED; }
  // tokens per cluster: the kernel is latency-bound, so many small tiles beat
  // fewer large ones (measured: 8/16-token tiles slow both batch-64 decode
  // and 512-token prefill)
  const int TT = T == 1 ? 1 : (T == 2 ? 2 : 4);
  const bool fuse = perm_offsets && perm_pairs && perm_active && T <= TT && T * k_max <= 32;
  RouterArgs a{x, h2_out, w_router, T, d, E, n_extra, k_max, k_tok, replay, replay_mask, reuse_gates,
               gate_norm, logits_out, extra_out, idx_out, gates_out, flags,
               fuse ? perm_offsets : nullptr, fuse ? perm_pairs : nullptr, fuse ? perm_active : nullptr,
               (pf_bytes >= 16 && (pf_stride & 15) == 0 && (reinterpret_cast<uintptr_t>(pf_base) & 15) == 0)
                   ? reinterpret_cast<const char*>(pf_base) : nullptr,
               pf_stride, pf_bytes & ~15LL};
  cudaStream_t s = (cudaStream_t)stream;
  int st;
  if (w_dtype == MOBILE_BF16) st = launch_router_tt<__nv_bfloat16>(a, TT, s);
  else if (w_dtype == MOBILE_F32) st = launch_router_tt<float>(a, TT, s);
  else { set_error("router: unsupported weight dtype %d", w_dtype); return MOBILE_ERR_UNSUPPORTED; }
  if (st || !perm_offsets || fuse) return st;
  return mobile_permute(idx_out, k_tok, T, k_max, E, perm_offsets, perm_pairs, perm_active, stream);
}

extern "C" int mobile_topk_rows(const void* rows, int dtype, int R, int E, int k, int* idx_out,
                                int* flags, void* stream) {
  if (R < 0 || E <= 0) { set_error("topk_rows: bad shape R=%d E=%d", R, E); return MOBILE_ERR_INVALID; }
  if (k > E) { set_error("k (%d) exceeds number of experts (%d)", k, E); return MOBILE_ERR_K_EXCEEDS; }
  if (k < 0) { set_error("topk_rows: negative k"); return MOBILE_ERR_INVALID; }
  if (R == 0 || k == 0) return MOBILE_OK;
  const int wpb = 4;
  const size_t smem = sizeof(unsigned long long) * (size_t)wpb * E;
  if (smem > 200 * 1024) { set_error("topk_rows: E=%d too large", E); return MOBILE_ERR_UNSUPPORTED; }
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((R + wpb - 1) / wpb), block(32 * wpb);
  if (dtype == MOBILE_F64) {
    set_smem_once((const void*)topk_rows_kernel<double>, smem);
    topk_rows_kernel<double><<<grid, block, smem, s>>>((const double*)rows, R, E, k, idx_out, flags);
  } else if (dtype == MOBILE_F32) {
    set_smem_once((const void*)topk_rows_kernel<float>, smem);
    topk_rows_kernel<float><<<grid, block, smem, s>>>((const float*)rows, R, E, k, idx_out, flags);
  } else {
    set_error("topk_rows: unsupported dtype %d", dtype);
    return MOBILE_ERR_UNSUPPORTED;
  }
  MOBILE_CHECK_LAUNCH("topk_rows");
  return MOBILE_OK;
}
