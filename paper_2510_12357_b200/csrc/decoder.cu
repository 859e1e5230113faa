// Decode-step kernels around the MoE layer: token embedding + position,
// (LN +) dense GEMV for the attention projections, and single-query
// attention over the KV cache.  They exist so the whole per-token step is
// libmobile kernels reading the position from device memory -- capturable in
// one CUDA graph -- instead of a few hundred framework ops.  Semantics follow
// toymoe.py:171-186 (sinusoidal positions added to the embedding; pre-LN
// attention, scale 1/sqrt(head_dim), softmax, residual).
#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace mobile {

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;

// y[t, r] = (residual ? residual[t, r] : 0) + sum_k xin[t, k] * W[r, k]
// xin = LN(x[t]) if do_ln else x[t].  One pass of TT tokens; warps stream two
// weight rows at a time with no-allocate 16-byte loads.
template <typename W, int TT>
__global__ void __launch_bounds__(kGemvThreads) dense_gemv_kernel(const float* __restrict__ x, int T, int d,
                                                                  int do_ln, const W* __restrict__ w, int N,
                                                                  const float* __restrict__ residual,
                                                                  float* __restrict__ y) {
  extern __shared__ __align__(16) float sh[];
  float* h = sh;  // TT * d
  __shared__ float red[kGemvWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = min(TT, T);
  for (int t = 0; t < nt; ++t) {
    const float* xr = x + (size_t)t * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) h[(size_t)t * d + i] = xr[i];
  }
  __syncthreads();
  if (do_ln) {
    for (int t = 0; t < nt; ++t) {
      float* row = h + (size_t)t * d;
      float s = 0.f;
      for (int i = threadIdx.x; i < d; i += blockDim.x) s += row[i];
      s = warp_sum(s);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      float mean = 0.f;
      for (int i = 0; i < kGemvWarps; ++i) mean += red[i];
      mean /= (float)d;
      __syncthreads();
      float q = 0.f;
      for (int i = threadIdx.x; i < d; i += blockDim.x) { float c = row[i] - mean; q += c * c; }
      q = warp_sum(q);
      if (lane == 0) red[warp] = q;
      __syncthreads();
      float var = 0.f;
      for (int i = 0; i < kGemvWarps; ++i) var += red[i];
      const float inv = 1.0f / sqrtf(var / (float)d + 1e-5f);
      __syncthreads();
      for (int i = threadIdx.x; i < d; i += blockDim.x) row[i] = (row[i] - mean) * inv;
    }
    __syncthreads();
  }
  constexpr int Vn = WVec<W>::N;
  const int nvec = d / Vn;
  const int rows_per_iter = 2 * kGemvWarps;
  for (int r0 = blockIdx.x * rows_per_iter; r0 < N; r0 += gridDim.x * rows_per_iter) {
    const int r = r0 + warp * 2;
    if (r >= N) continue;
    const bool two = r + 1 < N;
    float acc[2][TT];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int t = 0; t < TT; ++t) acc[i][t] = 0.f;
    const W* w0 = w + (size_t)r * d;
    const W* w1 = w0 + d;
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
        for (int t = 0; t < TT; ++t) {
          if (t < nt) {
            const float* hr = h + (size_t)t * d + k0;
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
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          float v = warp_sum(acc[i][t]);
          if (lane == 0) {
            const size_t o = (size_t)t * N + r + i;
            y[o] = residual ? residual[o] + v : v;
          }
        }
      }
    }
  }
}

// Single-query attention over the KV cache for B sequences (one new position
// each, at pos[b]).  qkv (B, 3d) = [q | k | v]; the new k/v rows are written to
// the cache first.  One CTA per (sequence, head), head_dim <= 256.
__global__ void attn_decode_kernel(const float* __restrict__ qkv, float* __restrict__ kc,
                                   float* __restrict__ vc, const int* __restrict__ pos, int d, int H, int Hkv,
                                   int max_len, float* __restrict__ out) {
  extern __shared__ __align__(16) float sc[];  // max_len scores + hd q + hd new k + hd new v
  __shared__ float red[32];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x / H, hh = blockIdx.x % H;
  const int hd = d / H;
  const int p = pos[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (p < 0 || p >= max_len) {  // position outside the cache: poison the output, touch nothing
    for (int e = threadIdx.x; e < d / H; e += blockDim.x) out[(size_t)b * d + hh * (d / H) + e] = __int_as_float(0x7fc00000);
    return;
  }
  float* q = sc + max_len;
  float* knew = q + hd;
  float* vnew = knew + hd;
  // grouped-query attention: query head hh reads key/value head g; the new
  // position's K/V come from this step's qkv row (other query heads of the
  // group run in other CTAs), the group's first head writes them to the cache
  const int grp = H / Hkv, g = hh / grp, kvd = Hkv * hd;
  const float* src = qkv + (size_t)b * (d + 2 * kvd);
  // head-major cache (B, Hkv, max_len, hd)
  const size_t head0 = ((size_t)b * Hkv + g) * max_len;
  float* kr = kc + (head0 + p) * hd;
  float* vr = vc + (head0 + p) * hd;
  for (int e = threadIdx.x; e < hd; e += blockDim.x) {
    q[e] = src[hh * hd + e];
    knew[e] = src[d + g * hd + e];
    vnew[e] = src[d + kvd + g * hd + e];
    if (hh % grp == 0) {
      kr[e] = knew[e];
      vr[e] = vnew[e];
    }
  }
  __syncthreads();
  const float scale = 1.0f / sqrtf((float)hd);
  // scores: one warp per position
  float mx = -INFINITY;
  for (int j = warp; j <= p; j += nw) {
    const float* kj = j == p ? knew : kc + (head0 + j) * hd;
    float s = 0.f;
    for (int e = lane; e < hd; e += 32) s = fmaf(q[e], kj[e], s);
    s = warp_sum(s) * scale;
    if (lane == 0) sc[j] = s;
    mx = fmaxf(mx, s);
  }
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int i = 0; i < nw; ++i) mx = fmaxf(mx, red[i]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j <= p; j += blockDim.x) {
    float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
  for (int i = 0; i < nw; ++i) sum += red[i];
  const float inv = 1.0f / sum;
  for (int e = threadIdx.x; e < hd; e += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < p; ++j) acc = fmaf(sc[j], vc[(head0 + j) * hd + e], acc);
    acc = fmaf(sc[p], vnew[e], acc);
    out[(size_t)b * d + hh * hd + e] = acc * inv;
  }
}

// The same attention, coalesced and vectorised for head_dim 64 / 128 (the
// large-batch decode regime, where the KV cache is the dominant HBM stream):
//  scores  lanes in groups of HD/16, each lane 16 dims (4 x float4) of one
//          position's K row, group-reduced by shuffles; 32*16/HD positions per
//          warp iteration, warps interleaved over positions
//  P.V     lanes in groups of HD/4 (one float4 of the V row each), 128/HD
//          positions per warp iteration; per-warp partial rows reduced over
//          warps in a fixed order
constexpr int kAttnThreads = 256;

// PF (split launches, few (sequence, head) pairs): V rows issued before the
// softmax and in groups of 4, K rows double-buffered -- fewer dependent HBM
// round trips per CTA.  Without PF (B*H >= SMs: many CTAs per SM hide the
// latency) the kernel keeps its registers low for occupancy.
#ifndef MOBILE_ATTN_L2PF
#define MOBILE_ATTN_L2PF 1  // 1: L2 prefetch of the split's K / V rows before the PDL wait
#endif
template <int HD, bool PF>
__global__ void __launch_bounds__(kAttnThreads) attn_decode_vec_kernel(const float* __restrict__ qkv,
                                                                       float* __restrict__ kc, float* __restrict__ vc,
                                                                       const int* __restrict__ pos, int d, int H,
                                                                       int Hkv, int max_len, float* __restrict__ out,
                                                                       int nsplit,
                                                                       float* __restrict__ ws, unsigned* __restrict__ tk) {
  constexpr int NW = kAttnThreads / 32;
  constexpr int LS = HD / 16, PS = 32 / LS;  // score lanes per position, positions per warp step
  constexpr int LV = HD / 4, PV = 32 / LV;   // P.V lanes per position, positions per warp step
  extern __shared__ __align__(16) float sc[];  // this split's scores
  __shared__ __align__(16) float qs[HD], knew[HD], vnew[HD];
  __shared__ __align__(16) float part[NW * PV][HD];
  __shared__ float red[NW];
  __shared__ int last_s;
  pdl_trigger();
#if MOBILE_ATTN_L2PF
  // before the wait on the previous kernel (the QKV projection): start this
  // split's cached K / V rows toward L2.  A hint only -- the rows are read
  // again after the wait, and L2 is the coherence point, so a prefetch from a
  // stale position can cost bandwidth but never change a value.
  // split launches only (few (sequence, head) pairs, batch-1 decode): with
  // many CTAs per SM the rows are read right after anyway and the batched
  // passes measured 4-12% slower with it (C4 B = 64 / 256)
  if (PF && threadIdx.x == 0) {
    const int bh0 = blockIdx.x / nsplit, sp0 = blockIdx.x - bh0 * nsplit;
    const int b0 = bh0 / H, p0 = *(volatile const int*)(pos + b0);
    if (p0 > 0 && p0 < max_len) {
      const int n0 = p0 + 1, ns0 = max(1, min(nsplit, n0 / 32));
      if (sp0 < ns0) {
        const int a0 = (int)((long long)n0 * sp0 / ns0), a1 = min((int)((long long)n0 * (sp0 + 1) / ns0), p0);
        const int g0 = (bh0 % H) / (H / Hkv);
        const size_t off = (((size_t)b0 * Hkv + g0) * max_len + a0) * HD;
        const unsigned bytes = (unsigned)(a1 - a0) * HD * 4u;
        if (a1 > a0) {
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kc + off), "r"(bytes) : "memory");
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vc + off), "r"(bytes) : "memory");
        }
      }
    }
  }
#endif
  pdl_wait();
  const int bh = blockIdx.x / nsplit, sp = blockIdx.x - bh * nsplit;
  const int b = bh / H, hh = bh % H;
  const int p = pos[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (p < 0 || p >= max_len) {  // position outside the cache: poison the output, touch nothing
    if (sp == 0)
      for (int e = threadIdx.x; e < HD; e += blockDim.x) out[(size_t)b * d + hh * HD + e] = __int_as_float(0x7fc00000);
    return;
  }
  // split sp owns positions [j0, j1) of [0, p]; the split holding p writes the new row
  const int n = p + 1;
  // splits actually used at this context length: at least 32 positions each
  // (the launch's nsplit is sized for the cache capacity; early in a long
  // cache most of them would be empty)
  const int ns = max(1, min(nsplit, n / 32));
  if (sp >= ns) return;
  const int j0 = (int)((long long)n * sp / ns), j1 = (int)((long long)n * (sp + 1) / ns);
  // grouped-query attention: query head hh reads key/value head g; position
  // p's K/V come from this step's qkv row (query heads of the group run in
  // other CTAs); the group's first head (its split holding p) writes them
  const int grp = H / Hkv, g = hh / grp, kvd = Hkv * HD;
  const float* src = qkv + (size_t)b * (d + 2 * kvd);
  const size_t head0 = ((size_t)b * Hkv + g) * max_len;  // head-major cache (B, Hkv, max_len, HD)
  for (int e = threadIdx.x; e < HD; e += blockDim.x) {
    qs[e] = src[hh * HD + e];
    knew[e] = src[d + g * HD + e];
    vnew[e] = src[d + kvd + g * HD + e];
    if (j1 == n && hh % grp == 0) {
      kc[(head0 + p) * HD + e] = knew[e];
      vc[(head0 + p) * HD + e] = vnew[e];
    }
  }
  __syncthreads();
  const float scale = 1.0f / sqrtf((float)HD);
  // ---- scores
  const int sg = lane / LS, sl = lane % LS;
  float qv[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 q4 = reinterpret_cast<const float4*>(qs + sl * 16)[i];
    qv[4 * i] = q4.x; qv[4 * i + 1] = q4.y; qv[4 * i + 2] = q4.z; qv[4 * i + 3] = q4.w;
  }
  float mx = -INFINITY;
  // K rows double-buffered: the next step's row is in flight while this one
  // is reduced (long contexts run several steps per split)
  float4 kn[4];
  auto load_k = [&](int j, float4 (&dst)[4]) {
    if (j < j1 && j >= j0 && j != p) {
      const float4* kr = reinterpret_cast<const float4*>(kc + (head0 + j) * HD + sl * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) dst[i] = __ldcs(kr + i);
    }
  };
  if (PF) load_k(j0 + warp * PS + sg, kn);
  for (int jj = j0 + warp * PS; jj < j1; jj += NW * PS) {
    const int j = jj + sg;
    float s = 0.f;
    float4 k4[4];
    if (PF) {
#pragma unroll
      for (int i = 0; i < 4; ++i) k4[i] = kn[i];
      load_k(j + NW * PS, kn);
    } else {
      load_k(j, k4);
    }
    if (j < j1) {
      if (j == p) {
#pragma unroll
        for (int i = 0; i < 4; ++i) k4[i] = reinterpret_cast<const float4*>(knew + sl * 16)[i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        s += qv[4 * i] * k4[i].x + qv[4 * i + 1] * k4[i].y + qv[4 * i + 2] * k4[i].z + qv[4 * i + 3] * k4[i].w;
    }
#pragma unroll
    for (int o = LS / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (j < j1) {
      s *= scale;
      if (sl == 0) sc[j - j0] = s;
      mx = fmaxf(mx, s);
    }
  }
  // the first V rows of this thread's P.V loop are independent of the
  // scores: issue them now so they land while the softmax reduces
  const int vg = lane / LV, vl = lane % LV;
  constexpr int VU = PF ? 4 : 1;  // V rows in flight per thread
  constexpr int VSTEP = NW * PV;
  const int jv0 = j0 + warp * PV + vg;
  float4 vpre[VU];
  if constexpr (PF) {
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      const int j = jv0 + u * VSTEP;
      vpre[u] = j < j1 && j != p ? __ldcs(reinterpret_cast<const float4*>(vc + (head0 + j) * HD) + vl)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NW; ++i) mx = fmaxf(mx, red[i]);
  __syncthreads();
  float sum = 0.f;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const float e = expf(sc[j - j0] - mx);
    sc[j - j0] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) sum += red[i];
  // ---- P.V: groups of VU rows, loads first (the first group was issued
  // before the softmax); same accumulation order as one row at a time
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jb = jv0; jb < j1; jb += VU * VSTEP) {
    float4 v4[VU];
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      const int j = jb + u * VSTEP;
      if (PF && jb == jv0) v4[u] = vpre[u];
      else v4[u] = j < j1 && j != p ? __ldcs(reinterpret_cast<const float4*>(vc + (head0 + j) * HD) + vl)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      if (j == p) v4[u] = reinterpret_cast<const float4*>(vnew)[vl];
    }
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      const int j = jb + u * VSTEP;
      if (j < j1) {
        const float w = sc[j - j0];
        acc.x = fmaf(w, v4[u].x, acc.x); acc.y = fmaf(w, v4[u].y, acc.y);
        acc.z = fmaf(w, v4[u].z, acc.z); acc.w = fmaf(w, v4[u].w, acc.w);
      }
    }
  }
  reinterpret_cast<float4*>(part[warp * PV + vg])[vl] = acc;
  __syncthreads();
  if (ns == 1) {
    const float inv = 1.0f / sum;
    for (int e = threadIdx.x; e < HD; e += blockDim.x) {
      float o = 0.f;
#pragma unroll
      for (int i = 0; i < NW * PV; ++i) o += part[i][e];
      out[(size_t)b * d + hh * HD + e] = o * inv;
    }
    return;
  }
  // ---- split-KV: this split's (m, s, o) partial; the (b, h)'s last split merges in split order
  float* wp = ws + (size_t)blockIdx.x * (HD + 2);
  for (int e = threadIdx.x; e < HD; e += blockDim.x) {
    float o = 0.f;
#pragma unroll
    for (int i = 0; i < NW * PV; ++i) o += part[i][e];
    wp[2 + e] = o;
  }
  if (threadIdx.x == 0) { wp[0] = mx; wp[1] = sum; }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_s = atomicAdd(tk + bh, 1u) == (unsigned)(ns - 1);
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  const float* w0 = ws + (size_t)bh * nsplit * (HD + 2);
  // every split's (m, s) in one round trip (thread q loads split q), then the
  // merge factors in split order from shared memory
  float* ms = sc;  // the scores are consumed: reuse as 2 * ns floats
  for (int q = threadIdx.x; q < ns; q += blockDim.x) {
    const float* w = w0 + (size_t)q * (HD + 2);
    ms[2 * q] = __ldcg(w);
    ms[2 * q + 1] = __ldcg(w + 1);
  }
  __syncthreads();
  float M = -INFINITY;
  for (int q = 0; q < ns; ++q)
    if (ms[2 * q + 1] != 0.f) M = fmaxf(M, ms[2 * q]);
  float S = 0.f;
  for (int q = 0; q < ns; ++q) {
    const float sq = ms[2 * q + 1];
    if (sq != 0.f) S += sq * expf(ms[2 * q] - M);
  }
  const float inv = 1.0f / S;
  for (int e = threadIdx.x; e < HD; e += blockDim.x) {
    float o = 0.f;
#pragma unroll 8
    for (int q = 0; q < ns; ++q) {
      const float sq = ms[2 * q + 1];
      const float ov = __ldcg(w0 + (size_t)q * (HD + 2) + 2 + e);
      if (sq != 0.f) o = fmaf(ov, expf(ms[2 * q] - M), o);
    }
    out[(size_t)b * d + hh * HD + e] = o * inv;
  }
  if (threadIdx.x == 0) tk[bh] = 0u;
}

// x[b] = embed[tok[b]] + pe[pos[b]]  (toymoe.py:172), optionally ln_out = LN(x)
__global__ void embed_kernel(const int* __restrict__ tok, const int* __restrict__ pos,
                             const float* __restrict__ embed, const float* __restrict__ pe, int d,
                             float* __restrict__ x, float* __restrict__ ln_out) {
  __shared__ float red[32];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const float* er = embed + (size_t)tok[b] * d;
  const float* pr = pe + (size_t)pos[b] * d;
  float sum = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = er[i] + pr[i];
    x[(size_t)b * d + i] = v;
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
    const float c = x[(size_t)b * d + i] - mean;
    q += c * c;
  }
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  float var = 0.f;
  for (int w = 0; w < nw; ++w) var += red[w];
  const float inv = 1.0f / sqrtf(var / (float)d + 1e-5f);
  for (int i = threadIdx.x; i < d; i += blockDim.x) ln_out[(size_t)b * d + i] = (x[(size_t)b * d + i] - mean) * inv;
}

__global__ void advance_kernel(int* pos, int B, int* tok, const int* next_tok) {
  pdl_trigger();
  pdl_wait();
  const int b = threadIdx.x;
  if (b < B) {
    pos[b] += 1;
    if (next_tok) tok[b] = next_tok[b];
  }
}

template <typename W>
static int launch_gemv(const float* x, int T, int d, int do_ln, const W* w, int N, const float* res, float* y,
                       cudaStream_t s) {
  const size_t smem = sizeof(float) * (size_t)((T <= 1 ? 1 : T <= 2 ? 2 : T <= 4 ? 4 : 8)) * d;
  const int rows_per_iter = 2 * kGemvWarps;
  int grid = (N + rows_per_iter - 1) / rows_per_iter;
  const int cap = sm_count() * 4;
  if (grid > cap) grid = cap;
#define GEMV_CASE(TTV)                                                                              \
  {                                                                                                 \
    auto k = dense_gemv_kernel<W, TTV>;                                                             \
    set_smem_once((const void*)k, smem);                                                           \
    k<<<grid, kGemvThreads, smem, s>>>(x, T, d, do_ln, w, N, res, y);                               \
  }
  if (T <= 1) GEMV_CASE(1) else if (T <= 2) GEMV_CASE(2) else if (T <= 4) GEMV_CASE(4) else GEMV_CASE(8)
#undef GEMV_CASE
  MOBILE_CHECK_LAUNCH("dense_gemv");
  return MOBILE_OK;
}

}  // namespace mobile

using namespace mobile;

extern "C" int mobile_dense_gemv(const float* x, int T, int d, int do_ln, const void* w, int w_dtype, int N,
                                 const float* residual, float* y, void* stream) {
  if (T < 0 || T > 8 || d <= 0 || N <= 0) { set_error("dense_gemv: bad shape T=%d d=%d N=%d (T <= 8)", T, d, N); return MOBILE_ERR_INVALID; }
  if (T == 0) return MOBILE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (w_dtype == MOBILE_BF16) {
    if (d % 8) { set_error("dense_gemv: d=%d must be a multiple of 8", d); return MOBILE_ERR_UNSUPPORTED; }
    return launch_gemv<__nv_bfloat16>(x, T, d, do_ln, (const __nv_bfloat16*)w, N, residual, y, s);
  }
  if (w_dtype == MOBILE_F32) {
    if (d % 4) { set_error("dense_gemv: d=%d must be a multiple of 4", d); return MOBILE_ERR_UNSUPPORTED; }
    return launch_gemv<float>(x, T, d, do_ln, (const float*)w, N, residual, y, s);
  }
  set_error("dense_gemv: unsupported dtype %d", w_dtype);
  return MOBILE_ERR_UNSUPPORTED;
}

namespace mobile {
// split-KV fan-out when (sequence, head) pairs alone leave SMs idle: splits per (sequence, head): about 2 CTAs per SM over the grid, at most 16,
// at least 32 cached positions each (the launch is sized for the cache
// capacity; the kernel uses only the splits the current context fills).
// Measured per-op little pass, ctx 512: 32 vs 64 positions minimum C3 1875 ->
// 1863 us; 4 CTAs per SM / 32 splits: C5 4024 -> 4141 us.
static int attn_nsplit(int B, int H, int max_len) {
  const int bhn = B * H;
  if (bhn >= sm_count() || max_len < 256) return 1;
  return std::min(std::min(16, (2 * sm_count() + bhn - 1) / bhn), max_len / 32);
}
}  // namespace mobile

extern "C" int mobile_attn_split_ws(int B, int d, int H, int max_len, int* ws_floats, int* n_tickets) {
  if (B <= 0 || d <= 0 || H <= 0 || d % H || max_len <= 0 || !ws_floats || !n_tickets) {
    set_error("attn_split_ws: bad shape");
    return MOBILE_ERR_INVALID;
  }
  const int hd = d / H, ns = (hd == 64 || hd == 128) ? attn_nsplit(B, H, max_len) : 1;
  *ws_floats = ns > 1 ? B * H * ns * (hd + 2) : 0;
  *n_tickets = ns > 1 ? B * H : 0;
  return MOBILE_OK;
}

// ws / tickets: caller-owned split-KV workspace (mobile_attn_split_ws sizes it;
// tickets zeroed once, every launch leaves them zero).  One workspace per
// concurrently running caller (stream / graph): two launches sharing one race.
extern "C" int mobile_attn_decode_ws(const float* qkv, float* k_cache, float* v_cache, const int* pos, int B, int d,
                                     int H, int Hkv, int max_len, float* out, float* ws, unsigned* tickets,
                                     int ws_floats, int n_tickets, void* stream) {
  if (B <= 0 || d <= 0 || H <= 0 || d % H || max_len <= 0 || Hkv <= 0 || H % Hkv) {
    set_error("attn_decode: bad shape");
    return MOBILE_ERR_INVALID;
  }
  const int hd = d / H;
  if ((hd == 64 || hd == 128) && (d & 3) == 0) {
    const size_t vsmem = sizeof(float) * (size_t)max_len;
    if (vsmem > 160 * 1024) { set_error("attn_decode: max_len=%d too long", max_len); return MOBILE_ERR_UNSUPPORTED; }
    int nsplit = attn_nsplit(B, H, max_len);
    const int bhn = B * H;
    if (nsplit > 1 && (!ws || !tickets || ws_floats < bhn * nsplit * (hd + 2) || n_tickets < bhn)) nsplit = 1;
    auto kern = nsplit > 1 ? (hd == 64 ? attn_decode_vec_kernel<64, true> : attn_decode_vec_kernel<128, true>)
                           : (hd == 64 ? attn_decode_vec_kernel<64, false> : attn_decode_vec_kernel<128, false>);
    if (int st = set_smem_once((const void*)kern, vsmem)) return st;
    return launch_pdl(kern, dim3(bhn * nsplit), dim3(kAttnThreads), vsmem, (cudaStream_t)stream, 1, "attn_decode", qkv,
                      k_cache, v_cache, pos, d, H, Hkv, max_len, out, nsplit, nsplit > 1 ? ws : nullptr,
                      nsplit > 1 ? tickets : nullptr);
  }
  const size_t smem = sizeof(float) * ((size_t)max_len + 3 * (d / H));
  if (smem > 200 * 1024) { set_error("attn_decode: max_len=%d too long", max_len); return MOBILE_ERR_UNSUPPORTED; }
  set_smem_once((const void*)attn_decode_kernel, smem);
  return launch_pdl(attn_decode_kernel, dim3(B * H), dim3(128), smem, (cudaStream_t)stream, 1, "attn_decode", qkv,
                    k_cache, v_cache, pos, d, H, Hkv, max_len, out);
}

extern "C" int mobile_attn_decode(const float* qkv, float* k_cache, float* v_cache, const int* pos, int B, int d,
                                  int H, int max_len, float* out, void* stream) {
  return mobile_attn_decode_ws(qkv, k_cache, v_cache, pos, B, d, H, H, max_len, out, nullptr, nullptr, 0, 0, stream);
}

extern "C" int mobile_embed(const int* tok, const int* pos, const float* embed, const float* pe, int B, int d,
                            float* x, float* ln_out, void* stream) {
  if (B <= 0 || d <= 0) { set_error("embed: bad shape"); return MOBILE_ERR_INVALID; }
  return launch_pdl(embed_kernel, dim3(B), dim3(256), 0, (cudaStream_t)stream, 1, "embed", tok, pos, embed, pe, d, x,
                    ln_out);
}

extern "C" int mobile_advance(int* pos, int B, int* tok, const int* next_tok, void* stream) {
  if (B <= 0 || B > 1024) { set_error("advance: bad B"); return MOBILE_ERR_INVALID; }
  return launch_pdl(advance_kernel, dim3(1), dim3(1024), 0, (cudaStream_t)stream, 1, "advance", pos, B, tok,
                    next_tok);
}
