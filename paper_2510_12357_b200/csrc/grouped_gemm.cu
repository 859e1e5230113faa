// Grouped expert GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA)
// for prefill / batched decode, where experts see many tokens and the expert
// FFN becomes a dense contraction (SURVEY.md §2.3 `grouped_ffn_sm100`).
//
//   D_e[m, n] = sum_k A[row(e, m), k] * B_e[n, k]        (bf16 x bf16 -> f32)
//
// A is the expert-sorted (permuted) activation matrix (P x K bf16, rows of
// expert e contiguous at offsets[e]..offsets[e+1]); B_e are the expert's
// weight rows (out-major, K-major), addressed through a 3-D TMA map
// (K, N, slot).  Persistent: one CTA per SM walks the 128 x BN output tiles
// (BN = 256, or 128 for N = 128) in a grid stride:
//   warp 0      TMA producer: A and B K-blocks of 64 (128 B, SWIZZLE_128B)
//               into a smem ring that runs across tiles (full/empty mbarriers)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer into one of
//               two TMEM accumulators (tile i+1 accumulates while the
//               epilogue drains tile i), tcgen05.commit frees stages / hands
//               the accumulator to the epilogue
//   warps 2-5   epilogue: tcgen05.ld of the 128 x BN f32 accumulator
//               (warp w reads TMEM lanes 32*(w%4)..), then
//                 SWIGLU: 16-column groups [8 gate | 8 up] -> silu(g)*u, bf16
//                 STORE : f32, row scattered to its pair id (combine input)
//                 ACCUM : f32 out += acc (residual projections: out holds x)
// Tiles are enumerated on the device from the expert offsets (a per-CTA
// prefix table in smem), so no host sync is needed between routing and the
// GEMM.  For decode batches (a few rows per expert) the kernel is a weight
// stream: every B byte is read once, the ring keeps 128-192 KB in flight/SM.
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "umma.cuh"

namespace mobile {

constexpr int kGgBM = 128, kGgBK = 64;
constexpr int kGgThreads = 192;
constexpr int kGgABytes = kGgBM * kGgBK * 2;  // 16 KB
constexpr int kGgMaxActive = 256;

template <int BN>
struct GgCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kBBytes = BN * kGgBK * 2;
  static constexpr int kStageBytes = kGgABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr size_t kSmem = (size_t)kStages * kStageBytes + 1024;
};

enum GgEpi { kGgStoreF32Scatter = 0, kGgSwigluBf16 = 1, kGgStoreBf16 = 2, kGgAccumF32 = 3 };

struct GgArgs {
  CUtensorMap tma_a;       // (K, rows_a)      box (64, 128)
  CUtensorMap tma_b;       // (K, N, slots)    box (64, BN, 1)
  const int* offsets;      // (E+1) row offsets of A per expert; NULL = dense
  const int* active;       // [n, ids] (NULL = dense)
  const int* slot;         // expert -> B slot (NULL = identity / dense expert index)
  const int* row_to_pair;  // permuted row -> output row for STORE scatter (NULL = same row)
  int dense_rows;          // dense: A rows (all experts see rows 0..dense_rows)
  int dense_experts;       // dense: number of B experts (each gets all rows)
  int K, N;
  int epi;
  float* out_f32;          // STORE: out_f32[(row_to_pair[r]) * ldo + n]
  __nv_bfloat16* out_bf16; // SWIGLU / STORE bf16: out[r * ldo + col]
  int ldo;
  int out_expert_stride;   // dense experts: column offset of expert e in the output (elements)
  int ksplit;              // dense mode split-K: K-block ranges per tile (1 = off)
  int nkp;                 // K blocks per split
  float* ws;               // split-K partial tiles (item-major, 128 x BN f32 each)
  unsigned* tickets;       // split-K arrival counter per tile (reset by the reducer)
};

struct GgTile {
  int e, row0, nrows, n0, bslot;
};

// Per-CTA tile table: active expert i owns tiles [base[i], base[i+1]).
struct GgSched {
  int total;
  int na;
  int e[kGgMaxActive], off[kGgMaxActive], n[kGgMaxActive], base[kGgMaxActive + 1];
};

// tile id -> (expert, m-tile, n-tile): experts in active order, then n-tiles,
// m fastest: the CTAs that share a B (weight) tile run together, so an
// expert's weights stream from HBM once however many 128-row m-tiles it has
// (its A rows are small and stay in L2).
template <int BN>
__device__ __forceinline__ GgTile gg_tile(const GgArgs& a, const GgSched& S, int tile) {
  GgTile t;
  const int nt = (a.N + BN - 1) / BN;
  if (!a.offsets) {
    const int mt = (a.dense_rows + kGgBM - 1) / kGgBM;
    const int per = mt * nt;
    const int e = tile / per;
    const int r = tile - e * per;
    t.e = e;
    t.row0 = (r % mt) * kGgBM;  // m fastest: the CTAs sharing a B tile run together (B read once from HBM)
    t.nrows = min(kGgBM, a.dense_rows - t.row0);
    t.n0 = (r / mt) * BN;
    t.bslot = a.slot ? a.slot[e] : e;
    return t;
  }
  int lo = 0, hi = S.na - 1;  // largest i with base[i] <= tile (empty experts own no tiles)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (S.base[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const int r = tile - S.base[lo];
  const int mt = (S.n[lo] + kGgBM - 1) / kGgBM;
  t.e = S.e[lo];
  t.row0 = S.off[lo] + (r % mt) * kGgBM;
  t.nrows = min(kGgBM, S.off[lo] + S.n[lo] - t.row0);
  t.n0 = (r / mt) * BN;
  t.bslot = a.slot ? a.slot[t.e] : t.e;
  return t;
}

// one 16-column chunk of an output row through the epilogue
__device__ __forceinline__ void gg_store(const GgArgs& a, const GgTile& T, int row, int orow, int n, const float (&v)[16]) {
  if (a.epi == kGgSwigluBf16) {
    const int f0 = (n / 16) * 8;  // 8 features: cols 0-7 gate, 8-15 up
    __nv_bfloat16* o = a.out_bf16 + (size_t)row * a.ldo + (size_t)T.e * a.out_expert_stride + f0;
    uint4 pk;
    uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float h0 = silu_f(v[2 * j]) * v[8 + 2 * j];
      const float h1 = silu_f(v[2 * j + 1]) * v[8 + 2 * j + 1];
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(h0, h1);
      pw[j] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    *reinterpret_cast<uint4*>(o) = pk;
  } else if (a.epi == kGgAccumF32) {
    float* o = a.out_f32 + (size_t)row * a.ldo + (size_t)T.e * a.out_expert_stride + n;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      float4 r4 = *reinterpret_cast<const float4*>(o + j);
      r4.x += v[j]; r4.y += v[j + 1]; r4.z += v[j + 2]; r4.w += v[j + 3];
      *reinterpret_cast<float4*>(o + j) = r4;
    }
  } else if (a.epi == kGgStoreF32Scatter) {
    float* o = a.out_f32 + (size_t)orow * a.ldo + (size_t)T.e * a.out_expert_stride + n;
#pragma unroll
    for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  } else {
    __nv_bfloat16* o = a.out_bf16 + (size_t)row * a.ldo + (size_t)T.e * a.out_expert_stride + n;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[j], v[j + 1]);
      *reinterpret_cast<__nv_bfloat162*>(o + j) = b2;
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(kGgThreads, 1) grouped_gemm_kernel(const __grid_constant__ GgArgs a) {
  using Cfg = GgCfg<BN>;
  constexpr int S_ = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ __align__(8) uint64_t full[S_], empty[S_], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ GgSched sched;
  __shared__ int red_last;  // split-K: this CTA reduces the tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 1024-byte aligned stage buffers (SWIZZLE_128B atoms)
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm) + 1023) & ~uintptr_t(1023));

  if (tid == 0) {
    umma::prefetch_tmap(&a.tma_a);
    umma::prefetch_tmap(&a.tma_b);
    for (int s = 0; s < S_; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&tfull[b], 1);
      umma::mbar_init(&tempty[b], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) umma::tmem_alloc(&tmem_base, Cfg::kTmemCols);
  pdl_trigger();
  pdl_wait();
  if (warp == 2) {  // tile table (offsets / active come from the routing kernels)
    const int nt = (a.N + BN - 1) / BN;
    if (!a.offsets) {
      if (lane == 0) sched.total = a.dense_experts * ((a.dense_rows + kGgBM - 1) / kGgBM) * nt;
    } else {
      const int na = min(a.active[0], kGgMaxActive);
      int run = 0;
      for (int i0 = 0; i0 < na; i0 += 32) {
        const int i = i0 + lane;
        int cnt = 0;
        if (i < na) {
          const int e = a.active[1 + i], off = a.offsets[e], n = a.offsets[e + 1] - off;
          sched.e[i] = e;
          sched.off[i] = off;
          sched.n[i] = n;
          cnt = ((n + kGgBM - 1) / kGgBM) * nt;
        }
        int x = cnt;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (i < na) sched.base[i] = run + x - cnt;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) {
        sched.base[na] = run;
        sched.total = run;
        sched.na = na;
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tmem_base;
  const int nk = a.K / kGgBK;
  const int ks = a.ksplit;
  const int total = sched.total * ks;  // work items: (tile, K split), split fastest

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (ring continues across tiles)
      uint32_t g = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        const GgTile T = gg_tile<BN>(a, sched, item / ks);
        const int kb0 = (item % ks) * a.nkp, kb1 = min(nk, kb0 + a.nkp);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = (int)(g % S_);
          if (g >= (uint32_t)S_) umma::mbar_wait(&empty[s], ((g / S_) - 1) & 1);
          uint8_t* sa = base + (size_t)s * Cfg::kStageBytes;
          umma::mbar_expect_tx(&full[s], Cfg::kStageBytes);
          umma::tma_load_2d(sa, &a.tma_a, kb * kGgBK, T.row0, &full[s]);
          umma::tma_load_3d(sa + kGgABytes, &a.tma_b, kb * kGgBK, T.n0, T.bslot, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (one thread for the whole CTA)
      constexpr uint32_t idesc = umma::idesc_bf16_f32(kGgBM, BN);
      uint32_t g = 0;
      int it = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
        const int b = it & 1;
        if (it >= 2) umma::mbar_wait(&tempty[b], ((it >> 1) - 1) & 1);  // epilogue drained this buffer
        umma::fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        const int kb0 = (item % ks) * a.nkp, kb1 = min(nk, kb0 + a.nkp);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = (int)(g % S_);
          umma::mbar_wait(&full[s], (g / S_) & 1);
          umma::fence_after();
          const uint8_t* sa = base + (size_t)s * Cfg::kStageBytes;
          const uint8_t* sb = sa + kGgABytes;
#pragma unroll
          for (int k = 0; k < kGgBK / 16; ++k) {
            // advance the start address by 16 elements (32 B) inside the 128 B swizzle atom
            umma::mma_bf16(d, umma::sdesc_sw128(sa + k * 32), umma::sdesc_sw128(sb + k * 32), idesc,
                           (kb != kb0) || k != 0);
          }
          umma::mma_commit(&empty[s]);  // stage free once these MMAs have read it
        }
        umma::mma_commit(&tfull[b]);  // accumulator b complete
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> global
    const int q = warp & 3;       // TMEM lane quarter this warp may read
    const int r = q * 32 + lane;  // tile row = TMEM lane
    int it = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
      const int b = it & 1;
      const int tile = item / ks;
      const GgTile T = gg_tile<BN>(a, sched, tile);
      umma::mbar_wait(&tfull[b], (it >> 1) & 1);
      umma::fence_after();
      const bool live = r < T.nrows;
      const int row = T.row0 + r;  // row of A (permuted / dense)
      const int orow = a.epi == kGgStoreF32Scatter && live && a.row_to_pair ? a.row_to_pair[row] : row;
      float* wp = ks > 1 ? a.ws + (size_t)item * kGgBM * BN + (size_t)r * BN : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        const int n = T.n0 + c * 16;
        if (n >= a.N) break;  // partial last n-tile (N % 128 == 0): warp-uniform
        float v[16];
        umma::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 16), v);
        if (!live) continue;
        if (wp) {  // split-K partial
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            __stcg(reinterpret_cast<float4*>(wp + c * 16 + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
        } else {
          gg_store(a, T, row, orow, n, v);
        }
      }
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&tempty[b]);  // buffer b may be overwritten
      if (ks > 1) {
        // the last of the tile's ks items sums the partials in split order
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) red_last = atomicAdd(a.tickets + tile, 1u) == (unsigned)(ks - 1);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (red_last) {
          __threadfence();
          // the 128 epilogue threads split the live (row, 16-column chunk)
          // pairs, so every partial load of the reduction is in flight at once
          // (one L2 round trip instead of one per chunk); each output element
          // still sums its ks partials in split order (deterministic)
          const float* w0 = a.ws + (size_t)tile * ks * kGgBM * BN;
          const int nch = min(BN, a.N - T.n0) / 16;
          for (int u = (warp - 2) * 32 + lane; u < T.nrows * nch; u += 128) {
            const int rr = u / nch, c = u - rr * nch;
            const int n = T.n0 + c * 16;
            const int row2 = T.row0 + rr;
            const int orow2 = a.epi == kGgStoreF32Scatter && a.row_to_pair ? a.row_to_pair[row2] : row2;
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            for (int sp = 0; sp < ks; ++sp) {
              const float4* src = reinterpret_cast<const float4*>(w0 + (size_t)sp * kGgBM * BN + (size_t)rr * BN + c * 16);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 f = __ldcg(src + j);
                v[4 * j] += f.x; v[4 * j + 1] += f.y; v[4 * j + 2] += f.z; v[4 * j + 3] += f.w;
              }
            }
            gg_store(a, T, row2, orow2, n, v);
          }
          if (warp == 2 && lane == 0) a.tickets[tile] = 0u;  // reusable by the next launch
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, Cfg::kTmemCols);
  }
}

// activation gather: X[r, :] = bf16(src[row_to_src(r), :])
__global__ void gather_bf16_kernel(const float* __restrict__ src, const int* __restrict__ pairs, int div, int P,
                                   int d, __nv_bfloat16* __restrict__ X) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= P) return;
  const int srow = pairs ? pairs[r] / div : r;
  const float* s = src + (size_t)srow * d;
  __nv_bfloat16* o = X + (size_t)r * d;
  for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2)
    *reinterpret_cast<__nv_bfloat162*>(o + i) = __floats2bfloat162_rn(s[i], s[i + 1]);
}

// X[r, :] = bf16(LN(src[row_to_src(r), :])): the pre-MoE LayerNorm
// (toymoe.py:129-132, 188) with the router kernel's exact reduction (256
// threads, strided per-thread sums, warp butterflies, warp 0 over the warp
// partials: router.cu tile_layer_norm), so the rows equal bf16(h2) of the
// router launch bit for bit.  Lets the shared experts start from the
// residual before the router has run.
constexpr int kGatherLnThreads = 256;
__global__ void __launch_bounds__(kGatherLnThreads) gather_ln_bf16_kernel(const float* __restrict__ src,
                                                                          const int* __restrict__ pairs, int div,
                                                                          int P, int d, __nv_bfloat16* __restrict__ X) {
  __shared__ float red[kGatherLnThreads / 32 + 2];
  constexpr int NW = kGatherLnThreads / 32;
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= P) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* row = src + (size_t)(pairs ? pairs[r] / div : r) * d;
  float s = 0.f;
  for (int i = tid; i < d; i += kGatherLnThreads) s += row[i];
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (warp == 0) {
    float v = lane < NW ? red[lane] : 0.f;
    v = warp_sum(v);
    if (lane == 0) red[NW] = v / (float)d;
  }
  __syncthreads();
  const float mean = red[NW];
  float q = 0.f;
  for (int i = tid; i < d; i += kGatherLnThreads) {
    const float c = row[i] - mean;
    q += c * c;
  }
  q = warp_sum(q);
  __syncthreads();
  if (lane == 0) red[warp] = q;
  __syncthreads();
  if (warp == 0) {
    float v = lane < NW ? red[lane] : 0.f;
    v = warp_sum(v);
    if (lane == 0) red[NW + 1] = v / (float)d;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[NW + 1] + 1e-5f);
  __nv_bfloat16* o = X + (size_t)r * d;
  for (int i = tid; i < d; i += kGatherLnThreads) o[i] = __float2bfloat16_rn((row[i] - mean) * inv);
}

// the same gather from bf16 rows (expert-parallel mailboxes hold bf16 rows)
__global__ void gather_rows_bf16_kernel(const __nv_bfloat16* __restrict__ src, const int* __restrict__ pairs, int div,
                                        int P, int d, __nv_bfloat16* __restrict__ X) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= P) return;
  const int srow = pairs ? pairs[r] / div : r;
  const __nv_bfloat16* s = src + (size_t)srow * d;
  __nv_bfloat16* o = X + (size_t)r * d;
  if ((d & 7) == 0) {
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x)
      reinterpret_cast<uint4*>(o)[i] = reinterpret_cast<const uint4*>(s)[i];
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = s[i];
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                    const cuuint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return MOBILE_ERR_CUDA; }
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return MOBILE_ERR_CUDA; }
  return MOBILE_OK;
}

// split-K workspace: nsm partial tiles of 128 x 256 f32 + one ticket per tile
static float* g_split_ws = nullptr;
static unsigned* g_split_tickets = nullptr;

static bool split_k_disabled() {  // opt-in (MOBILE_GG_SPLITK=1): the one-CTA reduction is L2-latency bound
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MOBILE_GG_SPLITK");
    v = (e && std::strcmp(e, "1") == 0) ? 0 : 1;
  }
  return v == 1;
}

static bool ensure_split_ws(int nsm, cudaStream_t stream) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (g_split_ws) return true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
  void* w = nullptr;
  void* t = nullptr;
  if (cudaMalloc(&w, (size_t)nsm * kGgBM * 256 * sizeof(float)) != cudaSuccess) return false;
  if (cudaMalloc(&t, (size_t)nsm * sizeof(unsigned)) != cudaSuccess || cudaMemset(t, 0, (size_t)nsm * sizeof(unsigned)) != cudaSuccess) {
    cudaFree(w);
    return false;
  }
  cudaDeviceSynchronize();
  g_split_ws = (float*)w;
  g_split_tickets = (unsigned*)t;
  return true;
}

static int gg_narrow_max_rows() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MOBILE_GG_NARROW_ROWS");
    v = e ? std::atoi(e) : 2048;
  }
  return v;
}

}  // namespace mobile

using namespace mobile;

extern "C" int mobile_grouped_gemm(const void* A, int rows_a, int K, const void* B_base, long long b_expert_stride,
                                   int n_slots, int N, const int* offsets, const int* active, const int* slot,
                                   int max_tiles, int dense_rows, int dense_experts, int epi, float* out_f32,
                                   void* out_bf16, int ldo, int out_expert_stride, const int* row_to_pair,
                                   void* stream) {
  if (K <= 0 || K % kGgBK || N <= 0 || N % 128 || rows_a <= 0 || n_slots <= 0) {
    set_error("grouped_gemm: K=%d must be a multiple of 64 and N=%d of 128", K, N);
    return MOBILE_ERR_UNSUPPORTED;
  }
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B_base) & 15) || (b_expert_stride & 15)) {
    set_error("grouped_gemm: operands must be 16-byte aligned");
    return MOBILE_ERR_INVALID;
  }
  // 128 x 256 tiles (partial last n-tile when N % 256 == 128); dense GEMMs with
  // few tiles (decode-batch projections) take 128 x 128 tiles: twice the CTAs
  // streaming B, 6 stages in flight each
  int BN = N % 256 == 0 || N > 256 ? 256 : 128;
  if (!offsets && BN == 256 &&
      dense_experts * ((dense_rows + kGgBM - 1) / kGgBM) * ((N + 255) / 256) < sm_count())
    BN = 128;
  // decode batches (a few rows per expert): 128-wide n-tiles double the tile
  // count, so the last wave of weight streams leaves fewer SMs idle (C4
  // batch 8 / 64 decode passes 5.37 / 7.68 -> 5.12 / 7.43 ms); prefill keeps
  // 256 (its A tiles are re-read once per n-tile)
  if (offsets && BN == 256 && rows_a <= gg_narrow_max_rows()) BN = 128;
  GgArgs a{};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows_a};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {kGgBK, kGgBM};
    if (int st = make_map(&a.tma_a, A, 2, dims, strides, box)) return st;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)n_slots};
    const cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)b_expert_stride};
    const cuuint32_t box[3] = {kGgBK, (cuuint32_t)BN, 1};
    if (int st = make_map(&a.tma_b, B_base, 3, dims, strides, box)) return st;
  }
  a.offsets = offsets;
  a.active = active;
  a.slot = slot;
  a.row_to_pair = row_to_pair;
  a.dense_rows = dense_rows;
  a.dense_experts = dense_experts;
  a.K = K;
  a.N = N;
  a.epi = epi;
  a.out_f32 = out_f32;
  a.out_bf16 = reinterpret_cast<__nv_bfloat16*>(out_bf16);
  a.ldo = ldo;
  a.out_expert_stride = out_expert_stride;
  if (max_tiles <= 0) return MOBILE_OK;
  const int nsm = sm_count();
  // Dense mode with fewer tiles than SMs (the decode-batch projections: 8-24
  // tiles of a weight stream): split K so every SM streams B.  Deterministic:
  // partials land in a library workspace, the tile's last CTA sums them in
  // split order.  The workspace is allocated once (never during a capture;
  // captured graphs keep using it), so launches sharing it must be stream-
  // ordered -- one GEMM at a time per process, as the engines issue them.
  a.ksplit = 1;
  a.nkp = K / kGgBK;
  if (!offsets && !split_k_disabled()) {
    const int nk = K / kGgBK;
    const int tiles = dense_experts * ((dense_rows + kGgBM - 1) / kGgBM) * ((N + BN - 1) / BN);
    int ks = min(nsm / max(tiles, 1), nk / 4);
    if (ks >= 2) {
      const int nkp = (nk + ks - 1) / ks;
      ks = (nk + nkp - 1) / nkp;
      if (ensure_split_ws(nsm, (cudaStream_t)stream)) {
        a.ksplit = ks;
        a.nkp = nkp;
        a.ws = g_split_ws;
        a.tickets = g_split_tickets;
        max_tiles = tiles * ks;
      }
    }
  }
  // persistent: at most one CTA per SM (max_tiles bounds the 128-wide tiles)
  const int grid = max(1, min(max_tiles, nsm));
  if (BN == 256) {
    if (int st = set_smem_once((const void*)grouped_gemm_kernel<256>, GgCfg<256>::kSmem)) return st;
    return launch_pdl(grouped_gemm_kernel<256>, dim3(grid), dim3(kGgThreads), GgCfg<256>::kSmem,
                      (cudaStream_t)stream, 1, "grouped_gemm", a);
  }
  if (int st = set_smem_once((const void*)grouped_gemm_kernel<128>, GgCfg<128>::kSmem)) return st;
  return launch_pdl(grouped_gemm_kernel<128>, dim3(grid), dim3(kGgThreads), GgCfg<128>::kSmem, (cudaStream_t)stream,
                    1, "grouped_gemm", a);
}

extern "C" int mobile_gather_rows_bf16(const void* src, const int* pairs, int div, int P, int d, void* X, void* stream) {
  if (P <= 0) return MOBILE_OK;
  return launch_pdl(gather_rows_bf16_kernel, dim3(P), dim3(256), 0, (cudaStream_t)stream, 1, "gather_rows_bf16",
                    reinterpret_cast<const __nv_bfloat16*>(src), pairs, div > 0 ? div : 1, P, d,
                    reinterpret_cast<__nv_bfloat16*>(X));
}

extern "C" int mobile_gather_ln_bf16(const float* src, const int* pairs, int div, int P, int d, void* X,
                                     void* stream) {
  if (P <= 0) return MOBILE_OK;
  if (d <= 0) { set_error("gather_ln: bad d"); return MOBILE_ERR_INVALID; }
  return launch_pdl(gather_ln_bf16_kernel, dim3(P), dim3(kGatherLnThreads), 0, (cudaStream_t)stream, 1,
                    "gather_ln_bf16", src, pairs, div > 0 ? div : 1, P, d, reinterpret_cast<__nv_bfloat16*>(X));
}

extern "C" int mobile_gather_bf16(const float* src, const int* pairs, int div, int P, int d, void* X, void* stream) {
  if (P <= 0) return MOBILE_OK;
  if (d % 2) { set_error("gather: d must be even"); return MOBILE_ERR_UNSUPPORTED; }
  return launch_pdl(gather_bf16_kernel, dim3(P), dim3(256), 0, (cudaStream_t)stream, 1, "gather_bf16", src, pairs,
                    div > 0 ? div : 1, P, d, reinterpret_cast<__nv_bfloat16*>(X));
}
