// Bulk-copy (TMA) weight-streaming GEMV engine for batch-1..4 decode.
//
// Every decode-time matrix product on the MoBiLE path is HBM-bound: each
// weight byte is used by 1-4 tokens.  This kernel streams weight tiles into
// shared memory with cp.async.bulk (the Blackwell bulk-copy/TMA engine; SASS
// UBLKCP) on a full/empty mbarrier ring of 6 x 32 KB stages per CTA, one CTA
// per SM, so ~192 KB per SM is in flight with no register cost.  Warp 8 is the
// producer (one lane issues the copies); warps 0-7 consume: warp w owns rows
// {w, w+8} of every 16-row unit, so each output is one warp's dot product and
// the epilogue needs no block barrier (SwiGLU pairs gate row w with up row
// w+8 in the same warp).
//
// Work is a list of UNITS = (group, active expert, block of R output rows).
// A launch can carry several groups (e.g. routed + shared experts), so one
// launch covers a layer's whole gate-up (or down) and the unit count is large
// enough to balance 148 SMs.  Weight rows of a unit are streamed in K chunks
// of 2 KB (R bulk copies per chunk, one per row), accumulators
// live across chunks, and the epilogue runs on the unit's last chunk:
//   STORE  : y = acc (+ residual)
//   RELU   : y = max(acc, 0)                       (toy expert, toymoe.py:203)
//   SWIGLU : 16-row groups [8 gate | 8 up] -> silu(g) * u for 8 features
// Reductions are fixed-order (butterfly within warps, then warp order), so the
// results are deterministic.
#include "common.cuh"

namespace mobile {

constexpr int kSgConsumerWarps = 8;
constexpr int kSgThreads = (kSgConsumerWarps + 1) * 32;  // + 1 producer warp
constexpr int kSgStages = 6;
constexpr int kSgStageBytes = 32 * 1024;
constexpr int kSgRowChunkBytes = 2048;  // bytes of one weight row per K chunk
constexpr int kSgMaxGroups = 4;

enum SgEpi { kEpiStore = 0, kEpiRelu = 1, kEpiSwiglu = 2 };

struct SgGroup {
  const char* w_base;       // weights of expert e at w_base + slot[e] * stride (bytes)
  long long stride;
  const int* slot;          // NULL = identity
  const float* x;           // activation rows (K floats each)
  int x_div;                // activation row = pair / x_div
  const int* offsets;       // (E+1) or NULL (dense: one expert, pairs 0..T-1)
  const int* pairs;
  const int* active;        // [n, ids...] or NULL (dense)
  int dense_T;
  int max_active;
  int K;                    // input dim (weight row length)
  int rows;                 // weight rows per expert
  int R;                    // rows per unit
  int out_dim;              // output features per pair
  float* out;
  const float* residual;    // STORE only, same indexing as out
  int epi;
  int units;                // max_active * (rows / R)
};

struct SgArgs {
  SgGroup g[kSgMaxGroups];
  int n_groups;
  int total_units;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Iterator over this CTA's (unit, token-chunk, k-chunk) items.
template <int TT>
struct SgIter {
  int unit;      // global unit index (strided by gridDim.x)
  int g, a, rb;  // decoded unit
  int e, p0, n;  // expert, first pair index, #pairs of the expert
  int tc, kc;    // token chunk, k chunk
  bool valid;

  __device__ bool decode(const SgArgs& A) {
    int u = unit;
    for (g = 0; g < A.n_groups; ++g) {
      if (u < A.g[g].units) break;
      u -= A.g[g].units;
    }
    if (g >= A.n_groups) return false;
    const SgGroup& G = A.g[g];
    const int upe = G.rows / G.R;
    a = u / upe;
    rb = u - a * upe;
    if (G.active) {
      if (a >= G.active[0]) return false;
      e = G.active[1 + a];
      p0 = G.offsets[e];
      n = G.offsets[e + 1] - p0;
    } else {
      e = 0;
      p0 = 0;
      n = G.dense_T;
    }
    return n > 0;
  }
  __device__ void seek(const SgArgs& A) {  // advance to the first valid unit >= unit
    while (unit < A.total_units && !decode(A)) unit += gridDim.x;
    valid = unit < A.total_units;
    tc = kc = 0;
  }
  __device__ void start(const SgArgs& A) {
    unit = blockIdx.x;
    seek(A);
  }
  __device__ void next(const SgArgs& A, int kc_elems) {
    const SgGroup& G = A.g[g];
    const int nk = (G.K + kc_elems - 1) / kc_elems;
    if (++kc < nk) return;
    kc = 0;
    if (++tc * TT < n) return;
    unit += gridDim.x;
    seek(A);
  }
};

// Issue the bulk copies of one item into a stage.
template <typename W, int TT>
__device__ void sg_issue(const SgArgs& A, const SgIter<TT>& it, char* stage, uint64_t* bar) {
  const SgGroup& G = A.g[it.g];
  const int s = G.slot ? G.slot[it.e] : it.e;
  const char* base = G.w_base + (long long)s * G.stride + (size_t)it.rb * G.R * G.K * sizeof(W);
  constexpr int KC = kSgRowChunkBytes / sizeof(W);
  const int k0 = it.kc * KC;
  const int kn = min(KC, G.K - k0);
  const uint32_t row_bytes = (uint32_t)(kn * sizeof(W));
  mbar_expect_tx(bar, row_bytes * G.R);
  for (int r = 0; r < G.R; ++r)
    bulk_g2s(stage + (size_t)r * row_bytes, base + ((size_t)r * G.K + k0) * sizeof(W), row_bytes, bar);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename W, int TT>
__global__ void __launch_bounds__(kSgThreads, 1) stream_gemv_kernel(const __grid_constant__ SgArgs A) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kSgStages];
  __shared__ __align__(8) uint64_t empty[kSgStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int V = WVec<W>::N;
  constexpr int KC = kSgRowChunkBytes / sizeof(W);

  if (tid == 0) {
    for (int s = 0; s < kSgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSgConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kSgConsumerWarps) {
    // ---------------- producer: one lane streams every item of this CTA
    if (lane == 0) {
      SgIter<TT> prod;
      prod.start(A);
      int stage = 0;
      uint32_t empty_phase = 0;
      for (int i = 0; prod.valid; ++i) {
        if (i >= kSgStages) {
          mbar_wait(&empty[stage], (empty_phase >> stage) & 1u);
          empty_phase ^= 1u << stage;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        sg_issue<W, TT>(A, prod, smem + (size_t)stage * kSgStageBytes, &full[stage]);
        prod.next(A, KC);
        stage = stage + 1 == kSgStages ? 0 : stage + 1;
      }
    }
    return;
  }

  // ---------------- consumers: warp w owns rows {w, w + 8} of each unit
  SgIter<TT> cons;
  cons.start(A);
  uint32_t full_phase = 0;
  int stage = 0;
  float acc[2][TT];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[i][t] = 0.f;

  while (cons.valid) {
    const SgGroup& G = A.g[cons.g];
    const int R = G.R;
    const int k0 = cons.kc * KC;
    const int kn = min(KC, G.K - k0);
    const int nt = min(TT, cons.n - cons.tc * TT);
    const bool has0 = warp < R, has1 = warp + 8 < R;
    int pair[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t)
      pair[t] = t < nt ? (G.active ? G.pairs[cons.p0 + cons.tc * TT + t] : cons.tc * TT + t) : 0;
    mbar_wait(&full[stage], (full_phase >> stage) & 1u);
    full_phase ^= 1u << stage;
    if (has0) {
      const W* row0 = reinterpret_cast<const W*>(smem + (size_t)stage * kSgStageBytes) + (size_t)warp * kn;
      const W* row1 = row0 + (size_t)8 * kn;
      const int nvec = kn / V;
      for (int vi = lane; vi < nvec; vi += 32) {
        float xv[TT][V];
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          if (t < nt) {
            const float4* xp = reinterpret_cast<const float4*>(G.x + (size_t)(pair[t] / G.x_div) * G.K + k0 + vi * V);
#pragma unroll
            for (int q = 0; q < V / 4; ++q) {
              const float4 f = __ldg(xp + q);
              xv[t][4 * q] = f.x; xv[t][4 * q + 1] = f.y; xv[t][4 * q + 2] = f.z; xv[t][4 * q + 3] = f.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q) xv[t][q] = 0.f;
          }
        }
        {
          float f[V];
          WVec<W>::widen(*reinterpret_cast<const uint4*>(row0 + vi * V), f);
#pragma unroll
          for (int t = 0; t < TT; ++t)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[0][t] = fmaf(f[q], xv[t][q], acc[0][t]);
        }
        if (has1) {
          float f[V];
          WVec<W>::widen(*reinterpret_cast<const uint4*>(row1 + vi * V), f);
#pragma unroll
          for (int t = 0; t < TT; ++t)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[1][t] = fmaf(f[q], xv[t][q], acc[1][t]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
    stage = stage + 1 == kSgStages ? 0 : stage + 1;

    if ((cons.kc + 1) * KC >= G.K) {
      // ---------------- warp-local epilogue for (unit, token chunk)
      if (has0) {
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const float s0 = warp_sum(acc[0][t]);
          const float s1 = has1 ? warp_sum(acc[1][t]) : 0.f;
          if (lane == 0 && t < nt) {
            if (G.epi == kEpiSwiglu) {  // row w = gate f, row w+8 = up f
              G.out[(size_t)pair[t] * G.out_dim + cons.rb * 8 + warp] = silu_f(s0) * s1;
            } else {
              const size_t o0 = (size_t)pair[t] * G.out_dim + (size_t)cons.rb * R + warp;
              float v0 = s0, v1 = s1;
              if (G.epi == kEpiRelu) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
              else if (G.residual) { v0 += G.residual[o0]; if (has1) v1 += G.residual[o0 + 8]; }
              G.out[o0] = v0;
              if (has1) G.out[o0 + 8] = v1;
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int t = 0; t < TT; ++t) acc[i][t] = 0.f;
    }
    cons.next(A, KC);
  }
}

template <typename W, int TT>
static int sg_launch(const SgArgs& A, cudaStream_t s) {
  auto k = stream_gemv_kernel<W, TT>;
  const size_t smem = (size_t)kSgStages * kSgStageBytes;
  if (int st = set_smem_once((const void*)k, smem)) return st;
  int grid = sm_count();
  if (A.total_units < grid) grid = A.total_units;
  if (grid <= 0) return MOBILE_OK;
  k<<<grid, kSgThreads, smem, s>>>(A);
  MOBILE_CHECK_LAUNCH("stream_gemv");
  return MOBILE_OK;
}

int sg_dispatch(SgArgs& A, int w_dtype, int max_tok, cudaStream_t s) {
  A.total_units = 0;
  for (int i = 0; i < A.n_groups; ++i) A.total_units += A.g[i].units;
  if (A.total_units == 0) return MOBILE_OK;
  const int TT = max_tok <= 1 ? 1 : max_tok <= 2 ? 2 : 4;
  if (w_dtype == MOBILE_BF16) {
    if (TT == 1) return sg_launch<__nv_bfloat16, 1>(A, s);
    if (TT == 2) return sg_launch<__nv_bfloat16, 2>(A, s);
    return sg_launch<__nv_bfloat16, 4>(A, s);
  }
  if (w_dtype == MOBILE_F32) {
    if (TT == 1) return sg_launch<float, 1>(A, s);
    if (TT == 2) return sg_launch<float, 2>(A, s);
    return sg_launch<float, 4>(A, s);
  }
  set_error("stream_gemv: unsupported dtype %d", w_dtype);
  return MOBILE_ERR_UNSUPPORTED;
}

}  // namespace mobile

using namespace mobile;

// Rows per unit: 16 (SwiGLU needs the whole 8+8 group; 16 rows x 4 KB chunk =
// one 64 KB stage), else the largest power of two <= 16 dividing `rows`.
static int pick_R(int rows, int epi) {
  if (epi == kEpiSwiglu) return rows % 16 == 0 ? 16 : -1;
  int R = 16;
  while (R > 1 && rows % R) R >>= 1;
  return R;
}

static int fill_group(SgGroup& G, const mobile_sg_group* in, int w_dtype) {
  const int V = w_dtype == MOBILE_BF16 ? 8 : 4;
  if (in->K <= 0 || in->rows <= 0 || in->K % V) {
    set_error("stream_gemv: K=%d must be a positive multiple of %d", in->K, V);
    return MOBILE_ERR_UNSUPPORTED;
  }
  G.w_base = (const char*)in->w_base;
  G.stride = in->stride;
  G.slot = in->slot;
  G.x = in->x;
  G.x_div = in->x_div > 0 ? in->x_div : 1;
  G.offsets = in->offsets;
  G.pairs = in->pairs;
  G.active = in->active;
  G.dense_T = in->dense_T;
  G.max_active = in->active ? in->max_active : 1;
  G.K = in->K;
  G.rows = in->rows;
  G.epi = in->epi;
  G.R = pick_R(in->rows, in->epi);
  if (G.R < 1 || in->rows % G.R) {
    set_error("stream_gemv: rows=%d K=%d epi=%d cannot be tiled", in->rows, in->K, in->epi);
    return MOBILE_ERR_UNSUPPORTED;
  }
  G.out_dim = in->epi == kEpiSwiglu ? in->rows / 2 : in->rows;
  G.out = in->out;
  G.residual = in->residual;
  G.units = G.max_active * (in->rows / G.R);
  return MOBILE_OK;
}

extern "C" int mobile_stream_gemv(const mobile_sg_group* groups, int n_groups, int w_dtype, int max_tokens,
                                  void* stream) {
  if (n_groups < 1 || n_groups > kSgMaxGroups) { set_error("stream_gemv: 1..%d groups", kSgMaxGroups); return MOBILE_ERR_INVALID; }
  SgArgs A{};
  A.n_groups = n_groups;
  for (int i = 0; i < n_groups; ++i)
    if (int st = fill_group(A.g[i], &groups[i], w_dtype)) return st;
  return sg_dispatch(A, w_dtype, max_tokens, (cudaStream_t)stream);
}
