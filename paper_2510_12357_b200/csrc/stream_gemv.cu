// Bulk-copy (TMA) weight-streaming GEMV engine for batch-1..4 decode.
//
// Every decode-time matrix product on the MoBiLE path is HBM-bound: each
// weight byte is used by 1-4 tokens.  This kernel streams weights into shared
// memory with cp.async.bulk (the Blackwell bulk-copy engine; SASS UBLKCP) on a
// full/empty mbarrier ring (3 stages at batch 1, 2 above), one CTA per SM, so
// ~200 KB per SM is in flight with no register cost.  A stage holds one 64 KB
// weight tile AND the matching activation slices (bulk-copied too), so the
// consumers' inner loop reads shared memory only.
//
// Weights are row-major.  A pipeline item is a tile of 16 rows x 4 KB of K
// (2048 bf16 / 1024 f32): when a whole row fits the chunk the tile is one
// contiguous bulk copy of up to 64 KB, otherwise 16 row copies.
//
// The last warp is the producer: its 32 lanes run the item iterator in
// lockstep, lane 0 arms the stage's mbarrier and the lanes split a tile's row
// copies (16 rows x 4 KB when rows are longer than the chunk) and activation
// slices.  16 consumer warps: warps w and w + 8 own rows {w, w + 8} of every
// 16-row tile, each over one half of the tile's K chunk (interleaved 16-byte
// vectors); at the end of a row the second half's row sums join the first's
// (fixed order, one named barrier), so each output is a fixed-order dot
// product and every epilogue is warp-local to warp w < 8:
//   STORE  : y = acc (+ residual)
//   RELU   : y = max(acc, 0)                      (toy expert, toymoe.py:203)
//   SWIGLU : tile rows [8 gate | 8 up] -> silu(g_w) * u_w   (extension)
//   HEAD   : logits = acc * scale; online (max, sum-exp, first argmax) per
//            token; CTA partials merged by the last CTA (atomic ticket) into
//            conf = 1 / sum, argmax, fallback = conf <= gamma
//            (toymoe.py:209-210, 273; policy.py:69-79)
// Work is a list of UNITS = (group, active expert, 16-row block); a launch can
// carry several groups (routed + shared experts) so one launch covers a
// layer's whole gate-up (or down); each CTA owns a contiguous unit range.
#include "common.cuh"

namespace mobile {

#ifndef MOBILE_SG_KSPLIT
#define MOBILE_SG_KSPLIT 2  // consumer warps per row pair (each takes 1/KSPLIT of a tile's K chunk)
#endif
constexpr int kSgKSplit = MOBILE_SG_KSPLIT;
constexpr int kSgConsumerWarps = 8 * kSgKSplit;
constexpr int kSgThreads = (kSgConsumerWarps + 1) * 32;  // + 1 producer warp
#ifndef MOBILE_SG_ROW_BYTES
#define MOBILE_SG_ROW_BYTES 4096  // K chunk per tile row (bytes of weight)
#endif
#ifndef MOBILE_SG_WARP_ISSUE
#define MOBILE_SG_WARP_ISSUE 1  // 1: the producer warp's 32 lanes issue a tile's row copies in parallel
#endif
#ifndef MOBILE_SG_STAGES1
#define MOBILE_SG_STAGES1 3       // ring depth at batch 1
#endif
constexpr int kSgTileRows = 16;
constexpr int kSgTileRowBytes = MOBILE_SG_ROW_BYTES;
constexpr int kSgWBytes = kSgTileRows * kSgTileRowBytes;  // weight tile region of a stage
constexpr int kSgMaxGroups = 4;
constexpr int kSgMaxTok = 4;

enum SgEpi { kEpiStore = 0, kEpiRelu = 1, kEpiSwiglu = 2, kEpiHead = 3 };

struct SgGroup {
  const char* w_base;       // tiled weights of expert e at w_base + slot[e] * stride (bytes)
  long long stride;
  const int* slot;          // NULL = identity
  const float* x;           // activation rows (K floats each)
  int x_div;                // activation row = pair / x_div
  const int* offsets;       // (E+1); NULL = dense (one expert, pairs 0..T-1)
  const int* pairs;
  const int* active;        // [n, ids...]
  int dense_T;
  int max_active;
  int K;
  int rows;
  int out_dim;
  float* out;
  const float* residual;
  int epi;
  int prefetch;             // weights + expert lists independent of the previous kernel
  int units;                // max_active * ceil(rows / 16)
};

struct SgHead {             // HEAD epilogue state (one dense group)
  float scale, gamma;
  float* conf;
  int* argmax;
  uint8_t* fallback;
  float* partials;          // gridDim.x * kSgMaxTok * 3
  unsigned* ticket;         // left at 0
};

struct SgArgs {
  SgGroup g[kSgMaxGroups];
  SgHead head;
  int n_groups;
  int total_units;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {  // no arrival
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

template <int TT>
struct SgCfg {
  static constexpr int kStages = TT == 1 ? MOBILE_SG_STAGES1 : 2;
  // TT f32 activation slices of one K chunk (bf16 weights: 2 x the row bytes)
  static constexpr int kXBytes = TT * 2 * kSgTileRowBytes;
  static constexpr int kStageBytes = kSgWBytes + kXBytes;
};

// Iterator over this CTA's (unit, token-chunk, k-chunk) items.  A CTA owns a
// contiguous range of units, i.e. consecutive row blocks of mostly one expert,
// so the expert-level lookups (active list, offsets, slot, pair ids: dependent
// global loads) are cached and re-read only when the expert or token chunk
// changes -- the producer's issue loop is then pure arithmetic.
template <int TT>
struct SgIter {
  int unit, unit_end;
  int g, a, rb, rr;  // group, active slot, row block, rows in block
  int e, p0, n, slot;
  int tc, kc;
  int cg, ca, ctc;   // cache keys
  int pair[TT];
  bool valid;
  bool static_only;  // before the PDL wait: refuse groups that depend on the previous kernel
  bool blocked;

  __device__ bool decode(const SgArgs& A) {
    int u = unit;
    int gg = 0;
    for (; gg < A.n_groups; ++gg) {
      if (u < A.g[gg].units) break;
      u -= A.g[gg].units;
    }
    if (gg >= A.n_groups) return false;
    const SgGroup& G = A.g[gg];
    if (static_only && !G.prefetch) {
      blocked = true;
      return true;  // stop here without touching dependent data
    }
    const int upe = (G.rows + kSgTileRows - 1) / kSgTileRows;
    const int aa = u / upe;
    rb = u - aa * upe;
    rr = min(kSgTileRows, G.rows - rb * kSgTileRows);
    if (gg != cg || aa != ca) {
      cg = gg;
      ca = aa;
      ctc = -1;
      if (G.offsets) {
        if (aa >= G.active[0]) { n = 0; e = 0; p0 = 0; slot = 0; }
        else {
          e = G.active[1 + aa];
          p0 = G.offsets[e];
          n = G.offsets[e + 1] - p0;
          slot = G.slot ? G.slot[e] : e;
        }
      } else {
        e = 0; p0 = 0; n = G.dense_T; slot = 0;
      }
    }
    g = gg;
    a = aa;
    return n > 0;
  }
  __device__ void load_pairs(const SgArgs& A) {
    if (ctc == tc) return;
    ctc = tc;
    const SgGroup& G = A.g[g];
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      const int q = tc * TT + t;
      pair[t] = q < n ? (G.offsets ? G.pairs[p0 + q] : q) : 0;
    }
  }
  __device__ void seek(const SgArgs& A) {
    while (unit < unit_end && !decode(A)) ++unit;
    valid = unit < unit_end && !blocked;
    tc = kc = 0;
    if (valid) load_pairs(A);
  }
  __device__ void start(const SgArgs& A, bool static_only_ = false) {
    unit = (int)(((long long)A.total_units * blockIdx.x) / gridDim.x);
    unit_end = (int)(((long long)A.total_units * (blockIdx.x + 1)) / gridDim.x);
    cg = ca = ctc = -1;
    static_only = static_only_;
    blocked = false;
    seek(A);
  }
  __device__ void next(const SgArgs& A, int kc_elems) {
    const SgGroup& G = A.g[g];
    if (++kc * kc_elems < G.K) return;
    kc = 0;
    if (++tc * TT < n) { load_pairs(A); return; }
    ++unit;
    seek(A);
  }
};

template <typename W, int TT>
__device__ void sg_issue(const SgArgs& A, const SgIter<TT>& it, char* stage, uint64_t* bar, int lane = 0,
                         int nl = 1) {
  constexpr int KC = kSgTileRowBytes / sizeof(W);
  const SgGroup& G = A.g[it.g];
  const int s = it.slot;
  const int k0 = it.kc * KC;
  const int kn = min(KC, G.K - k0);
  const char* rows = G.w_base + (long long)s * G.stride + (size_t)it.rb * kSgTileRows * G.K * sizeof(W);
  const uint32_t wbytes = (uint32_t)(it.rr * kn * sizeof(W));
  const int nt = min(TT, it.n - it.tc * TT);
  const uint32_t xbytes = (uint32_t)(kn * sizeof(float));
  if (lane == 0) mbar_expect_tx(bar, wbytes + nt * xbytes);
  if (nl > 1) __syncwarp();
  if (kn == G.K) {  // whole rows: one contiguous copy
    if (lane == 0) bulk_g2s(stage, rows, wbytes, bar);
  } else {
    const uint32_t rb = (uint32_t)(kn * sizeof(W));
    for (int r = lane; r < it.rr; r += nl)
      bulk_g2s(stage + (size_t)r * rb, rows + ((size_t)r * G.K + k0) * sizeof(W), rb, bar);
  }
  for (int t = nl > 1 ? lane - 16 : 0; t < nt; t += nl)  // activation slices x[row, k0:k0+kn]
    if (t >= 0)
      bulk_g2s(stage + kSgWBytes + (size_t)t * xbytes, G.x + (size_t)(it.pair[t] / G.x_div) * G.K + k0, xbytes, bar);
}

// L2 prefetch of an item's weight tile (no shared memory cost): the producer
// runs this kSgL2Ahead items ahead of its bulk copies so that, under a loaded
// memory system, most bulk copies hit L2 instead of waiting on DRAM.
constexpr int kSgL2Ahead = 0;  // measured: L2 prefetch did not help (kept for experiments)
template <typename W, int TT>
__device__ void sg_prefetch(const SgArgs& A, const SgIter<TT>& it) {
  constexpr int KC = kSgTileRowBytes / sizeof(W);
  const SgGroup& G = A.g[it.g];
  const int k0 = it.kc * KC;
  const int kn = min(KC, G.K - k0);
  const char* rows = G.w_base + (long long)it.slot * G.stride + (size_t)it.rb * kSgTileRows * G.K * sizeof(W);
  if (kn == G.K) bulk_prefetch_l2(rows, (uint32_t)(it.rr * kn * sizeof(W)));
}

__device__ __forceinline__ void online_add(float& m, float& s, int& arg, float l, int idx) {
  if (l > m) {
    s = s * expf(m - l) + 1.0f;
    m = l;
    arg = idx;
  } else {
    s += expf(l - m);
  }
}
__device__ __forceinline__ void online_merge2(float& M, float& S, int& A_, float m, float s, int a) {
  if (s == 0.f) return;
  if (m > M) { S = S * expf(M - m) + s; M = m; A_ = a; }
  else { S += s * expf(m - M); if (m == M && a < A_) A_ = a; }
}

template <typename W, int TT>
__global__ void __launch_bounds__(kSgThreads, 1) stream_gemv_kernel(const __grid_constant__ SgArgs A) {
  constexpr int kSgStages = SgCfg<TT>::kStages;
  constexpr int kSgStageBytes = SgCfg<TT>::kStageBytes;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kSgStages];
  __shared__ __align__(8) uint64_t empty[kSgStages];
  __shared__ float hred[kSgConsumerWarps][kSgMaxTok][3];
  __shared__ float xred[2][8][2][kSgMaxTok];  // K-split partial row sums (double-buffered per epilogue)
  __shared__ bool is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w8 = warp & 7, kh = warp >> 3;  // consumer: row pair (w8, w8 + 8), K part kh
  constexpr int V = WVec<W>::N;
  constexpr int KC = kSgTileRowBytes / sizeof(W);

  if (tid == 0) {
    for (int s = 0; s < kSgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSgConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  pdl_trigger();
  if (warp == kSgConsumerWarps) {
    // ---------------- producer: one lane streams every item of this CTA (or
    // the whole warp in lockstep, lanes splitting each tile's row copies)
    constexpr int NL = MOBILE_SG_WARP_ISSUE ? 32 : 1;
    const int pl = NL > 1 ? lane : 0;
    if (NL > 1 || lane == 0) {
      // phase A (overlaps the previous kernel's tail): weight tiles of static
      // groups (dense / shared experts) for the first stages
      int npre = 0;
      {
        SgIter<TT> pre;
        pre.start(A, /*static_only=*/true);
        while (npre < kSgStages && pre.valid) {
          const SgGroup& G = A.g[pre.g];
          const int k0 = pre.kc * KC, kn = min(KC, G.K - k0);
          const char* rows = G.w_base + (long long)pre.slot * G.stride + (size_t)pre.rb * kSgTileRows * G.K * sizeof(W);
          const uint32_t wbytes = (uint32_t)(pre.rr * kn * sizeof(W));
          if (pl == 0) mbar_expect_tx_only(&full[npre], wbytes);
          if (NL > 1) __syncwarp();
          char* st = smem + (size_t)npre * kSgStageBytes;
          if (kn == G.K) {
            if (pl == 0) bulk_g2s(st, rows, wbytes, &full[npre]);
          } else {
            const uint32_t rbytes = (uint32_t)(kn * sizeof(W));
            for (int r = pl; r < pre.rr; r += NL)
              bulk_g2s(st + (size_t)r * rbytes, rows + ((size_t)r * G.K + k0) * sizeof(W), rbytes, &full[npre]);
          }
          ++npre;
          pre.next(A, KC);
        }
      }
      pdl_wait();  // activations / routing of the previous kernel are now visible
      SgIter<TT> prod;
      prod.start(A);
      SgIter<TT> pf = prod;  // L2-prefetch cursor, kSgStages + kSgL2Ahead items ahead
      for (int j = 0; j < kSgStages && pf.valid; ++j) pf.next(A, KC);
      for (int j = 0; j < kSgL2Ahead && pf.valid; ++j) {
        if (pl == 0) sg_prefetch<W, TT>(A, pf);
        pf.next(A, KC);
      }
      int stage = 0;
      uint32_t empty_phase = 0;
      for (int i = 0; prod.valid; ++i) {
        if (kSgL2Ahead > 0 && i >= kSgStages && pf.valid) {
          if (pl == 0) sg_prefetch<W, TT>(A, pf);
          pf.next(A, KC);
        }
        if (i < npre) {  // weights already in flight: add the activation slices
          const SgGroup& G = A.g[prod.g];
          const int k0 = prod.kc * KC, kn = min(KC, G.K - k0);
          const int nt = min(TT, prod.n - prod.tc * TT);
          const uint32_t xbytes = (uint32_t)(kn * sizeof(float));
          if (pl == 0) mbar_expect_tx(&full[stage], nt * xbytes);
          if (NL > 1) __syncwarp();
          for (int t = pl; t < nt; t += NL)
            bulk_g2s(smem + (size_t)stage * kSgStageBytes + kSgWBytes + (size_t)t * xbytes,
                     G.x + (size_t)(prod.pair[t] / G.x_div) * G.K + k0, xbytes, &full[stage]);
        } else {
          if (i >= kSgStages) {
            mbar_wait(&empty[stage], (empty_phase >> stage) & 1u);
            empty_phase ^= 1u << stage;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
          sg_issue<W, TT>(A, prod, smem + (size_t)stage * kSgStageBytes, &full[stage], pl, NL);
        }
        prod.next(A, KC);
        stage = stage + 1 == kSgStages ? 0 : stage + 1;
      }
    }
    return;
  }

  pdl_wait();
  // ---------------- consumers: warp w owns rows {w, w + 8} of each tile
  SgIter<TT> cons;
  cons.start(A);
  uint32_t full_phase = 0;
  int stage = 0, epi_par = 0;
  float acc[2][TT];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[i][t] = 0.f;
  float hm[TT], hs[TT];
  int ha[TT];
#pragma unroll
  for (int t = 0; t < TT; ++t) { hm[t] = -INFINITY; hs[t] = 0.f; ha[t] = 0x7fffffff; }

  while (cons.valid) {
    const SgGroup& G = A.g[cons.g];
    const int k0 = cons.kc * KC;
    const int kn = min(KC, G.K - k0);
    const int nt = min(TT, cons.n - cons.tc * TT);
    const bool has0 = w8 < cons.rr, has1 = w8 + 8 < cons.rr;
    int pair[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) pair[t] = cons.pair[t];
    mbar_wait(&full[stage], (full_phase >> stage) & 1u);
    full_phase ^= 1u << stage;
    if (has0) {
      const char* st = smem + (size_t)stage * kSgStageBytes;
      const W* row0 = reinterpret_cast<const W*>(st) + (size_t)w8 * kn;
      const W* row1 = row0 + (size_t)8 * kn;
      const float* xs = reinterpret_cast<const float*>(st + kSgWBytes);
      const int nvec = kn / V;
#pragma unroll 4
      for (int vi = lane + 32 * kh; vi < nvec; vi += 32 * kSgKSplit) {
        float f0[V], f1[V];
        WVec<W>::widen(*reinterpret_cast<const uint4*>(row0 + vi * V), f0);
        if (has1) WVec<W>::widen(*reinterpret_cast<const uint4*>(row1 + vi * V), f1);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          if (t < nt) {
            const float4* xp = reinterpret_cast<const float4*>(xs + (size_t)t * kn + vi * V);
#pragma unroll
            for (int q = 0; q < V / 4; ++q) {
              const float4 xq = xp[q];
              acc[0][t] = fmaf(f0[4 * q], xq.x, acc[0][t]);
              acc[0][t] = fmaf(f0[4 * q + 1], xq.y, acc[0][t]);
              acc[0][t] = fmaf(f0[4 * q + 2], xq.z, acc[0][t]);
              acc[0][t] = fmaf(f0[4 * q + 3], xq.w, acc[0][t]);
              if (has1) {
                acc[1][t] = fmaf(f1[4 * q], xq.x, acc[1][t]);
                acc[1][t] = fmaf(f1[4 * q + 1], xq.y, acc[1][t]);
                acc[1][t] = fmaf(f1[4 * q + 2], xq.z, acc[1][t]);
                acc[1][t] = fmaf(f1[4 * q + 3], xq.w, acc[1][t]);
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
    stage = stage + 1 == kSgStages ? 0 : stage + 1;

    if ((cons.kc + 1) * KC >= G.K) {
      // ---------------- warp-local epilogue for (tile, token chunk)
      float s0v[TT], s1v[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        s0v[t] = has0 ? warp_sum(acc[0][t]) : 0.f;
        s1v[t] = has1 ? warp_sum(acc[1][t]) : 0.f;
      }
      if constexpr (kSgKSplit > 1) {  // K part 1's row sums join part 0's (fixed order: part 0 + part 1)
        if (kh == 1 && lane == 0)
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            xred[epi_par][w8][0][t] = s0v[t];
            xred[epi_par][w8][1][t] = s1v[t];
          }
        asm volatile("bar.sync 2, %0;" ::"n"(kSgConsumerWarps * 32));
        if (kh == 0)
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            s0v[t] += xred[epi_par][w8][0][t];
            s1v[t] += xred[epi_par][w8][1][t];
          }
        epi_par ^= 1;
      }
      if (has0 && kh == 0) {
        const int r0 = cons.rb * kSgTileRows + w8;  // output row of acc[0]
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const float s0 = s0v[t];
          const float s1 = s1v[t];
          if (t < nt) {
            if (G.epi == kEpiHead) {
              const float l0 = s0 * A.head.scale, l1 = s1 * A.head.scale;
              if (lane == 0 && G.out) {
                G.out[(size_t)pair[t] * G.out_dim + r0] = l0;
                if (has1) G.out[(size_t)pair[t] * G.out_dim + r0 + 8] = l1;
              }
              online_add(hm[t], hs[t], ha[t], l0, r0);
              if (has1) online_add(hm[t], hs[t], ha[t], l1, r0 + 8);
            } else if (lane == 0) {
              if (G.epi == kEpiSwiglu) {  // row w = gate f, row w + 8 = up f
                G.out[(size_t)pair[t] * G.out_dim + cons.rb * 8 + w8] = silu_f(s0) * s1;
              } else {
                const size_t o0 = (size_t)pair[t] * G.out_dim + r0;
                float v0 = s0, v1 = s1;
                if (G.epi == kEpiRelu) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                else if (G.residual) { v0 += G.residual[o0]; if (has1) v1 += G.residual[o0 + 8]; }
                G.out[o0] = v0;
                if (has1) G.out[o0 + 8] = v1;
              }
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

  if (A.head.conf == nullptr) return;
  // ---------------- HEAD: merge warps (warp order), then CTAs (CTA order)
  const int T = A.g[0].dense_T;
  if (lane == 0)
    for (int t = 0; t < TT; ++t) {
      hred[warp][t][0] = hm[t];
      hred[warp][t][1] = hs[t];
      hred[warp][t][2] = __int_as_float(ha[t]);
    }
  asm volatile("bar.sync 1, %0;" ::"n"(kSgConsumerWarps * 32));
  if (tid < T) {
    float M = -INFINITY, S = 0.f;
    int Ai = 0x7fffffff;
    for (int w = 0; w < kSgConsumerWarps; ++w)
      online_merge2(M, S, Ai, hred[w][tid][0], hred[w][tid][1], __float_as_int(hred[w][tid][2]));
    float* p = A.head.partials + ((size_t)blockIdx.x * kSgMaxTok + tid) * 3;
    p[0] = M;
    p[1] = S;
    p[2] = __int_as_float(Ai);
  }
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"n"(kSgConsumerWarps * 32));
  if (tid == 0) is_last = atomicAdd(A.head.ticket, 1u) == gridDim.x - 1;
  asm volatile("bar.sync 1, %0;" ::"n"(kSgConsumerWarps * 32));
  if (!is_last) return;
  __threadfence();
  if (tid < T) {
    float M = -INFINITY, S = 0.f;
    int Ai = 0x7fffffff;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const volatile float* p = A.head.partials + ((size_t)b * kSgMaxTok + tid) * 3;
      online_merge2(M, S, Ai, p[0], p[1], __float_as_int(p[2]));
    }
    const float conf = 1.0f / S;
    A.head.conf[tid] = conf;
    if (A.head.argmax) A.head.argmax[tid] = Ai;
    if (A.head.fallback) A.head.fallback[tid] = conf <= A.head.gamma ? 1 : 0;
  }
  if (tid == 0) *A.head.ticket = 0u;
}

template <typename W, int TT>
static int sg_launch(const SgArgs& A, cudaStream_t s) {
  auto k = stream_gemv_kernel<W, TT>;
  const size_t smem = (size_t)SgCfg<TT>::kStages * SgCfg<TT>::kStageBytes;
  if (int st = set_smem_once((const void*)k, smem)) return st;
  int grid = sm_count();
  if (A.head.conf == nullptr && A.total_units < grid) grid = A.total_units;
  if (grid <= 0) return MOBILE_OK;
  return launch_pdl(k, dim3(grid), dim3(kSgThreads), smem, s, 1, "stream_gemv", A);
}

static int sg_dispatch(SgArgs& A, int w_dtype, int max_tok, cudaStream_t s) {
  A.total_units = 0;
  for (int i = 0; i < A.n_groups; ++i) A.total_units += A.g[i].units;
  if (A.total_units == 0 && A.head.conf == nullptr) return MOBILE_OK;
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

static int fill_group(SgGroup& G, const mobile_sg_group* in, int w_dtype) {
  const int V = w_dtype == MOBILE_BF16 ? 8 : 4;
  if (in->K <= 0 || in->rows <= 0 || in->K % V) {
    set_error("stream_gemv: K=%d must be a positive multiple of %d", in->K, V);
    return MOBILE_ERR_UNSUPPORTED;
  }
  if (in->epi == kEpiSwiglu && in->rows % kSgTileRows) {
    set_error("stream_gemv: SwiGLU rows=%d must be a multiple of 16", in->rows);
    return MOBILE_ERR_UNSUPPORTED;
  }
  if (!in->offsets && (in->dense_T < 0 || in->dense_T > 64 * 1024)) {
    set_error("stream_gemv: bad dense_T=%d", in->dense_T);
    return MOBILE_ERR_INVALID;
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
  G.max_active = in->offsets ? in->max_active : 1;
  G.K = in->K;
  G.rows = in->rows;
  G.epi = in->epi;
  G.out_dim = in->epi == kEpiSwiglu ? in->rows / 2 : in->rows;
  G.out = in->out;
  G.residual = in->residual;
  G.prefetch = in->prefetch;
  G.units = G.max_active * ((in->rows + kSgTileRows - 1) / kSgTileRows);
  return MOBILE_OK;
}

}  // namespace mobile

using namespace mobile;

extern "C" int mobile_stream_gemv(const mobile_sg_group* groups, int n_groups, int w_dtype, int max_tokens,
                                  void* stream) {
  if (n_groups < 1 || n_groups > kSgMaxGroups) { set_error("stream_gemv: 1..%d groups", kSgMaxGroups); return MOBILE_ERR_INVALID; }
  SgArgs A{};
  A.n_groups = n_groups;
  for (int i = 0; i < n_groups; ++i) {
    if (groups[i].epi == kEpiHead) { set_error("stream_gemv: use mobile_stream_head for the head"); return MOBILE_ERR_INVALID; }
    if (int st = fill_group(A.g[i], &groups[i], w_dtype)) return st;
  }
  return sg_dispatch(A, w_dtype, max_tokens, (cudaStream_t)stream);
}

extern "C" size_t mobile_stream_head_ws_bytes(void) {
  return 256 + sizeof(float) * 3 * kSgMaxTok * (size_t)sm_count();
}

extern "C" int mobile_stream_head(const float* x_ln, int T, int d, const void* w_head, int w_dtype, int V,
                                  float logit_scale, float gamma, float* logits_out, float* conf_out,
                                  int* argmax_out, uint8_t* fallback_out, void* workspace, void* stream) {
  if (T < 1 || T > kSgMaxTok || d <= 0 || V <= 0) { set_error("stream_head: bad shape T=%d (1..4)", T); return MOBILE_ERR_INVALID; }
  SgArgs A{};
  A.n_groups = 1;
  mobile_sg_group in{};
  in.w_base = w_head;
  in.x = x_ln;
  in.x_div = 1;
  in.dense_T = T;
  in.K = d;
  in.rows = V;
  in.out = logits_out;
  in.epi = kEpiHead;
  in.prefetch = 1;
  if (int st = fill_group(A.g[0], &in, w_dtype)) return st;
  A.head.scale = logit_scale;
  A.head.gamma = gamma;
  A.head.conf = conf_out;
  A.head.argmax = argmax_out;
  A.head.fallback = fallback_out;
  A.head.ticket = reinterpret_cast<unsigned*>(workspace);
  A.head.partials = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + 256);
  return sg_dispatch(A, w_dtype, T, (cudaStream_t)stream);
}

