// Persistent decode-pass kernel: one launch runs a whole MoBiLE decode pass
// (or one offload segment of it) for B <= 4 sequences.
//
// Why: at batch 1 every decode matrix is HBM-streamed exactly once and is
// small (8-70 MB, 1-10 us at roofline), so a kernel-per-op step loses most of
// its time to launch ramp, pipeline fill and drain (measured: an isolated
// 8 MB GEMV reaches 32% of HBM, 70 MB 57%, 2 GB 80%).  Here 148 CTAs (one per
// SM) live for the whole pass; a producer warp per CTA streams every weight
// tile the CTA will ever consume through one cp.async.bulk / mbarrier ring,
// running ACROSS phase boundaries: weights of static matrices (attention
// projections, router, shared experts, head) are in flight while the previous
// phase is still computing, so the HBM stream does not drain at every op.
// Phases are separated by grid barriers (an arrival counter in global
// memory); only the data a phase produces (activations, routing) waits.
//
// A pass is a PROGRAM of phases: per layer (toymoe.py:171-207 with a KV cache)
//   qkv     GEMV  x = LN(x_l) [embed (layer 0) / combine of layer l-1 fused
//                 into the input build]; epilogue writes q and the new K/V rows
//   attn    single-query attention, position-split, last-arriver merge
//   o       GEMV  x = att, + residual -> xa
//   router  GEMV  x = LN(xa): router logits (+ sigmoid shared-gate rows)
//                 + shared-expert gate-up (SwiGLU)             (toymoe.py:188-190)
//   [publish]     offload only: CTA 0 writes the layer's active expert list
//   gu      routed gate-up (x = LN(xa)) + shared down; every CTA derives the
//           selection itself from the logits: stable top-k / replay / gate
//           softmax (toymoe.py:193-201) and the stable (expert, pair) permute
//   down    routed down -> Y; the weighted combine + residual + LN is fused
//           into the next layer's input build (toymoe.py:204, 207)
// then the head (toymoe.py:209-210, 273; policy.py:69-79) with an online
// max / sum-exp / first-argmax merge.  The program is a handful of per-layer
// phase TEMPLATES held in the kernel's constant-bank parameter; a phase is
// (template, layer) and every per-layer pointer is base + layer * stride, so
// no descriptor is ever fetched from global memory.  Offloaded passes run the
// same program in L+1 launches cut before each layer's routed experts
// (engine.py:121-169: the host issues the copies in between).
//
// Consumer arithmetic: warp w owns a 256-element K slice of every row of a
// 16-row weight tile (each weight and activation byte leaves shared memory
// once); rows are reduced over lanes by a fixed butterfly and over warps in
// warp order -- fixed-order fp32, no float atomics, deterministic and
// independent of the grid size.
#include "common.cuh"

namespace mobile {
namespace dp {

constexpr int kCW = 8;                      // consumer warps
constexpr int kRW = kCW + 1;                // route warp (early routing; registers come free: 4-warp granules)
constexpr int kThreads = (kCW + 2) * 32;    // + 1 producer warp + 1 route warp
constexpr int kTileRows = 16;
constexpr int kChunk = 4096;                // bytes of K per tile row
constexpr int kWBytes = kTileRows * kChunk; // 64 KB weight tile per stage
constexpr int kMaxB = 4;
constexpr int kMaxPairs = 32;
constexpr int kMaxG = 3;
constexpr int kMaxE = 256;
constexpr int kMaxStages = 3;
constexpr int kMaxGate = 4;                 // shared experts (and sigmoid gates) per layer
constexpr int kMaxTmpl = 9;
constexpr int kAttnPart = 4;  // attention partial layout: [m, s, pad, pad, o[hd]]

enum GroupKind { GK_DENSE = 0, GK_SHARED = 1, GK_ROUTED = 2 };
enum Epi { EP_STORE = 0, EP_RELU = 1, EP_SWIGLU = 2, EP_QKV = 3, EP_LOGITS = 4, EP_HEAD = 5 };
enum XKind { XK_NONE = 0, XK_LN = 1, XK_PLAIN = 2, XK_COMBINE_LN = 3, XK_EMBED_LN = 4, XK_ATTN = 5 };
enum PhaseType { PT_GEMV = 0, PT_ATTN = 1, PT_PUBLISH = 2 };

struct Group {
  const char* w;        // layer-0 matrix (dense) / expert 0 (shared, resident routed) / slot 0 (offload)
  long long w_l;        // bytes per layer
  long long stride;     // bytes between experts
  const int* slot;      // routed: slot table (NULL = identity)
  float* out;
  long long out_l;      // floats per layer
  float* out2;          // EP_LOGITS: rows >= split (shared-gate logits)
  long long out2_l;
  const float* resid;   // EP_STORE: residual added (same indexing as out)
  const float* xg;      // staged activations: row (pair) r at xg + r * K
  int slot_l;           // ints per layer
  int K, rows, kind, epi, n_exp, xstage, units, out_ld, split;
};

struct alignas(16) Tmpl {  // 16-byte multiple: copied to shared memory as int4s
  int type, n_groups, xkind, xkind0, keep_x, end_bar, units, has_routed;
  const float* xsrc;    // XK_LN / XK_PLAIN source; XK_COMBINE_LN residual (xa)
  float* xdst;          // XK_COMBINE_LN / XK_EMBED_LN: where CTA 0 writes the new residual
  Group g[kMaxG];
};

struct Plan {
  Tmpl t[kMaxTmpl];     // [0, ppl): one layer's phases; [ppl]: head
  int ppl, L, n_phases, bpl, upl, router_j;
  int B, d, H, E, k, S, n_gate, gate_norm, reuse_gates, max_len, V, nc_max, TT;
  int hd, npi;           // head dim; K/V positions per ring stage
  int Hkv, grp;          // key/value heads; query heads per key/value head (grouped-query attention)
  int pf_window;         // L2 prefetch distance ahead of the ring, bytes per CTA (0 = off)
  float logit_scale, gamma;
  const int* tok;
  const int* pos;
  const float* embed;
  const float* pe;
  float* kc;
  float* vc;
  float* q;
  float* att;
  float* Y;
  float* Ys;
  float* states;        // (L, B, E) own router logits
  float* extra;         // (L, B, n_gate)
  const float* replay;  // (L, B, E) or NULL
  int* idx_out;         // (L, B, k)
  float* gates_out;     // (L, B, k)
  int* active_out;      // (L, E + 1) or NULL
  float* head_logits;   // (B, V) or NULL
  float* conf;
  int* argmax;
  uint8_t* fallback;
  unsigned* sync;       // [0] barrier, [1] exit, [2] head ticket, [64 + b*H + h] attention tickets
  struct Route* route_pub;  // per layer: the selection computed by the CTA that finished the last router unit
  unsigned* route_sync;     // [l] router units done, [L + l] route published (reset at exit)
  float* attn_part;
  float* head_part;
  int* flags;
  unsigned long long* trace;  // optional: per (phase, CTA) [barrier passed, inputs ready, work done] ns
  // zero-sync offload pass (mobile_dp_run_offload_pass): the kernel publishes
  // each layer's selection to mapped host memory, the host cache driver answers
  // with (slot, ticket) per expert, copies land in the background
  int zs;
  unsigned zs_epoch, zs_prog_base;
  const unsigned* zs_done;     // device: per slot, ticket of the last copy landed
  unsigned* zs_prog;           // device: progress (layers consumed) for slot reuse
  unsigned* zs_prog_h;         // mapped mirror of zs_prog
  int* zs_route_h;             // mapped (L, E + 1) active lists
  int* zs_route_flag_h;        // mapped (L): epoch when published
  const int* zs_slots_h;       // mapped (L, E, 2): slot, ticket
  const int* zs_slots_flag_h;  // mapped (L): epoch when written
  int* zs_slots_d;             // device copy relayed by CTA 0 (only one warp reads host memory)
  int* zs_slots_flag_d;
  int* diag;                  // optional mapped host int[16]: watchdog diagnostics (survive the trap)
  unsigned long long* evt;    // optional event log: per CTA and role (0 producer, 1 consumers) kEvt x {time, code}
};

static_assert(sizeof(Tmpl) % 16 == 0, "templates are copied as int4s (a 3-group template's tail was dropped)");

struct Route {          // one layer's selection + permute, in shared memory (E <= 256)
  int n_active;
  uint8_t act_e[kMaxPairs], act_p0[kMaxPairs], act_n[kMaxPairs];
  uint8_t pairs[kMaxPairs];
  uint8_t idx[kMaxPairs];
  float gates[kMaxPairs];
};

struct StageMeta {      // written by the weight cursor, read by the activation cursor
  const float* xrow[kMaxB];
  int nt, xbytes, needx;
  unsigned tgt;         // barrier count the activations wait for
};

// ------------------------------------------------------------------ primitives
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_tx_only(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(b)), "r"(parity) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes or the hint expires (no issue slots burnt polling)
__device__ __forceinline__ bool mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(su32(b)), "r"(parity), "r"(20000u) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Acquire side of the grid barrier / flags: a relaxed poll observed the
// released value, then an acquire-only fence (PTX 8.6).  Measured on B200: a
// fence with RELEASE semantics (fence.acq_rel, red.release, __threadfence)
// waits for every memory operation the SM has in flight -- including the
// producer's 64 KB bulk copies -- so under the weight stream it costs 1-3 us;
// fence.acquire does not (scripts/barrier_load_bench.cu).
#ifndef MOBILE_DP_ACQ_FENCE
#define MOBILE_DP_ACQ_FENCE 1
#endif
__device__ __forceinline__ void fence_acquire() {
#if MOBILE_DP_ACQ_FENCE
  asm volatile("fence.acquire.gpu;" ::: "memory");
#else
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kCW * 32) : "memory"); }

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
#if MOBILE_DP_ARRIVE_RELAXED  // timing experiment only: no release ordering
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}

// Sum of 16 per-lane row partials over the 32 lanes of a warp: recursive
// halving (16 + 8 + 4 + 2 + 1 shuffles); lanes 2i and 2i+1 end with row i.
template <int TT>
__device__ __forceinline__ float reduce_rows16(float (&a)[16][TT], int t, int lane) {
  float v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = a[r][t];
#pragma unroll
  for (int h = 8, off = 16; h >= 1; h >>= 1, off >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int r = 0; r < h; ++r) {
      const float send = hi ? v[r] : v[r + h];
      const float keep = hi ? v[r + h] : v[r];
      v[r] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

constexpr int kEvt = 1024;
constexpr int kTraceSlots = 6;
enum EvtCode { EV_W = 1, EV_X = 2, EV_FULL = 3, EV_UNIT = 4, EV_ARRIVE = 5, EV_PASS = 6, EV_READY = 7, EV_ROUTE = 8, EV_WAIT = 9, EV_RED = 10 };
__device__ __forceinline__ void log_evt(const unsigned long long* base_, int role, int& n, int code, int p, int item) {
  unsigned long long* base = const_cast<unsigned long long*>(base_);
  if (base == nullptr || n >= kEvt) return;
  unsigned long long* e = base + (((size_t)blockIdx.x * 2 + role) * kEvt + n) * 2;
  e[0] = gtimer();
  e[1] = ((unsigned long long)code << 56) | ((unsigned long long)(p & 0xffff) << 32) | (unsigned)item;
  ++n;
}

constexpr unsigned long long kWatchdogNs = 4000000000ull;  // 4 s: a stuck pass traps instead of hanging

// ------------------------------------------------------------------ program
// phase p -> (template j, layer l); the head is the last phase
__device__ __forceinline__ void phase_jl(const Plan& P, int p, int& j, int& l) {
  if (p == P.n_phases - 1) { j = P.ppl; l = P.L; }
  else { l = p / P.ppl; j = p - l * P.ppl; }
}
// end barriers in phases [0, p]
__device__ __forceinline__ int bar_cum(const Plan& P, int p) {
  if (p < 0) return 0;
  int j, l;
  phase_jl(P, p, j, l);
  int n = l * P.bpl;
  if (j < P.ppl)
    for (int i = 0; i <= j; ++i) n += P.t[i].end_bar;
  return n;
}
// the latest phase before p with an end barrier (-1: none)
__device__ __forceinline__ int dep_of(const Plan& P, int p) {
  for (int q = p - 1; q >= 0; --q) {
    int j, l;
    phase_jl(P, q, j, l);
    if (P.t[j].end_bar) return q;
  }
  return -1;
}
// barrier count (x grid) after which phase q's outputs are visible, within a launch from `first`
__device__ __forceinline__ unsigned bar_target(const Plan& P, int q, int first) {
  if (q < first) return 0u;
  return (unsigned)(bar_cum(P, q) - bar_cum(P, first - 1)) * gridDim.x;
}
__device__ __forceinline__ int rot_of(const Plan& P, int j, int l) {
  long long c = (long long)l * P.upl;
  if (j < P.ppl)
    for (int i = 0; i < j; ++i) c += P.t[i].units;
  return (int)(c % gridDim.x);
}
__device__ __forceinline__ Group grp_t(const Group& G0, int l) {
  Group G = G0;
  G.w += (long long)l * G.w_l;
  if (G.slot) G.slot += (size_t)l * G.slot_l;
  if (G.out) G.out += (size_t)l * G.out_l;
  if (G.out2) G.out2 += (size_t)l * G.out2_l;
  return G;
}

__device__ void spin_until(const Plan& P, unsigned target, int p = -1, unsigned long long* tr = nullptr) {
  if (target == 0u) return;
  if (ld_relaxed(P.sync) < target) {
    const unsigned long long t0 = gtimer();
    while (ld_relaxed(P.sync) < target) {
      __nanosleep(64);
      if (gtimer() - t0 > kWatchdogNs) {
        atomicOr(P.flags, 4);
        if (P.diag && atomicCAS(P.diag, 0, 2) == 0) {
          P.diag[1] = blockIdx.x; P.diag[2] = p; P.diag[3] = (int)target; P.diag[4] = (int)ld_relaxed(P.sync);
          __threadfence_system();
        }
        __trap();
      }
    }
  }
  if (tr) tr[0] = gtimer();
  fence_acquire();
  if (tr) tr[1] = gtimer();
}

// ------------------------------------------------------------------ routing
// One warp: stable top-k (toymoe.py:80-88 order: value desc, index asc,
// -0.0 == +0.0), replay (toymoe.py:194-200), gate softmax in selection order
// (toymoe.py:201) or HF softmax-over-all, then the deterministic permute of
// the B*k (token, slot) pairs sorted by (expert, pair) (permute.cu contract).
// Ranks are computed by all-pairs comparison (independent broadcasts, no
// dependent shuffle chains): expert e is selected at position rank(e) < k.
template <int kPer>
__device__ __forceinline__ void compute_route_k(const Plan& P, int l, Route& R, bool publish) {
  const int lane = threadIdx.x & 31;
  const int E = P.E, k = P.k, B = P.B;
  bool bad = false;
  int e_me = 0x7fff;  // lane q < B*k: expert of pair q (token q / k, selection slot q % k)
  float g_me = 0.f;   // its normalised gate
  for (int b = 0; b < B; ++b) {
    const float* own = P.states + ((size_t)l * B + b) * E;
    const float* rep = P.replay ? P.replay + ((size_t)l * B + b) * E : nullptr;
    const float* sel_src = rep ? rep : own;
    const float* gate_src = (rep && P.reuse_gates) ? rep : own;
    unsigned long long cand[kPer];  // (order key, ~index): max wins, ties -> lower index
    float gv[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane + 32 * i;
      const float v = e < E ? __ldcg(sel_src + e) : 0.f;
      gv[i] = e < E ? (gate_src == sel_src ? v : __ldcg(gate_src + e)) : -INFINITY;
      bad |= e < E && !isfinite(v);
      cand[i] = e < E ? topk_key(v, e) : 0ull;
    }
    // k rounds of a warp arg-max (value desc, index asc, -0.0 == +0.0)
    int sel = 0x7fff;
    float gsel = 0.f;
#pragma unroll 1
    for (int r = 0; r < k; ++r) {
      unsigned long long best = cand[0];
#pragma unroll
      for (int i = 1; i < kPer; ++i) best = cand[i] > best ? cand[i] : best;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        best = ob > best ? ob : best;
      }
      const int e = (int)(0xFFFFFFFFu - (uint32_t)best);
      float g = 0.f;
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (cand[i] == best) { cand[i] = 0ull; g = gv[i]; }
      g = __shfl_sync(0xffffffffu, g, e & 31);  // the owner lane's gate logit
      if (lane == r) { sel = e; gsel = g; }
    }
    // gate normalisation (toymoe.py:201 softmax over the selection, summed in
    // selection order; or HF softmax over all experts)
    float gn;
    if (P.gate_norm == MOBILE_GATE_SELECTED_SOFTMAX) {
      float m = -INFINITY;
#pragma unroll 1
      for (int j = 0; j < k; ++j) m = fmaxf(m, __shfl_sync(0xffffffffu, gsel, j));
      float ssum = 0.f;
#pragma unroll 1
      for (int j = 0; j < k; ++j) ssum += expf(__shfl_sync(0xffffffffu, gsel, j) - m);
      gn = expf(gsel - m) / ssum;
    } else {
      float mall = -INFINITY;
#pragma unroll
      for (int i = 0; i < kPer; ++i) mall = fmaxf(mall, gv[i]);
      mall = warp_max(mall);
      float zall = 0.f;
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (lane + 32 * i < E) zall += expf(gv[i] - mall);
      zall = warp_sum(zall);
      gn = expf(gsel - mall) / zall;
    }
    // token b's k pairs live in lanes b*k .. b*k+k-1
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
      const int ej = __shfl_sync(0xffffffffu, sel, j);
      const float gj = __shfl_sync(0xffffffffu, gn, j);
      if (lane == b * k + j) { e_me = ej; g_me = gj; }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(P.flags, 1);
  // permute: pairs sorted by (expert, pair); active experts in ascending order
  const int NP = B * k;
  int pos = 0, first = 0, cnt = 0, a_me = 0;
  if (lane < NP) first = 1;
#pragma unroll 1
  for (int q = 0; q < NP; ++q) {
    const int eq = __shfl_sync(0xffffffffu, e_me, q);
    pos += (eq < e_me || (eq == e_me && q < lane)) ? 1 : 0;
    cnt += eq == e_me ? 1 : 0;
    if (eq == e_me && q < lane) first = 0;
  }
  if (lane >= NP) first = 0;
  const unsigned fm = __ballot_sync(0xffffffffu, first);
#pragma unroll 1
  for (int q = 0; q < NP; ++q) {  // active index = distinct experts below mine
    const int eq = __shfl_sync(0xffffffffu, e_me, q);
    a_me += (((fm >> q) & 1u) && eq < e_me) ? 1 : 0;
  }
  if (lane < NP) {
    R.idx[lane] = (uint8_t)e_me;
    R.gates[lane] = g_me;
    R.pairs[pos] = (uint8_t)lane;
    if (first) {
      R.act_e[a_me] = (uint8_t)e_me;
      R.act_p0[a_me] = (uint8_t)(pos);
      R.act_n[a_me] = (uint8_t)cnt;
    }
  }
  const int nact = __popc(fm);
  if (lane == 0) R.n_active = nact;
  __syncwarp();
  if (publish) {
    for (int i = lane; i < NP; i += 32) {
      P.idx_out[(size_t)l * NP + i] = R.idx[i];
      P.gates_out[(size_t)l * NP + i] = R.gates[i];
    }
    if (P.active_out) {
      int* ao = P.active_out + (size_t)l * (E + 1);
      if (lane == 0) ao[0] = nact;
      if (lane < nact) ao[1 + lane] = R.act_e[lane];
    }
  }
}

__device__ __forceinline__ void compute_route(const Plan& P, int l, Route& R, bool publish) {
  if (P.E <= 64) compute_route_k<2>(P, l, R, publish);
  else compute_route_k<8>(P, l, R, publish);
}

// Early routing: the warp that writes the last router unit's logits computes
// the layer's selection once (while the rest of the router phase -- the shared
// gate-up -- is still streaming), publishes it to global memory and releases a
// flag; every CTA copies it instead of recomputing it after the barrier.  Only
// within one launch (the flags are reset at exit): a phase that routes a layer
// whose router phase ran in an earlier launch computes the route itself.
__device__ __forceinline__ bool route_early(const Plan& P, int l, int first) {
  return P.route_pub != nullptr && l * P.ppl + P.router_j >= first;
}
__device__ __forceinline__ bool route_ready(const Plan& P, int l) {  // lane 0
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(P.route_sync + P.L + l) : "memory");
  return v != 0;
}
// selection -> mapped host memory, then the flag (engine.py:137: the demand requests of the layer)
__device__ __forceinline__ void publish_host(const Plan& P, int l, const Route& R) {  // one warp
  const int lane = threadIdx.x & 31;
  int* r = P.zs_route_h + (size_t)l * (P.E + 1);
  if (lane == 0) r[0] = R.n_active;
  if (lane < R.n_active) r[1 + lane] = R.act_e[lane];
  __threadfence_system();
  __syncwarp();
  if (lane == 0)
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(P.zs_route_flag_h + l), "r"((int)P.zs_epoch) : "memory");
}
__device__ __forceinline__ void route_copy(const Plan& P, int l, Route& R) {  // one warp, flag observed
  const int lane = threadIdx.x & 31;
  const int* src = reinterpret_cast<const int*>(P.route_pub + l);
  int* dst = reinterpret_cast<int*>(&R);
  for (int i = lane; i < (int)(sizeof(Route) / 4); i += 32) dst[i] = __ldcg(src + i);
  __syncwarp();
}

// ------------------------------------------------------------------ work items
// Units of a GEMV phase: (group, expert slot a, 16-row block).  CTA c owns the
// units u with (u + rot) % G == c; an item is (unit, K chunk).
struct Item {           // everything the producer and the consumers need about one unit
  int g, a, rb, rr, nkc, n;
  int routed;
  int zslot, tkt;             // zero-sync: slot and copy ticket of a routed unit
  int attn, b, h, c, p0, np;  // attention unit: sequence, head, chunk of old positions [p0, p0 + np)
  int K, rows, epi, xstage, out_ld, split;
  const char* wrow;     // first byte of the tile's rows (chunk 0)
  const float* xg;
  float* out;
  float* out2;
  const float* resid;
  int kind;
};
// output pair / token of token slot t of a unit (no per-unit arrays: they
// would be indexed dynamically in the epilogue and land in local memory)
__device__ __forceinline__ int unit_pair(const Plan& P, const Item& it, const Route& R, int t) {
  if (it.kind == GK_ROUTED) return R.pairs[R.act_p0[it.a] + t];
  if (it.kind == GK_SHARED) return t * P.S + it.a;
  return t;
}
__device__ __forceinline__ int unit_token(const Plan& P, const Item& it, const Route& R, int t) {
  return it.kind == GK_ROUTED ? R.pairs[R.act_p0[it.a] + t] / P.k : t;
}

// decode unit u of (template j, layer l); false = no work (inactive routed slot)
template <typename W>
__device__ __forceinline__ bool decode_unit(const Plan& P, const Tmpl& T, int l, int u, const Route& R, Item& it,
                                            bool zs = false, int zs_slot = 0, int zs_tkt = 0) {
  int uu = u, g = 0;
  for (; g < T.n_groups - 1; ++g) {
    if (uu < T.g[g].units) break;
    uu -= T.g[g].units;
  }
  const Group G = grp_t(T.g[g], l);
  const int upe = (G.rows + kTileRows - 1) / kTileRows;
  const int a = uu / upe;
  it.g = g;
  it.a = a;
  it.rb = uu - a * upe;
  it.rr = min(kTileRows, G.rows - it.rb * kTileRows);
  it.nkc = (G.K * (int)sizeof(W) + kChunk - 1) / kChunk;
  const char* base;
  if (G.kind == GK_ROUTED) {
    if (a >= R.n_active) return false;
    const int e = R.act_e[a];
    int s = G.slot ? G.slot[e] : e;
    if (zs) {  // warp-uniform: lane a holds active expert a's (slot, ticket)
      s = __shfl_sync(0xffffffffu, zs_slot, a & 31);
      it.tkt = __shfl_sync(0xffffffffu, zs_tkt, a & 31);
      it.zslot = s;
    }
    base = G.w + (long long)s * G.stride;
    it.n = R.act_n[a];
  } else if (G.kind == GK_SHARED) {
    base = G.w + (long long)a * G.stride;
    it.n = P.B;
  } else {
    base = G.w;
    it.n = P.B;
  }
  it.wrow = base + (size_t)it.rb * kTileRows * G.K * sizeof(W);
  it.attn = 0;
  it.routed = G.kind == GK_ROUTED;
  it.kind = G.kind;
  it.K = G.K; it.rows = G.rows; it.epi = G.epi; it.xstage = G.xstage; it.out_ld = G.out_ld; it.split = G.split;
  it.xg = G.xg; it.out = G.out; it.out2 = G.out2; it.resid = G.resid;
  return true;
}
// Attention units: (sequence b, head h, chunk c) over the positions [0, pos)
// already in the KV cache; the new position's K/V (written by this pass's
// qkv phase) is added by the last chunk.  nc chunks per head, B*H*nc <= grid.
__device__ __forceinline__ int attn_nc(const Plan& P, const int* spos) {
  int ctx = 1;
  for (int b = 0; b < P.B; ++b) ctx = max(ctx, spos[b] + 1);
  return max(1, min(min((int)gridDim.x / (P.B * P.H), P.nc_max), (ctx + 7) / 8));
}
__device__ __forceinline__ void decode_attn(const Plan& P, int u, int nc, const int* spos, Item& it) {
  it.attn = 1;
  it.routed = 0;
  it.b = u / (P.H * nc);
  const int r = u - it.b * P.H * nc;
  it.h = r / nc;
  it.c = r - it.h * nc;
  const int old = spos[it.b];
  it.p0 = (int)((long long)old * it.c / nc);
  it.np = (int)((long long)old * (it.c + 1) / nc) - it.p0;
  it.nkc = (it.np + P.npi - 1) / P.npi;
}

__device__ __forceinline__ int group_of_unit(const Tmpl& T, int u) {
  int g = 0;
  for (; g < T.n_groups - 1; ++g) {
    if (u < T.g[g].units) break;
    u -= T.g[g].units;
  }
  return g;
}

// ------------------------------------------------------------------ x loads
// Consumers build the phase's activation rows in shared memory (xbuf, B x K).
__device__ void block_ln_rows(float* x, int B, int d, float* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = 0; b < B; ++b) {
    float* row = x + (size_t)b * d;
    float s = 0.f;
    for (int i = tid; i < d; i += kCW * 32) s += row[i];
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    cbar();
    float mean = 0.f;
    for (int w = 0; w < kCW; ++w) mean += red[w];
    mean /= (float)d;
    cbar();
    float q = 0.f;
    for (int i = tid; i < d; i += kCW * 32) {
      const float c = row[i] - mean;
      q += c * c;
    }
    q = warp_sum(q);
    if (lane == 0) red[warp] = q;
    cbar();
    float var = 0.f;
    for (int w = 0; w < kCW; ++w) var += red[w];
    const float inv = 1.0f / sqrtf(var / (float)d + 1e-5f);
    for (int i = tid; i < d; i += kCW * 32) row[i] = (row[i] - mean) * inv;
    cbar();
  }
}

__device__ void load_x(const Plan& P, int xkind, const float* xsrc, float* xdst, int combine_layer, float* xbuf, float* red,
                       const Route& R, const int* spos) {
  const int tid = threadIdx.x, B = P.B, d = P.d, nv = d / 4;
  const bool writer = blockIdx.x == 0;
  float4* xb4 = reinterpret_cast<float4*>(xbuf);
  if (xkind == XK_LN || xkind == XK_PLAIN) {
    const float4* src = reinterpret_cast<const float4*>(xsrc);
    float4 v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = tid + c * kCW * 32;
      if (i < B * nv) v[c] = __ldcg(src + i);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = tid + c * kCW * 32;
      if (i < B * nv) xb4[i] = v[c];
    }
    for (int i = tid + 4 * kCW * 32; i < B * nv; i += kCW * 32) xb4[i] = __ldcg(src + i);
    cbar();
    if (xkind == XK_LN) block_ln_rows(xbuf, B, d, red);
  } else if (xkind == XK_ATTN) {
    // att[b, h*hd + e] = merge of the head's chunk partials (chunk order): one
    // warp per (b, h); lane c holds chunk c's (m, s); two parallel round trips
    const int hd = P.hd, nc = attn_nc(P, spos), lane = tid & 31, warp = tid >> 5;
    for (int bh = warp; bh < B * P.H; bh += kCW) {
      const float* base = P.attn_part + (size_t)bh * P.nc_max * (hd + kAttnPart);
      float mc = -INFINITY, sc = 0.f;
      if (lane < nc) {
        const float2 ms = __ldcg(reinterpret_cast<const float2*>(base + (size_t)lane * (hd + kAttnPart)));
        mc = ms.x;
        sc = ms.y;
      }
      const float M = warp_max(sc != 0.f ? mc : -INFINITY);
      const float f = sc != 0.f ? expf(mc - M) : 0.f;
      float S = 0.f;
      for (int c = 0; c < nc; ++c) S += __shfl_sync(0xffffffffu, sc * f, c);
      const float inv = 1.0f / S;
      const int b = bh / P.H, h = bh - b * P.H;
      for (int e0 = 0; e0 < hd; e0 += 128) {  // warp-uniform trip count (shuffles below)
        const int e = e0 + lane * 4;
        const bool act = e < hd;
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c0 = 0; c0 < nc; c0 += 8) {
          float4 o4[8];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (act && c0 + c < nc)
              o4[c] = __ldcg(reinterpret_cast<const float4*>(base + (size_t)(c0 + c) * (hd + kAttnPart) + kAttnPart + e));
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float fc = __shfl_sync(0xffffffffu, f, (c0 + c) & 31);
            if (act && c0 + c < nc && fc != 0.f) {
              O.x = fmaf(o4[c].x, fc, O.x); O.y = fmaf(o4[c].y, fc, O.y);
              O.z = fmaf(o4[c].z, fc, O.z); O.w = fmaf(o4[c].w, fc, O.w);
            }
          }
        }
        if (act) xb4[((size_t)b * d + h * hd + e) / 4] = make_float4(O.x * inv, O.y * inv, O.z * inv, O.w * inv);
      }
    }
    cbar();
  } else if (xkind == XK_EMBED_LN) {  // x = embed[tok] + pe[pos]   (toymoe.py:172)
    for (int b = 0; b < B; ++b) {
      const float4* er = reinterpret_cast<const float4*>(P.embed + (size_t)P.tok[b] * d);
      const float4* pr = reinterpret_cast<const float4*>(P.pe + (size_t)spos[b] * d);
      float4* xd = reinterpret_cast<float4*>(xdst + (size_t)b * d);
      for (int i = tid; i < nv; i += kCW * 32) {
        const float4 e = er[i], q = pr[i];
        const float4 v = make_float4(e.x + q.x, e.y + q.y, e.z + q.z, e.w + q.w);
        xb4[(size_t)b * nv + i] = v;
        if (writer) xd[i] = v;
      }
    }
    cbar();
    block_ln_rows(xbuf, B, d, red);
  } else if (xkind == XK_COMBINE_LN) {
    // x_out = xa + sum_j g_j Y_j (selection order) + sum_s sigma_s Ys_s   (toymoe.py:204, 207)
    // Every thread loads the shared-gate logits it needs together with the
    // source rows of its column (no separate round trip + CTA barrier for the
    // gates: a dependent L2 load costs ~1 us under the weight stream).
    const int l = combine_layer, k = P.k, S = P.S;
    const float4* Y4 = reinterpret_cast<const float4*>(P.Y);
    const float4* Ys4 = reinterpret_cast<const float4*>(P.Ys);
    const float4* X4 = reinterpret_cast<const float4*>(xsrc);
    float4* xd = reinterpret_cast<float4*>(xdst);
    constexpr int NT = kCW * 32;
    for (int b = 0; b < B; ++b) {
      float glog[kMaxGate];
#pragma unroll
      for (int s2 = 0; s2 < kMaxGate; ++s2)
        glog[s2] = (s2 < S && P.n_gate) ? __ldcg(P.extra + ((size_t)l * B + b) * P.n_gate + s2) : 0.f;
      for (int i = tid; i < nv; i += NT) {
        float4 yv[8], ys[kMaxGate];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < k) yv[j] = __ldcg(Y4 + ((size_t)b * k + j) * nv + i);
#pragma unroll
        for (int s2 = 0; s2 < kMaxGate; ++s2)
          if (s2 < S) ys[s2] = __ldcg(Ys4 + ((size_t)b * S + s2) * nv + i);
        const float4 xv = __ldcg(X4 + (size_t)b * nv + i);
        float m[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < k) {
            const float g = R.gates[b * k + j];
            m[0] = fmaf(g, yv[j].x, m[0]); m[1] = fmaf(g, yv[j].y, m[1]);
            m[2] = fmaf(g, yv[j].z, m[2]); m[3] = fmaf(g, yv[j].w, m[3]);
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < kMaxGate; ++s2) {
          if (s2 < S) {
            const float g = P.n_gate ? sigmoid_f(glog[s2]) : 1.0f;
            m[0] += g * ys[s2].x; m[1] += g * ys[s2].y; m[2] += g * ys[s2].z; m[3] += g * ys[s2].w;
          }
        }
        const float4 v = make_float4(xv.x + m[0], xv.y + m[1], xv.z + m[2], xv.w + m[3]);
        xb4[(size_t)b * nv + i] = v;
        if (writer) xd[(size_t)b * nv + i] = v;
      }
    }
    cbar();
    block_ln_rows(xbuf, B, d, red);
  }
}

// ------------------------------------------------------------------ attention
// Single-query attention over the KV cache (toymoe.py:178-186 at one
// position).  A unit's K and V position blocks arrive through the weight ring
// (they are static during the pass); each warp runs an online softmax over
// its positions (4 in flight), the warps merge in warp order and the unit's
// partial (m, s, o) goes to global memory.  The o-projection's input build
// merges the chunks of every head in chunk order (XK_ATTN).

template <int PER>
__device__ void attn_unit(const Plan& P, int l, const Item& it, int nc, const char* smem, int stage_bytes, int nst,
                          uint32_t& ic, uint64_t* full, uint64_t* empty, float* scratch, const int* spos) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int H = P.H, d = P.d, hd = PER * 32, B = P.B;
  const float scale = 1.0f / sqrtf((float)hd);
  float qv[PER], o[PER];
  const float* qrow = P.q + (size_t)it.b * d + it.h * hd;
#pragma unroll
  for (int j = 0; j < PER; ++j) { qv[j] = __ldcg(qrow + lane + 32 * j); o[j] = 0.f; }
  float m = -INFINITY, s = 0.f;
  auto update = [&](float sc, const float* vr) {
    const float v = sc * scale;
    const float mn = fmaxf(m, v);
    const float a = expf(m - mn), e = expf(v - mn);
    s = s * a + e;
#pragma unroll
    for (int j = 0; j < PER; ++j) o[j] = o[j] * a + e * vr[lane + 32 * j];
    m = mn;
  };
  for (int item = 0; item < it.nkc; ++item, ++ic) {
    const int st = (int)(ic % (uint32_t)nst);
    const int n = min(P.npi, it.np - item * P.npi);
    mbar_wait(&full[st], (ic / nst) & 1u);
    const float* Ks = reinterpret_cast<const float*>(smem + (size_t)st * stage_bytes);
    const float* Vs = Ks + (size_t)P.npi * hd;
    for (int j0 = warp; j0 < n; j0 += kCW * 4) {
      float sc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = min(j0 + kCW * t, n - 1);
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < PER; ++e) dot = fmaf(qv[e], Ks[(size_t)j * hd + lane + 32 * e], dot);
        sc[t] = dot;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int t = 0; t < 4; ++t) sc[t] += __shfl_xor_sync(0xffffffffu, sc[t], off);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (j0 + kCW * t < n) update(sc[t], Vs + (size_t)(j0 + kCW * t) * hd);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (it.c == nc - 1 && warp == 0) {  // the new position, written by this pass's qkv phase
    const size_t row = (((size_t)l * B + it.b) * P.Hkv + it.h / P.grp) * P.max_len + spos[it.b];
    const float* kr = P.kc + row * hd;
    const float* vr = P.vc + row * hd;
    float kv[PER], vv[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) { kv[e] = __ldcg(kr + lane + 32 * e); vv[e] = __ldcg(vr + lane + 32 * e); }
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < PER; ++e) dot = fmaf(qv[e], kv[e], dot);
    dot = warp_sum(dot);
    const float v = dot * scale;
    const float mn = fmaxf(m, v);
    const float a = expf(m - mn), e2 = expf(v - mn);
    s = s * a + e2;
#pragma unroll
    for (int e = 0; e < PER; ++e) o[e] = o[e] * a + e2 * vv[e];
    m = mn;
  }
  // warps -> smem -> merged in warp order by warp 0 -> partial
  float* wp = scratch + (size_t)warp * (hd + kAttnPart);
  if (lane == 0) { wp[0] = m; wp[1] = s; }
#pragma unroll
  for (int e = 0; e < PER; ++e) wp[kAttnPart + lane + 32 * e] = o[e];
  cbar();
  if (warp == 0) {
    float M = -INFINITY;
    for (int w = 0; w < kCW; ++w) M = fmaxf(M, scratch[(size_t)w * (hd + kAttnPart)]);
    float S = 0.f, acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    for (int w = 0; w < kCW; ++w) {
      const float* q = scratch + (size_t)w * (hd + kAttnPart);
      if (q[1] == 0.f) continue;
      const float f = expf(q[0] - M);
      S += q[1] * f;
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] += q[kAttnPart + lane + 32 * e] * f;
    }
    if (nc == 1) {  // one unit per head: the final row directly (no partial, ticket or merge)
      const float inv = 1.0f / S;
#pragma unroll
      for (int e = 0; e < PER; ++e) P.att[(size_t)it.b * d + it.h * hd + lane + 32 * e] = acc[e] * inv;
      cbar();
      return;
    }
    float* part = P.attn_part + ((size_t)(it.b * H + it.h) * P.nc_max + it.c) * (hd + kAttnPart);
    if (lane == 0) { part[0] = M; part[1] = S; }
#pragma unroll
    for (int e = 0; e < PER; ++e) part[kAttnPart + lane + 32 * e] = acc[e];
    // the head's last chunk to finish merges its nc chunks in chunk order and
    // writes the final attention row: the o-projection then loads a plain row
    // instead of every CTA merging every head after the barrier
    __syncwarp();
    unsigned last = 0;
    unsigned* tk = P.sync + 64 + it.b * H + it.h;
    if (lane == 0) {
      __threadfence();
      last = atomicAdd(tk, 1u) == (unsigned)(nc - 1) ? 1u : 0u;
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      __threadfence();
      const float* base = P.attn_part + (size_t)(it.b * H + it.h) * P.nc_max * (hd + kAttnPart);
      float mc = -INFINITY, sc = 0.f;
      if (lane < nc) {
        const float2 ms = __ldcg(reinterpret_cast<const float2*>(base + (size_t)lane * (hd + kAttnPart)));
        mc = ms.x;
        sc = ms.y;
      }
      const float Mh = warp_max(sc != 0.f ? mc : -INFINITY);
      const float f = sc != 0.f ? expf(mc - Mh) : 0.f;
      float Sh = 0.f;
      for (int c = 0; c < nc; ++c) Sh += __shfl_sync(0xffffffffu, sc * f, c);
      const float inv = 1.0f / Sh;
      float O[PER];
#pragma unroll
      for (int e = 0; e < PER; ++e) O[e] = 0.f;
      for (int c = 0; c < nc; ++c) {
        const float fc = __shfl_sync(0xffffffffu, f, c);
        if (fc != 0.f) {
#pragma unroll
          for (int e = 0; e < PER; ++e)
            O[e] = fmaf(__ldcg(base + (size_t)c * (hd + kAttnPart) + kAttnPart + lane + 32 * e), fc, O[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < PER; ++e) P.att[(size_t)it.b * d + it.h * hd + lane + 32 * e] = O[e] * inv;
      if (lane == 0) *tk = 0u;  // ready for the next layer / launch
    }
  }
  cbar();
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
__device__ __forceinline__ void online_merge(float& M, float& S, int& A, float m, float s, int a) {
  if (s == 0.f) return;
  if (m > M) { S = S * expf(M - m) + s; M = m; A = a; }
  else { S += s * expf(m - M); if (m == M && a < A) A = a; }
}

// ------------------------------------------------------------------ the kernel
template <typename W, int TT>
__global__ void __launch_bounds__(kThreads, 1) decode_pass_kernel(const __grid_constant__ Plan P, int first,
                                                                   int last, int nst, int stage_bytes,
                                                                   int xbuf_off) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ __align__(8) uint64_t empty[kMaxStages];
  __shared__ StageMeta meta[kMaxStages];
  __shared__ Route rt_c, rt_p, rt_e;  // consumers' / producer's copy; rt_e: the early-route computation
  __shared__ int spos[kMaxB];
  __shared__ __align__(16) Tmpl cph, pph;  // consumers' / producer's copy of the current phase template
  __shared__ __align__(16) float red2b[2][kCW * kTileRows * TT];  // double-buffered cross-warp row sums
  __shared__ __align__(8) uint64_t rfull[2], rempty[2];            // row sums written / read by the epilogue
  float* red2 = red2b[0];                                          // LN / head-merge scratch
  __shared__ bool is_last;
  float* red = red2b[0];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int V = WVec<W>::N;
  constexpr int KC = kChunk / (int)sizeof(W);
  const int G = gridDim.x;
  float* xbuf = reinterpret_cast<float*>(smem + xbuf_off);

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&rfull[b], kCW);
      mbar_init(&rempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < P.B) {
    int p = P.pos[tid];
    if (p < 0 || p >= P.max_len) {  // position outside the KV cache: flag it, stay in bounds
      if (blockIdx.x == 0) atomicOr(P.flags, 16);
      p = 0;
    }
    spos[tid] = p;
  }
  __syncthreads();

  if (warp == kRW) {
    // ================================================================ route warp
    // One CTA computes each layer's selection as soon as the router units'
    // logits exist (their epilogues count them in route_sync[l]), publishes it
    // (global memory + release flag; mapped host memory for the offload
    // driver) while the rest of the router phase streams; every CTA copies it.
    if (blockIdx.x != G - 1 || !P.route_pub) return;
    const unsigned n_ru = (unsigned)((P.t[P.router_j].g[0].rows + kTileRows - 1) / kTileRows);
    for (int l = 0; l < P.L; ++l) {
      const int pr = l * P.ppl + P.router_j;
      if (pr < first || pr >= last) continue;
      if (lane == 0) {
        const unsigned long long t0 = gtimer();
        while (ld_relaxed(P.route_sync + l) < n_ru) {
          __nanosleep(64);
          if (gtimer() - t0 > kWatchdogNs) { atomicOr(P.flags, 4); __trap(); }
        }
      }
      __syncwarp();
      fence_acquire();
      compute_route(P, l, rt_e, true);
      int* dst = reinterpret_cast<int*>(P.route_pub + l);
      const int* src = reinterpret_cast<const int*>(&rt_e);
      for (int i = lane; i < (int)(sizeof(Route) / 4); i += 32) __stcg(dst + i, src[i]);
      if (P.zs) publish_host(P, l, rt_e);
      __threadfence();
      __syncwarp();
      if (lane == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(P.route_sync + P.L + l), "r"(1) : "memory");
    }
    return;
  }

  if (warp == kCW) {
    // ================================================================ producer
    // Weight cursor (W): issues the weight tile of every item into the ring as
    // soon as a stage is free and the tile's address is known (static
    // matrices: always; routed experts: once the layer's selection is).
    // Activation cursor (X): issues the staged activation slices of items
    // whose inputs come from the previous phase, once its barrier completed.
    int nev = 0;                  // event-log count (debug)
    int wp = first, wu = 0, wkc = 0, wj = 0, wl = 0;
    unsigned wtgt = 0;            // barrier count after which this phase's activations exist
    Item wit;
    int rt_layer = -1;
    int pph_j = -1;
    bool fresh = true;
    int zs_layer = -1, zs_slot = 0, zs_tkt = 0;  // zero-sync: lane a = active expert a
    auto seek = [&]() -> int {  // 0 = ok, 1 = done, 2 = blocked on routing (warp-uniform)
      while (wp < last) {
        phase_jl(P, wp, wj, wl);
        if (pph_j != wj) {  // template -> shared memory (one constant-bank read per phase)
          __syncwarp();
          const int4* src = reinterpret_cast<const int4*>(&P.t[wj]);
          int4* dst = reinterpret_cast<int4*>(&pph);
          for (int i = lane; i < (int)(sizeof(Tmpl) / 16); i += 32) dst[i] = src[i];
          __syncwarp();
          pph_j = wj;
        }
        const Tmpl& T = pph;
        if (T.type == PT_PUBLISH) { ++wp; fresh = true; continue; }
        if (T.type == PT_ATTN) {  // K/V blocks of the positions already cached
          if (fresh) { wu = (blockIdx.x - rot_of(P, wj, wl) + G) % G; wkc = 0; fresh = false; }
          const int nc = attn_nc(P, spos);
          for (; wu < P.B * P.H * nc; wu += G) {
            decode_attn(P, wu, nc, spos, wit);
            if (wit.nkc > 0) return 0;
          }
          ++wp;
          fresh = true;
          continue;
        }
        if (fresh) {
          wu = (blockIdx.x - rot_of(P, wj, wl) + G) % G;
          wkc = 0;
          const int dq = dep_of(P, wp);
          wtgt = dq >= 0 ? bar_target(P, dq, first) : 0u;
          fresh = false;
        }
        while (wu < T.units) {
          const int g = group_of_unit(T, wu);
          if (T.g[g].kind == GK_ROUTED && rt_layer != wl) {
            if (route_early(P, wl, first)) {  // published by the router phase (possibly before its barrier)
              unsigned ok = 0;
              if (lane == 0) ok = route_ready(P, wl) ? 1u : 0u;
              if (!__shfl_sync(0xffffffffu, ok, 0)) return 2;
              route_copy(P, wl, rt_p);
            } else {
              unsigned ok = 1;
              if (lane == 0 && !P.replay) {
                const unsigned tgt = bar_target(P, wl * P.ppl + P.router_j, first);
                ok = (tgt == 0u || ld_relaxed(P.sync) >= tgt) ? 1u : 0u;
              }
              ok = __shfl_sync(0xffffffffu, ok, 0);
              if (!ok) return 2;
              fence_acquire();
              compute_route(P, wl, rt_p, false);
            }
            rt_layer = wl;
            if (lane == 0) log_evt(P.evt, 0, nev, EV_ROUTE, wp, 0);
          }
          const bool routed = T.g[g].kind == GK_ROUTED;
          if (P.zs && routed && zs_layer != wl) {  // the host cache's answer for this layer
            int ok = 0;
            if (lane == 0) {
              int v;
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(P.zs_slots_flag_d + wl) : "memory");
              ok = v == (int)P.zs_epoch;
            }
            if (!__shfl_sync(0xffffffffu, ok, 0)) return 2;
            if (lane < rt_p.n_active) {
              const int* q = P.zs_slots_d + ((size_t)wl * P.E + rt_p.act_e[lane]) * 2;
              zs_slot = ld_volatile_s32(q);
              zs_tkt = ld_volatile_s32(q + 1);
            }
            zs_layer = wl;
          }
          if (decode_unit<W>(P, T, wl, wu, rt_p, wit, P.zs && routed, zs_slot, zs_tkt)) {
            if (P.zs && routed) {  // stream the expert's tiles once its copy has landed
              int ok = 0;
              if (lane == 0) ok = (int)(ld_volatile_u32(P.zs_done + wit.zslot) - (unsigned)wit.tkt) >= 0;
              if (!__shfl_sync(0xffffffffu, ok, 0)) return 2;
            }
            return 0;
          }
          wu += G;
        }
        ++wp;
        fresh = true;
      }
      return 1;
    };
    int st = 2;  // 2 = (re)seek needed
    // ---- L2 prefetch cursor: walks the same unit sequence ahead of the ring
    // and pulls static tiles (dense / shared weights, cached K/V blocks) into
    // L2 with cp.async.bulk.prefetch, so HBM keeps streaming while the ring is
    // full and the consumers wait on a barrier.  Routed units are skipped (their
    // address is only known after routing); it never blocks.
    int pp = first, pu = 0, pj = 0, pl = 0;
    bool pfresh = true, pdone = P.pf_window < 0;  // < 0: no prefetch cursor at all
    unsigned long long pf_bytes = 0, w_static = 0;  // prefetched / issued-by-W static bytes
    const unsigned long long pf_window = (unsigned long long)P.pf_window;
    auto pf_step = [&]() -> bool {  // one unit; false = nothing left
      while (pp < last) {
        phase_jl(P, pp, pj, pl);
        const Tmpl& T = P.t[pj];
        if (T.type == PT_PUBLISH) { ++pp; pfresh = true; continue; }
        if (pfresh) { pu = (blockIdx.x - rot_of(P, pj, pl) + G) % G; pfresh = false; }
        if (T.type == PT_ATTN) {
          const int nc = attn_nc(P, spos);
          if (pu < P.B * P.H * nc) {
            Item a;
            decode_attn(P, pu, nc, spos, a);
            pu += G;
            if (a.np > 0) {
              const uint32_t bytes = (uint32_t)a.np * P.hd * 4u;
              const size_t row = (((size_t)pl * P.B + a.b) * P.Hkv + a.h / P.grp) * P.max_len + a.p0;
              if (lane == 0) { prefetch_l2(P.kc + row * P.hd, bytes); prefetch_l2(P.vc + row * P.hd, bytes); }
              pf_bytes += 2ull * bytes;
            }
            return true;
          }
        } else if (pu < T.units) {
          const int g = group_of_unit(T, pu);
          const Group& Gg = T.g[g];
          if (Gg.kind != GK_ROUTED) {
            int uu = pu;
            for (int i = 0; i < g; ++i) uu -= T.g[i].units;
            const int upe = (Gg.rows + kTileRows - 1) / kTileRows;
            const int a = uu / upe, rb = uu - a * upe;
            const int rr = min(kTileRows, Gg.rows - rb * kTileRows);
            const char* w = Gg.w + (long long)pl * Gg.w_l + (Gg.kind == GK_SHARED ? (long long)a * Gg.stride : 0ll) +
                            (size_t)rb * kTileRows * Gg.K * sizeof(W);
            const uint32_t bytes = (uint32_t)((size_t)rr * Gg.K * sizeof(W));
            if (lane == 0) prefetch_l2(w, bytes);
            pf_bytes += bytes;
          }
          pu += G;
          return true;
        }
        ++pp;
        pfresh = true;
      }
      return false;
    };
    uint32_t iw = 0, ix = 0;      // items issued (weights) / completed (activations)
    int relay_l = 0;              // zero-sync: next layer whose slot table CTA 0 relays
    unsigned long long relay_t = 0;
    unsigned long long t0 = 0;
    unsigned seen = 0;            // last observed barrier counter
    while (true) {
      bool progress = false;
      if (st == 2) st = seek();
      // ---- weight cursor
      if (st == 0 && iw < ix + (uint32_t)nst) {
        const int s = (int)(iw % (uint32_t)nst);
        bool free_ = true;
        if (iw >= (uint32_t)nst) {
          unsigned ok = 0;
          if (lane == 0) ok = mbar_test(&empty[s], ((iw / nst) - 1) & 1u) ? 1u : 0u;
          free_ = __shfl_sync(0xffffffffu, ok, 0) != 0;
        }
        if (free_ && wit.attn) {
          const int q0 = wit.p0 + wkc * P.npi;
          const int n = min(P.npi, wit.p0 + wit.np - q0);
          const uint32_t bytes = (uint32_t)n * P.hd * 4u;
          if (lane == 0) {
            if (iw >= (uint32_t)nst) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            meta[s].needx = 0;
            char* stg = smem + (size_t)s * stage_bytes;
            const size_t row = (((size_t)wl * P.B + wit.b) * P.Hkv + wit.h / P.grp) * P.max_len + q0;
            mbar_arrive_tx(&full[s], 2u * bytes);
            bulk_g2s(stg, P.kc + row * P.hd, bytes, &full[s]);
            bulk_g2s(stg + (size_t)P.npi * P.hd * 4, P.vc + row * P.hd, bytes, &full[s]);
          }
          w_static += 2ull * bytes;
          if (lane == 0) log_evt(P.evt, 0, nev, EV_W, wp, (int)iw);
          ++iw;
          progress = true;
          if (++wkc >= wit.nkc) {
            wkc = 0;
            wu += G;
            st = 2;
          }
        } else if (free_) {
          const Item& Gr = wit;
          const int k0 = wkc * KC, kn = min(KC, Gr.K - k0);
          const uint32_t wbytes = (uint32_t)(wit.rr * kn * sizeof(W));
          if (!wit.routed) w_static += wbytes;
          if (lane == 0) log_evt(P.evt, 0, nev, EV_W, wp, (int)iw);
          char* stg = smem + (size_t)s * stage_bytes;
          if (lane == 0) {
            if (iw >= (uint32_t)nst) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            StageMeta& mt = meta[s];
            mt.needx = Gr.xstage;
            if (Gr.xstage) {
              mt.nt = wit.n;
              mt.xbytes = kn * (int)sizeof(float);
              mt.tgt = wtgt;
#pragma unroll
              for (int t = 0; t < kMaxB; ++t)
                mt.xrow[t] = Gr.xg + (size_t)(t < wit.n ? unit_pair(P, wit, rt_p, t) : 0) * Gr.K + k0;
              mbar_tx_only(&full[s], wbytes);
            } else {
              mbar_arrive_tx(&full[s], wbytes);
            }
            if (kn == Gr.K) {
              bulk_g2s(stg, wit.wrow, wbytes, &full[s]);
            } else {
              const uint32_t rb = (uint32_t)(kn * sizeof(W));
              for (int r = 0; r < wit.rr; ++r)
                bulk_g2s(stg + (size_t)r * rb, wit.wrow + ((size_t)r * Gr.K + k0) * sizeof(W), rb, &full[s]);
            }
          }
          ++iw;
          progress = true;
          if (++wkc >= wit.nkc) {
            wkc = 0;
            wu += G;
            st = 2;
          }
        }
      }
      // ---- zero-sync relay (CTA 0 only): the host's slot tables -> device memory
      if (P.zs && blockIdx.x == 0 && relay_l < P.L) {
        const unsigned long long now = gtimer();
        if (now - relay_t > 400) {
          relay_t = now;
          int ok = 0;
          if (lane == 0) ok = ld_acquire_sys(P.zs_slots_flag_h + relay_l) == (int)P.zs_epoch;
          if (__shfl_sync(0xffffffffu, ok, 0)) {
            const int n = P.E * 2;
            for (int i = lane; i < n; i += 32)
              P.zs_slots_d[(size_t)relay_l * n + i] = ld_volatile_s32(P.zs_slots_h + (size_t)relay_l * n + i);
            __syncwarp();
            if (lane == 0) {
              __threadfence();
              asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(P.zs_slots_flag_d + relay_l), "r"((int)P.zs_epoch)
                           : "memory");
            }
            ++relay_l;
            progress = true;
          }
        }
      }
      // ---- L2 prefetch cursor (bounded distance ahead of the ring)
      if (!pdone && pf_bytes < w_static + pf_window) {
        pdone = !pf_step();
        progress = true;
      }
      // ---- activation cursor
      __syncwarp();
      if (ix < iw) {
        const int s = (int)(ix % (uint32_t)nst);
        const StageMeta& mt = meta[s];
        if (!mt.needx) {
          ++ix;
          progress = true;
        } else {
          const unsigned tgt = mt.tgt;
          unsigned ok = 0;
          if (lane == 0) {
            if (seen < tgt) seen = ld_relaxed(P.sync);
            ok = seen >= tgt ? 1u : 0u;
          }
          if (__shfl_sync(0xffffffffu, ok, 0)) {
            if (lane == 0) {
              fence_acquire();
              asm volatile("fence.proxy.async.global;" ::: "memory");
              char* stg = smem + (size_t)s * stage_bytes + kWBytes;
              mbar_arrive_tx(&full[s], (uint32_t)(mt.nt * mt.xbytes));
              for (int t = 0; t < mt.nt; ++t)
                bulk_g2s(stg + (size_t)t * mt.xbytes, mt.xrow[t], (uint32_t)mt.xbytes, &full[s]);
              log_evt(P.evt, 0, nev, EV_X, 0, (int)ix);
            }
            ++ix;
            progress = true;
          }
        }
      }
      if (st == 1 && ix == iw && !(P.zs && blockIdx.x == 0 && relay_l < P.L)) break;
      if (!progress) {
        if (t0 == 0) t0 = gtimer();
        else if (gtimer() - t0 > kWatchdogNs) {
          if (lane == 0) {
            atomicOr(P.flags, 8);
            if (P.diag && atomicCAS(P.diag, 0, 1) == 0) {
              P.diag[1] = blockIdx.x; P.diag[2] = wp; P.diag[3] = wl; P.diag[4] = st; P.diag[5] = (int)iw;
              P.diag[6] = (int)ix; P.diag[7] = zs_layer; P.diag[8] = wit.zslot; P.diag[9] = wit.tkt;
              P.diag[10] = P.zs ? (int)ld_volatile_u32(P.zs_done + wit.zslot) : -1;
              P.diag[11] = (int)ld_relaxed(P.sync); P.diag[12] = P.zs ? ld_volatile_s32(P.zs_slots_flag_h + wl) : -1;
              P.diag[13] = (int)P.zs_epoch; P.diag[14] = rt_layer; P.diag[15] = wit.routed;
              __threadfence_system();
            }
          }
          __trap();
        }
        // The producer shares an SM sub-partition with consumer warps 0 and 4
        // and the scheduler favours the highest warp id: never busy-poll.
        // Ring full -> sleep in hardware on the stage's empty barrier;
        // waiting for a grid barrier / routing -> back off.
        const bool relaying = P.zs && blockIdx.x == 0 && relay_l < P.L;
        if (!relaying && st == 0 && iw >= (uint32_t)nst && iw < ix + (uint32_t)nst) {
          const int s = (int)(iw % (uint32_t)nst);
          if (lane == 0) mbar_wait_sleep(&empty[s], ((iw / nst) - 1) & 1u);
          __syncwarp();
        } else {
          __nanosleep(256);
        }
      } else {
        t0 = 0;
      }
    }
    return;
  }

  // ================================================================== consumers
  uint32_t ic = 0;  // items consumed
  float hm[2] = {-INFINITY, -INFINITY}, hs[2] = {0.f, 0.f};  // head: online (max, sum-exp, argmax)
  int ha[2] = {0x7fffffff, 0x7fffffff};                         // per (token, row) slot of this lane
  uint32_t uc = 0;  // units reduced (red2 double-buffer / epilogue rotation)
  int rtc_layer = -1;
  int cev = 0;
  constexpr int SL = KC / kCW;  // K elements of a chunk owned by one warp (= 32 lanes x V)
  for (int p = first; p < last; ++p) {
    int j, l;
    phase_jl(P, p, j, l);
    {  // the phase template -> shared memory (the previous phase ended with a cbar)
      const int4* src = reinterpret_cast<const int4*>(&P.t[j]);
      int4* dst = reinterpret_cast<int4*>(&cph);
      for (int i = tid; i < (int)(sizeof(Tmpl) / 16); i += kCW * 32) dst[i] = src[i];
    }
    const Tmpl& T = cph;
    // trace (debug): [0] inputs visible, [1] inputs built, [2] work done, [3] arrival
    // issued, [4] barrier observed, [5] acquire fence done
    unsigned long long* tr = P.trace ? P.trace + ((size_t)(p - first) * G + blockIdx.x) * kTraceSlots : nullptr;
    // ---- wait for the phase's inputs
    if (tid == 0) {
      const int dep = dep_of(P, p);
      if (dep >= first) spin_until(P, bar_target(P, dep, first), p, tr ? tr + 4 : nullptr);
    }
    cbar();
    if (tid == 0) log_evt(P.evt, 1, cev, EV_PASS, p, 0);
    if (tr && tid == 0) tr[0] = gtimer();
    const int rot = rot_of(P, j, l);
    // ---- the layer's selection (one call site: inlined once)
    const bool pub = T.type == PT_PUBLISH;
    const bool early = route_early(P, l, first);
    if (warp == 1 && (pub ? (blockIdx.x == 0 && !early) : (T.type == PT_GEMV && T.has_routed && rtc_layer != l))) {
      if (early) {  // copy the selection published during the router phase
        if (lane == 0) {
          const unsigned long long t0 = gtimer();
          while (!route_ready(P, l)) {
            __nanosleep(32);
            if (gtimer() - t0 > kWatchdogNs) { atomicOr(P.flags, 4); __trap(); }
          }
        }
        __syncwarp();
        route_copy(P, l, rt_c);
      } else {
        compute_route(P, l, rt_c, pub || blockIdx.x == 0);
        if (pub && P.zs) publish_host(P, l, rt_c);
      }
    }
    if (P.zs && blockIdx.x == 0 && tid == 0 && ((j == 0 && l > 0) || j == P.ppl)) {
      // every CTA is past layer l-1's routed down (this phase's barrier): its slots may be reused
      const unsigned v = P.zs_prog_base + (unsigned)l;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.zs_prog), "r"(v) : "memory");
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(P.zs_prog_h), "r"(v) : "memory");
    }
    if (!pub && T.type == PT_GEMV && T.has_routed) rtc_layer = l;
    if (pub) {
    } else if (T.type == PT_ATTN) {
      const int nc = attn_nc(P, spos);
      Item it;
      for (int u = (blockIdx.x - rot + G) % G; u < P.B * P.H * nc; u += G) {
        decode_attn(P, u, nc, spos, it);
        switch (P.hd / 32) {
          case 1: attn_unit<1>(P, l, it, nc, smem, stage_bytes, nst, ic, full, empty, xbuf, spos); break;
          case 2: attn_unit<2>(P, l, it, nc, smem, stage_bytes, nst, ic, full, empty, xbuf, spos); break;
          case 4: attn_unit<4>(P, l, it, nc, smem, stage_bytes, nst, ic, full, empty, xbuf, spos); break;
          default: attn_unit<8>(P, l, it, nc, smem, stage_bytes, nst, ic, full, empty, xbuf, spos); break;
        }
      }
    } else {
      const int xk = l == 0 ? T.xkind0 : T.xkind;
      if (xk != XK_NONE && (!T.keep_x || p == first)) load_x(P, xk, T.xsrc, T.xdst, l - 1, xbuf, red, rt_c, spos);
      cbar();
      if (tr && tid == 0) tr[1] = gtimer();
      if (tid == 0) log_evt(P.evt, 1, cev, EV_READY, p, 0);
      const bool head_phase = T.g[0].epi == EP_HEAD;
      if (head_phase) {
        hm[0] = hm[1] = -INFINITY;
        hs[0] = hs[1] = 0.f;
        ha[0] = ha[1] = 0x7fffffff;
      }
      Item it;
      for (int u = (blockIdx.x - rot + G) % G; u < T.units; u += G) {
        if (!decode_unit<W>(P, T, l, u, rt_c, it)) continue;
        const Item& Gr = it;
        const int nt = it.n, rr = it.rr;
        // warp w owns K elements [w*SL, (w+1)*SL) of every row of the tile
        float acc[kTileRows][TT];
#pragma unroll
        for (int r = 0; r < kTileRows; ++r)
#pragma unroll
          for (int t = 0; t < TT; ++t) acc[r][t] = 0.f;
        for (int kc = 0; kc < it.nkc; ++kc, ++ic) {
          const int s = (int)(ic % (uint32_t)nst);
          const int k0 = kc * KC, kn = min(KC, Gr.K - k0);
          const int e0 = warp * SL + lane * V;
          if (tid == 0) log_evt(P.evt, 1, cev, EV_WAIT, p, (int)ic);
          mbar_wait(&full[s], (ic / nst) & 1u);
          if (tid == 0) log_evt(P.evt, 1, cev, EV_FULL, p, (int)ic);
          if (e0 < kn) {
            const char* stg = smem + (size_t)s * stage_bytes;
            float xv[TT][V];  // absent token slots are zero: no predicates in the FMA chains
#pragma unroll
            for (int t = 0; t < TT; ++t) {
#pragma unroll
              for (int q = 0; q < V; ++q) xv[t][q] = 0.f;
              if (TT == 1 || t < nt) {
                const float* xr = Gr.xstage ? reinterpret_cast<const float*>(stg + kWBytes) + (size_t)t * kn + e0
                                            : xbuf + (size_t)unit_token(P, it, rt_c, t) * Gr.K + k0 + e0;
#pragma unroll
                for (int qq = 0; qq < V / 4; ++qq) {
                  const float4 x4 = reinterpret_cast<const float4*>(xr)[qq];
                  xv[t][4 * qq] = x4.x; xv[t][4 * qq + 1] = x4.y; xv[t][4 * qq + 2] = x4.z; xv[t][4 * qq + 3] = x4.w;
                }
              }
            }
            const W* wb = reinterpret_cast<const W*>(stg) + e0;
            // all 16 rows' vectors in flight first, then q-outer / row-inner
            // FMAs: 16 independent accumulation chains (same per-row order)
            constexpr int RB = TT == 1 ? 8 : 2;  // rows in flight
#pragma unroll
            for (int r0 = 0; r0 < kTileRows; r0 += RB) {
              // rows >= rr read stale stage bytes: their sums are never used (the
              // butterfly below never mixes rows), so no predicate either
              uint4 wv[RB];
#pragma unroll
              for (int r = 0; r < RB; ++r) wv[r] = *reinterpret_cast<const uint4*>(wb + (size_t)(r0 + r) * kn);
#pragma unroll
              for (int q = 0; q < V; ++q) {
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                  const float f = WVec<W>::elem(wv[r], q);
#pragma unroll
                  for (int t = 0; t < TT; ++t) acc[r0 + r][t] = fmaf(f, xv[t][q], acc[r0 + r][t]);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
        // ---- reduce: 16 rows over 32 lanes (butterfly), then over warps in order
        float rs[TT];
#pragma unroll
        for (int t = 0; t < TT; ++t) rs[t] = reduce_rows16<TT>(acc, t, lane);
        if (tid == 0) log_evt(P.evt, 1, cev, EV_RED, p, 0);
        // ---- hand the row sums to this unit's epilogue warp (uc % kCW) through
        // a double-buffered smem area: no CTA-wide barrier per unit
        const int bb = (int)(uc & 1u);
        if (uc >= 2) mbar_wait(&rempty[bb], ((uc - 2) >> 1) & 1u);
        float* rb = red2b[bb];
        if ((lane & 1) == 0)
#pragma unroll
          for (int t = 0; t < TT; ++t) rb[(warp * kTileRows + ((lane >> 1) & 15)) * TT + t] = rs[t];
        __syncwarp();
        if (lane == 0) mbar_arrive(&rfull[bb]);
        if (warp == (int)(uc % kCW)) {
          mbar_wait(&rfull[bb], (uc >> 1) & 1u);
          if (tid == (int)(uc % kCW) * 32) log_evt(P.evt, 1, cev, EV_UNIT, p, 0);
#pragma unroll
          for (int xi = 0; xi < 2; ++xi) {  // (token, row) slots lane and lane + 32
            const int x = lane + 32 * xi;
            const int t = x >> 4, i = x & 15;
            if (x < kTileRows * TT && t < nt && i < rr) {
              float v = 0.f;
#pragma unroll
              for (int w = 0; w < kCW; ++w) v += rb[(w * kTileRows + i) * TT + t];
              const int r0 = it.rb * kTileRows + i;
              const int pr = unit_pair(P, it, rt_c, t), tb = unit_token(P, it, rt_c, t);
              if (Gr.epi == EP_HEAD) {
                const float lg = v * P.logit_scale;
                if (P.head_logits) P.head_logits[(size_t)tb * P.V + r0] = lg;
                online_add(hm[xi], hs[xi], ha[xi], lg, r0);
              } else if (Gr.epi == EP_SWIGLU) {  // tile rows [8 gate | 8 up]
                if (i < 8) {
                  float u2 = 0.f;
#pragma unroll
                  for (int w = 0; w < kCW; ++w) u2 += rb[(w * kTileRows + i + 8) * TT + t];
                  Gr.out[(size_t)pr * Gr.out_ld + it.rb * 8 + i] = silu_f(v) * u2;
                }
              } else if (Gr.epi == EP_QKV) {
                const int d = P.d;
                const int kvd = P.Hkv * P.hd;  // rows [q (d) | k (kvd) | v (kvd)]
                if (r0 < d) P.q[(size_t)tb * d + r0] = v;
                else {
                  float* cache = r0 < d + kvd ? P.kc : P.vc;
                  const int c = r0 < d + kvd ? r0 - d : r0 - d - kvd;
                  const int hh = c / P.hd;
                  cache[((((size_t)l * P.B + tb) * P.Hkv + hh) * P.max_len + spos[tb]) * P.hd + (c - hh * P.hd)] = v;
                }
              } else if (Gr.epi == EP_LOGITS) {
                if (r0 < Gr.split) Gr.out[(size_t)tb * Gr.out_ld + r0] = v;
                else Gr.out2[(size_t)tb * (Gr.rows - Gr.split) + (r0 - Gr.split)] = v;
              } else {
                const size_t o0 = (size_t)pr * Gr.out_ld + r0;
                if (Gr.epi == EP_RELU) v = fmaxf(v, 0.f);
                else if (Gr.resid) v += __ldcg(Gr.resid + o0);
                Gr.out[o0] = v;
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[bb]);
          if (Gr.epi == EP_LOGITS && route_early(P, l, first) && lane == 0) {
            __threadfence();  // this unit's logits, then the count the route warp waits for
            atomicAdd(P.route_sync + l, 1u);
          }
        }
        ++uc;
      }
      if (head_phase) {
        // merge the 16 row-threads of each token (row order), then CTAs (CTA order) in the last CTA
        // merge each warp's 16 row slots per token (fixed butterfly), then the
        // warps in warp order, then CTAs (CTA order) in the last CTA
#pragma unroll
        for (int xi = 0; xi < 2; ++xi)
#pragma unroll
          for (int off = 8; off > 0; off >>= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, hm[xi], off);
            const float os = __shfl_xor_sync(0xffffffffu, hs[xi], off);
            const int oa = __shfl_xor_sync(0xffffffffu, ha[xi], off);
            online_merge(hm[xi], hs[xi], ha[xi], om, os, oa);
          }
        cbar();
#pragma unroll
        for (int xi = 0; xi < 2; ++xi) {
          const int x = lane + 32 * xi, t = x >> 4;
          if ((x & 15) == 0 && t < TT) {
            float* q = red2 + (warp * kMaxB + t) * 3;
            q[0] = hm[xi];
            q[1] = hs[xi];
            q[2] = __int_as_float(ha[xi]);
          }
        }
        cbar();
        if (tid < P.B) {
          float M = -INFINITY, S = 0.f;
          int A = 0x7fffffff;
          for (int w = 0; w < kCW; ++w) {
            const float* q = red2 + (w * kMaxB + tid) * 3;
            online_merge(M, S, A, q[0], q[1], __float_as_int(q[2]));
          }
          float* hp = P.head_part + ((size_t)blockIdx.x * kMaxB + tid) * 3;
          hp[0] = M; hp[1] = S; hp[2] = __int_as_float(A);
        }
        __threadfence();
        cbar();
        if (tid == 0) is_last = atomicAdd(P.sync + 2, 1u) == gridDim.x - 1;
        cbar();
        if (is_last) {
          __threadfence();
          if (tid < P.B) {
            float M = -INFINITY, S = 0.f;
            int A = 0x7fffffff;
            for (unsigned b = 0; b < gridDim.x; ++b) {
              const float* hp = P.head_part + ((size_t)b * kMaxB + tid) * 3;
              online_merge(M, S, A, __ldcg(hp), __ldcg(hp + 1), __float_as_int(__ldcg(hp + 2)));
            }
            const float conf = 1.0f / S;
            P.conf[tid] = conf;
            if (P.argmax) P.argmax[tid] = A;
            if (P.fallback) P.fallback[tid] = conf <= P.gamma ? 1 : 0;
          }
          if (tid == 0) P.sync[2] = 0u;
        }
      }
    }
    // ---- end of phase: grid barrier arrival
    cbar();
    if (tr && tid == 0) tr[2] = gtimer();
    if (tid == 0) log_evt(P.evt, 1, cev, EV_ARRIVE, p, 0);
    if (T.end_bar && tid == 0) red_release_add(P.sync, 1u);
    if (tr && tid == 0) tr[3] = gtimer();
  }
  // exit ticket: the last CTA out resets the barrier for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(P.sync + 1, 1u) == gridDim.x - 1) {
      P.sync[0] = 0u;
      P.sync[1] = 0u;
      if (P.route_sync)
        for (int i = 0; i < 2 * P.L; ++i) P.route_sync[i] = 0u;
      __threadfence();
    }
  }
}

#ifdef MOBILE_DP_ROUTE_BENCH
// debug: compute_route alone (one warp), cycles per call
__global__ void route_bench_kernel(Plan P, int iters, long long* out) {
  __shared__ Route R;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) compute_route(P, it % P.L, R, false);
  __syncwarp();
  if (threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
}
#endif
}  // namespace dp
}  // namespace mobile

// ====================================================================== host
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <vector>

using namespace mobile;
using namespace mobile::dp;

struct mobile_dp {
  Plan plan{};
  // zero-sync offload state (mapped host buffers)
  int* h_route = nullptr;
  int* h_route_flag = nullptr;
  int* h_slots = nullptr;
  int* h_slots_flag = nullptr;
  unsigned* h_prog = nullptr;
  unsigned epoch = 0, prog_base = 0;
  int* h_diag = nullptr;
  int* d_slots = nullptr;
  int* d_slots_flag = nullptr;
  std::vector<int> seg_first;  // offload: first phase of segment l (l = 0..L), seg_first[L+1] = n_phases
  void* d_ws = nullptr;
  int w_dtype = 0, TT = 1, nst = 3, stage_bytes = 0, xbuf_off = 0;
  size_t smem = 0;
  int grid = 0;
};

namespace {

template <typename W, int TT>
void* kernel_ptr() { return (void*)decode_pass_kernel<W, TT>; }

void* pick_kernel(int w_dtype, int TT) {
  if (w_dtype == MOBILE_BF16) return TT == 1 ? kernel_ptr<__nv_bfloat16, 1>() : TT == 2 ? kernel_ptr<__nv_bfloat16, 2>() : kernel_ptr<__nv_bfloat16, 4>();
  return TT == 1 ? kernel_ptr<float, 1>() : TT == 2 ? kernel_ptr<float, 2>() : kernel_ptr<float, 4>();
}

Group dense_group(const void* w, long long w_l, int K, int rows, int epi) {
  Group g{};
  g.w = (const char*)w;
  g.w_l = w_l;
  g.K = K;
  g.rows = rows;
  g.kind = GK_DENSE;
  g.epi = epi;
  g.n_exp = 1;
  g.split = rows;
  return g;
}

}  // namespace

extern "C" {

int mobile_dp_create(const mobile_dp_model* m, mobile_dp** out) {
  *out = nullptr;
  const int B = m->B, d = m->d, L = m->L, E = m->E, k = m->k, S = m->n_shared;
  const int eb = m->w_dtype == MOBILE_BF16 ? 2 : 4;
  if (m->w_dtype != MOBILE_BF16 && m->w_dtype != MOBILE_F32) { set_error("decode_pass: unsupported dtype"); return MOBILE_ERR_UNSUPPORTED; }
  if (B < 1 || B > kMaxB || B * k > kMaxPairs || k > 8 || E > kMaxE || S > kMaxGate || m->n_gate > S || m->H < 1 ||
      d % m->H || d / m->H > 256 || (d / m->H) % 32 || d % 8 || d > 4096 || L < 1) {
    set_error("decode_pass: unsupported shape B=%d k=%d E=%d S=%d d=%d H=%d", B, k, E, S, d, m->H);
    return MOBILE_ERR_UNSUPPORTED;
  }
  const int Hkv = m->Hkv > 0 ? m->Hkv : m->H;  // grouped-query attention: key/value heads
  if (m->H % Hkv) { set_error("decode_pass: Hkv=%d must divide H=%d", Hkv, m->H); return MOBILE_ERR_INVALID; }
  auto* o = new mobile_dp();
  o->w_dtype = m->w_dtype;
  o->TT = B == 1 ? 1 : B == 2 ? 2 : 4;
  const int G = sm_count();
  o->grid = G;
  // ---- shared memory: ring of (64 KB weights + TT activation slices) + xbuf
  // staged activation slices: TT rows of at most one K chunk of the widest
  // staged input (routed down K = ffn, shared down K = shared_ffn)
  const int kc_elems = kChunk / eb;
  int xk = std::min(kc_elems, m->ffn);
  if (S) xk = std::max(xk, std::min(kc_elems, m->shared_ffn));
  const int xslice = (xk * 4 + 127) / 128 * 128;
  o->stage_bytes = kWBytes + o->TT * xslice;
  const int hd = d / m->H;
  const size_t xbuf = std::max((size_t)B * d * 4, (size_t)kCW * (hd + kAttnPart) * 4);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, pick_kernel(m->w_dtype, o->TT));
  const size_t cap = (size_t)optin - fa.sharedSizeBytes;
  int nst = 3;
  if (const char* e = std::getenv("MOBILE_DP_STAGES")) nst = std::max(2, std::min(3, std::atoi(e)));
  while (nst > 1 && (size_t)nst * o->stage_bytes + xbuf > cap) --nst;
  if (nst < 2) { set_error("decode_pass: shared memory does not fit (B=%d d=%d)", B, d); delete o; return MOBILE_ERR_UNSUPPORTED; }
  o->nst = nst;
  o->xbuf_off = nst * o->stage_bytes;
  o->smem = (size_t)o->xbuf_off + xbuf;

  // ---- workspace: sync words, attention partials, head partials
  int nc_max = std::min(32, std::max(1, G / std::max(1, B * m->H)));
  if (const char* e = std::getenv("MOBILE_DP_ATTN_NC")) nc_max = std::max(1, std::min(nc_max, std::atoi(e)));
  const size_t sync_bytes = (4 * (64 + (size_t)B * m->H) + 511) / 256 * 256;
  const size_t attn_bytes = 4 * (size_t)B * m->H * nc_max * (hd + kAttnPart);
  const size_t head_bytes = 4 * (size_t)G * kMaxB * 3;
  const size_t route_bytes = ((sizeof(Route) * (size_t)L + 255) / 256) * 256;
  const size_t rsync_bytes = ((8 * (size_t)L + 255) / 256) * 256;
  const size_t ws = sync_bytes + attn_bytes + head_bytes + route_bytes + rsync_bytes;
  if (cudaMalloc(&o->d_ws, ws) != cudaSuccess || cudaMemset(o->d_ws, 0, ws) != cudaSuccess) {
    set_error("decode_pass: workspace allocation failed");
    delete o;
    return MOBILE_ERR_CUDA;
  }
  Plan& P = o->plan;
  P.B = B; P.d = d; P.H = m->H; P.E = E; P.k = k; P.S = S; P.n_gate = m->n_gate; P.gate_norm = m->gate_norm;
  P.reuse_gates = m->reuse_gates; P.max_len = m->max_len; P.L = L; P.V = m->V; P.nc_max = nc_max; P.TT = o->TT;
  P.logit_scale = m->logit_scale; P.gamma = m->gamma;
  P.hd = hd; P.npi = kWBytes / (2 * hd * 4);
  P.Hkv = Hkv; P.grp = m->H / Hkv;
  // measured: an L2 prefetch cursor ahead of (or trailing) the ring slows the
  // pass (C3 little 2037 -> 1906 us without it); MOBILE_DP_PF_KB >= 0 enables it
  P.pf_window = -1;
  if (const char* e = std::getenv("MOBILE_DP_PF_KB")) P.pf_window = std::max(-1, std::atoi(e)) * 1024;
  P.tok = m->tok; P.pos = m->pos; P.embed = m->embed; P.pe = m->pe; P.kc = m->kc; P.vc = m->vc;
  P.q = m->q; P.att = m->att; P.Y = m->Y; P.Ys = m->Ys; P.states = m->states; P.extra = m->extra;
  P.replay = m->replay; P.idx_out = m->idx_out; P.gates_out = m->gates_out; P.active_out = m->active_out;
  P.head_logits = m->head_logits; P.conf = m->conf; P.argmax = m->argmax; P.fallback = m->fallback;
  P.sync = (unsigned*)o->d_ws;
  P.attn_part = (float*)((char*)o->d_ws + sync_bytes);
  P.head_part = (float*)((char*)o->d_ws + sync_bytes + attn_bytes);
  P.route_pub = (Route*)((char*)o->d_ws + sync_bytes + attn_bytes + head_bytes);
  P.route_sync = (unsigned*)((char*)o->d_ws + sync_bytes + attn_bytes + head_bytes + route_bytes);
  // early routing pays when the router phase has other work to hide it under
  // (the shared experts' gate-up); without shared experts the phase is the 4
  // router units alone and every CTA computing the route itself is faster
  // (measured: C3 -4% / C2 +4.5% pass time with it)
  if (S == 0) P.route_pub = nullptr;
  if (const char* e = std::getenv("MOBILE_DP_EARLY_ROUTE")) {
    if (std::strcmp(e, "0") == 0) P.route_pub = nullptr;
    if (std::strcmp(e, "1") == 0) P.route_pub = (Route*)((char*)o->d_ws + sync_bytes + attn_bytes + head_bytes);
  }
  P.flags = m->flags;
  P.trace = nullptr;
  P.evt = nullptr;
  P.diag = nullptr;
  if (cudaHostAlloc((void**)&o->h_diag, sizeof(int) * 16, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
    std::memset(o->h_diag, 0, sizeof(int) * 16);
    void* dd = nullptr;
    cudaHostGetDevicePointer(&dd, o->h_diag, 0);
    P.diag = (int*)dd;
  }

  // ---- per-layer phase templates
  const long long Wsz = (long long)d * d * eb;
  const int I = m->ffn, Is = m->shared_ffn;
  const bool swiglu = m->activation == MOBILE_ACT_SWIGLU;
  const int r13 = swiglu ? 2 * I : I, r13s = swiglu ? 2 * Is : Is;
  const int act_epi = swiglu ? EP_SWIGLU : EP_RELU;
  const int ng1 = std::max(m->n_gate, 1);
  std::vector<Tmpl> ts;
  {  // qkv
    Tmpl t{};
    t.type = PT_GEMV; t.n_groups = 1; t.end_bar = 1;
    const int qkv_rows = d + 2 * (d / m->H) * Hkv;  // [q | k | v], k / v narrower under GQA
    t.g[0] = dense_group(m->qkv, (long long)qkv_rows * d * eb, d, qkv_rows, EP_QKV);
    t.xkind0 = XK_EMBED_LN; t.xkind = XK_COMBINE_LN; t.xsrc = m->xa; t.xdst = m->x;
    ts.push_back(t);
  }
  {  // attention
    Tmpl t{};
    t.type = PT_ATTN; t.end_bar = 1;
    ts.push_back(t);
  }
  {  // o + residual
    Tmpl t{};
    t.type = PT_GEMV; t.n_groups = 1; t.end_bar = 1;
    t.g[0] = dense_group(m->o, Wsz, d, d, EP_STORE);
    t.g[0].out = m->xa; t.g[0].out_ld = d; t.g[0].resid = m->x;
    t.xkind0 = t.xkind = XK_PLAIN; t.xsrc = m->att;  // merged per head by its last attention chunk
    ts.push_back(t);
  }
  const int router_j = (int)ts.size();
  {  // router logits (+ shared gates) + shared gate-up
    Tmpl t{};
    t.type = PT_GEMV; t.end_bar = 1;
    t.xkind0 = t.xkind = XK_LN; t.xsrc = m->xa;
    const int rrows = E + m->n_gate;
    t.g[0] = dense_group(m->router, (long long)rrows * d * eb, d, rrows, EP_LOGITS);
    t.g[0].out = m->states; t.g[0].out_l = (long long)B * E; t.g[0].out_ld = E; t.g[0].split = E;
    t.g[0].out2 = m->extra; t.g[0].out2_l = (long long)B * ng1;
    t.n_groups = 1;
    if (S) {
      Group g{};
      g.w = (const char*)m->shared; g.w_l = (long long)S * m->shared_stride;
      g.stride = m->shared_stride; g.K = d; g.rows = r13s; g.kind = GK_SHARED; g.epi = act_epi; g.n_exp = S;
      g.out = m->Us; g.out_ld = Is; g.split = r13s;
      t.g[t.n_groups++] = g;
    }
    ts.push_back(t);
  }
  if (m->offload) {  // publish the layer's selection for the host cache
    Tmpl t{};
    t.type = PT_PUBLISH;
    ts.push_back(t);
  }
  const int gu_j = (int)ts.size();
  {  // shared down (static weights first) + routed gate-up
    Tmpl t{};
    t.type = PT_GEMV; t.end_bar = 1; t.has_routed = 1;
    t.xkind0 = t.xkind = XK_LN; t.keep_x = 1; t.xsrc = m->xa;
    if (S) {
      Group g{};
      g.w = (const char*)m->shared + m->shared_w2_offset; g.w_l = (long long)S * m->shared_stride;
      g.stride = m->shared_stride; g.K = Is; g.rows = d; g.kind = GK_SHARED; g.epi = EP_STORE; g.n_exp = S;
      g.out = m->Ys; g.out_ld = d; g.xstage = 1; g.xg = m->Us; g.split = d;
      t.g[t.n_groups++] = g;
    }
    Group g{};
    g.w = (const char*)m->experts; g.w_l = m->expert_layer_stride;
    g.stride = m->expert_stride; g.slot = m->slot_table; g.slot_l = E;
    g.K = d; g.rows = r13; g.kind = GK_ROUTED; g.epi = act_epi; g.n_exp = std::min(E, B * k);
    g.out = m->U; g.out_ld = I; g.split = r13;
    t.g[t.n_groups++] = g;
    ts.push_back(t);
  }
  {  // routed down
    Tmpl t{};
    t.type = PT_GEMV; t.end_bar = 1; t.has_routed = 1; t.n_groups = 1;
    Group g{};
    g.w = (const char*)m->experts + m->expert_w2_offset; g.w_l = m->expert_layer_stride;
    g.stride = m->expert_stride; g.slot = m->slot_table; g.slot_l = E;
    g.K = I; g.rows = d; g.kind = GK_ROUTED; g.epi = EP_STORE; g.n_exp = std::min(E, B * k);
    g.out = m->Y; g.out_ld = d; g.xstage = 1; g.xg = m->U; g.split = d;
    t.g[0] = g;
    ts.push_back(t);
  }
  const int ppl = (int)ts.size();
  {  // head
    Tmpl t{};
    t.type = PT_GEMV; t.n_groups = 1; t.end_bar = 0;
    t.xkind0 = t.xkind = XK_COMBINE_LN; t.xsrc = m->xa; t.xdst = m->x;
    t.g[0] = dense_group(m->head, 0, d, m->V, EP_HEAD);
    ts.push_back(t);
  }
  int upl = 0, bpl = 0;
  for (size_t i = 0; i < ts.size(); ++i) {
    Tmpl& t = ts[i];
    t.units = 0;
    for (int g = 0; g < t.n_groups; ++g) {
      Group& gr = t.g[g];
      gr.units = gr.n_exp * ((gr.rows + kTileRows - 1) / kTileRows);
      t.units += gr.units;
      if (gr.K % (eb == 2 ? 8 : 4)) { set_error("decode_pass: K=%d not a multiple of the vector width", gr.K); delete o; return MOBILE_ERR_UNSUPPORTED; }
      if (gr.epi == EP_SWIGLU && gr.rows % kTileRows) { set_error("decode_pass: SwiGLU rows %% 16"); delete o; return MOBILE_ERR_UNSUPPORTED; }
    }
    if (t.type == PT_ATTN) t.units = B * m->H * nc_max;  // rotation only
    if ((int)i < ppl) { upl += t.units; bpl += t.end_bar; }
  }
  for (size_t i = 0; i < ts.size(); ++i) P.t[i] = ts[i];
  P.ppl = ppl; P.L = L; P.n_phases = ppl * L + 1; P.bpl = bpl; P.upl = upl; P.router_j = router_j;
  if (m->offload) {  // segments cut before each layer's routed gate-up
    o->seg_first.push_back(0);
    for (int l = 0; l < L; ++l) o->seg_first.push_back(l * ppl + gu_j);
    o->seg_first.push_back(P.n_phases);
  }
  void* kern = pick_kernel(o->w_dtype, o->TT);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)o->smem) != cudaSuccess) {
    set_error("decode_pass: cannot reserve %zu B of shared memory", o->smem);
    cudaFree(o->d_ws);
    delete o;
    return MOBILE_ERR_UNSUPPORTED;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, o->smem);
  if (occ < 1) { set_error("decode_pass: kernel does not fit on an SM"); cudaFree(o->d_ws); delete o; return MOBILE_ERR_UNSUPPORTED; }
  *out = o;
  return MOBILE_OK;
}

void mobile_dp_destroy(mobile_dp* o) {
  if (!o) return;
  if (o->h_route) cudaFreeHost(o->h_route);
  if (o->h_route_flag) cudaFreeHost(o->h_route_flag);
  if (o->h_slots) cudaFreeHost(o->h_slots);
  if (o->h_slots_flag) cudaFreeHost(o->h_slots_flag);
  if (o->h_prog) cudaFreeHost(o->h_prog);
  if (o->h_diag) cudaFreeHost(o->h_diag);
  if (o->d_slots) cudaFree(o->d_slots);
  if (o->d_slots_flag) cudaFree(o->d_slots_flag);
  cudaFree(o->d_ws);
  delete o;
}

int mobile_dp_num_segments(const mobile_dp* o) { return o->seg_first.empty() ? 1 : (int)o->seg_first.size() - 1; }

int mobile_dp_info(const mobile_dp* o, int* out4) {
  out4[0] = o->plan.n_phases;
  out4[1] = o->nst;
  out4[2] = (int)o->smem;
  out4[3] = o->grid;
  return MOBILE_OK;
}

int mobile_dp_diag(const mobile_dp* o, int* out16) {
  if (!o->h_diag) return MOBILE_ERR_INVALID;
  for (int i = 0; i < 16; ++i) out16[i] = ((volatile int*)o->h_diag)[i];
  return MOBILE_OK;
}

int mobile_dp_set_events(mobile_dp* o, unsigned long long* evt) {
  o->plan.evt = evt;
  return MOBILE_OK;
}

int mobile_dp_set_trace(mobile_dp* o, unsigned long long* trace) {
  o->plan.trace = trace;
  return MOBILE_OK;
}

// Launch the whole pass (segment = -1) or one offload segment.
int mobile_dp_launch(mobile_dp* o, int segment, void* stream) {
  int first = 0, last = o->plan.n_phases;
  if (segment >= 0) {
    if (o->seg_first.empty() || segment + 1 >= (int)o->seg_first.size()) { set_error("decode_pass: bad segment %d", segment); return MOBILE_ERR_INVALID; }
    first = o->seg_first[segment];
    last = o->seg_first[segment + 1];
  }
  void* kern = pick_kernel(o->w_dtype, o->TT);
  void* args[] = {(void*)&o->plan, (void*)&first, (void*)&last, (void*)&o->nst, (void*)&o->stage_bytes, (void*)&o->xbuf_off};
  // cooperative launch: the grid barriers need every CTA co-resident, which a
  // cooperative launch guarantees (or refuses) instead of assuming it
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(o->grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = o->smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, kern, args);
  if (e != cudaSuccess) return cuda_status(e, "decode_pass launch");
  return MOBILE_OK;
}

// ---------------------------------------------------------------- zero-sync offload pass
// One launch runs the whole pass; this host loop is StreamSimulator.run_pass
// (engine.py:121-169) against the running kernel:
//   per layer l: unpin layer l-1 (engine.py:152-153) -> issue window
//   (planned pass, engine.py:98-119) -> the layer's selection (planned: the
//   replayed targets; demand: published by the kernel into mapped memory, the
//   host's sync point) -> request + pin, misses issued (engine.py:137-145) ->
//   (slot, ticket) of every selected expert back to the kernel.
// Cache decisions are the same function of the request sequence as in the
// segmented driver; copies overlap the kernel's hits / shared experts / next
// phases instead of waiting for a launch boundary.
namespace {
struct ZsWait {
  volatile unsigned* prog;  // the runtime's mapped progress mirror
  unsigned need;
};
int zs_wait_progress(void* ctx) {  // deadlock stall: the kernel consumed every earlier layer
  auto* w = (ZsWait*)ctx;
  volatile unsigned* pr = w->prog;
  const auto t0 = std::chrono::steady_clock::now();
  while ((int)(*pr - w->need) < 0) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
      set_error("decode_pass: zero-sync stall timed out waiting for kernel progress (need %u, at %u)", w->need,
                (unsigned)*pr);
      return MOBILE_ERR_CUDA;
    }
  }
  return MOBILE_OK;
}
}  // namespace

int mobile_dp_run_offload_pass(mobile_dp* dp, mobile_offload* o, int planned, const int* targets, int k, int lookahead,
                               void* stream, int* fresh_out) {
  Plan& P = dp->plan;
  const int L = P.L, E = P.E;
  if (!dp->h_route) {
    const unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
    if (cudaHostAlloc((void**)&dp->h_route, sizeof(int) * L * (E + 1), fl) != cudaSuccess ||
        cudaHostAlloc((void**)&dp->h_route_flag, sizeof(int) * L, fl) != cudaSuccess ||
        cudaHostAlloc((void**)&dp->h_slots, sizeof(int) * L * E * 2, fl) != cudaSuccess ||
        cudaHostAlloc((void**)&dp->h_slots_flag, sizeof(int) * L, fl) != cudaSuccess) {
      set_error("decode_pass: mapped host allocation failed");
      return MOBILE_ERR_CUDA;
    }
    if (cudaMalloc((void**)&dp->d_slots, sizeof(int) * L * E * 2) != cudaSuccess ||
        cudaMalloc((void**)&dp->d_slots_flag, sizeof(int) * L) != cudaSuccess ||
        cudaMemset(dp->d_slots_flag, 0, sizeof(int) * L) != cudaSuccess) {
      set_error("decode_pass: device slot-table allocation failed");
      return MOBILE_ERR_CUDA;
    }
    P.zs_slots_d = dp->d_slots;
    P.zs_slots_flag_d = dp->d_slots_flag;
    std::memset(dp->h_route_flag, 0, sizeof(int) * L);
    std::memset(dp->h_slots_flag, 0, sizeof(int) * L);
    void *d1, *d2, *d3, *d4;
    cudaHostGetDevicePointer(&d1, dp->h_route, 0);
    cudaHostGetDevicePointer(&d2, dp->h_route_flag, 0);
    cudaHostGetDevicePointer(&d3, dp->h_slots, 0);
    cudaHostGetDevicePointer(&d4, dp->h_slots_flag, 0);
    P.zs_route_h = (int*)d1;
    P.zs_route_flag_h = (int*)d2;
    P.zs_slots_h = (const int*)d3;
    P.zs_slots_flag_h = (const int*)d4;
  }
  void *done = nullptr, *prog = nullptr, *mirror_d = nullptr, *mirror_h = nullptr;
  if (int rc = mobile_offload_zs_enable(o, &done, &prog, &mirror_d, &mirror_h)) return rc;
  P.zs_done = (const unsigned*)done;
  P.zs_prog = (unsigned*)prog;
  P.zs_prog_h = (unsigned*)mirror_d;
  P.zs = 1;
  P.zs_epoch = ++dp->epoch;
  long long* pbase = mobile_offload_zs_base(o);  // shared by every pass kind on this runtime
  P.zs_prog_base = (unsigned)*pbase;
  const unsigned base = (unsigned)*pbase;
  int rc = mobile_dp_launch(dp, -1, stream);
  P.zs = 0;
  if (rc) return rc;
  volatile int* route_flag = dp->h_route_flag;
  volatile int* slots_flag = dp->h_slots_flag;
  std::vector<std::tuple<int, int, int>> waiting;  // (earliest_issue_layer, layer, expert), policy.py:86-106
  if (planned) {
    for (int l = 0; l < L; ++l)
      for (int j = 0; j < k; ++j) waiting.emplace_back(std::max(0, l - lookahead), l, targets[l * k + j]);
    std::sort(waiting.begin(), waiting.end());
  }
  std::vector<int> prev, cur, out2;
  int fresh = 0;
  for (int l = 0; l < L; ++l) {
    if (l > 0) mobile_offload_zs_release(o, l - 1, prev.data(), (int)prev.size(), (long long)base + l);
    if (planned) {  // speculative issue window at the layer boundary
      std::vector<std::tuple<int, int, int>> kept;
      size_t i = 0;
      for (; i < waiting.size(); ++i) {
        const auto& en = waiting[i];
        if (std::get<0>(en) > l) break;
        if (std::get<1>(en) < l) continue;
        int st = 0;
        const int r = mobile_offload_zs_prefetch(o, std::get<1>(en), std::get<2>(en), &st);
        if (r == MOBILE_ERR_DEFERRED) kept.push_back(en);
        else if (r != MOBILE_OK) return r;
      }
      kept.insert(kept.end(), waiting.begin() + i, waiting.end());
      waiting.swap(kept);
      cur.assign(targets + l * k, targets + (l + 1) * k);
    } else {  // the kernel publishes the layer's selection: the pass's sync point
      const auto t0 = std::chrono::steady_clock::now();
      while (route_flag[l] != (int)P.zs_epoch) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
          set_error("decode_pass: zero-sync pass timed out waiting for layer %d routing", l);
          return MOBILE_ERR_CUDA;
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      mobile_offload_sync(o);
      const int* r = dp->h_route + (size_t)l * (E + 1);
      cur.assign(r + 1, r + 1 + r[0]);
    }
    out2.resize(2 * cur.size());
    int issued = 0;
    ZsWait wctx{(volatile unsigned*)mirror_h, base + (unsigned)l};
    if (int r = mobile_offload_zs_require(o, l, cur.data(), (int)cur.size(), out2.data(), &issued, zs_wait_progress, &wctx))
      return r;
    fresh += issued;
    int* tbl = dp->h_slots + (size_t)l * E * 2;
    for (size_t i = 0; i < cur.size(); ++i) {
      tbl[2 * cur[i]] = out2[2 * i];
      tbl[2 * cur[i] + 1] = out2[2 * i + 1];
    }
    std::atomic_thread_fence(std::memory_order_release);
    slots_flag[l] = (int)P.zs_epoch;
    prev.swap(cur);
  }
  mobile_offload_zs_release(o, L - 1, prev.data(), (int)prev.size(), (long long)base + L);
  *pbase = (long long)base + L;
  if (fresh_out) *fresh_out = fresh;
  return MOBILE_OK;
}

}  // extern "C"

#ifdef MOBILE_DP_ROUTE_BENCH
extern "C" int mobile_dp_route_bench(mobile_dp* o, int iters, long long* out_dev) {
  mobile::dp::route_bench_kernel<<<1, 32>>>(o->plan, iters, out_dev);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -1;
}
#endif
