/*
 * mobile.h -- C ABI of the B200-native MoBiLE MoE layer (libmobile.so).
 *
 * The reference (`moesim`, /root/reference/pkg/src/moesim) is pure Python with
 * no FFI layer: its MoE block is inlined in `toymoe.forward`
 * (toymoe.py:188-207) and the decision/plan/cache logic lives in policy.py and
 * memory.py.  Each entry point below replaces one of those reference
 * operations; the citation next to it names the reference code it stands in
 * for.  The Python package `paper_2510_12357_b200` binds these with ctypes
 * (see INTEGRATION.md for the binding a maintainer would add to `moesim`).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device buffers are caller-owned; kernels
 *    never allocate.  `stream` is a cudaStream_t passed as void*.
 *  - Every function returns a status code (MOBILE_OK == 0); no exceptions
 *    cross the ABI.  The Python layer maps codes back to the reference's
 *    exception types and message substrings (ValueError "exceeds",
 *    "finite", "empty", ...; CapacityDeadlock).
 *  - Matrices are row-major.  Weights use the "out-major" layout
 *    (rows = output features, contiguous over the input dimension), i.e. the
 *    transpose of the reference's `h @ W` matrices.
 *  - Determinism: no float atomics; every reduction has a fixed order.
 */
#ifndef MOBILE_H_
#define MOBILE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define MOBILE_OK 0
#define MOBILE_ERR_INVALID 1      /* bad argument / shape ("shape", "empty") */
#define MOBILE_ERR_K_EXCEEDS 2    /* k > E  (toymoe.py:83-84 "exceeds")      */
#define MOBILE_ERR_NONFINITE 3    /* non-finite logits (toymoe.py:85-86)     */
#define MOBILE_ERR_CUDA 4         /* CUDA runtime error                      */
#define MOBILE_ERR_DEADLOCK 5     /* CapacityDeadlock (memory.py:137-144)    */
#define MOBILE_ERR_DEFERRED 6     /* speculative request deferred (None)     */
#define MOBILE_ERR_UNSUPPORTED 7  /* shape/dtype outside the kernel's range  */
#define MOBILE_ERR_NOT_FOUND 8    /* key not resident (KeyError)             */

/* ---- dtypes / enums ---------------------------------------------------- */
#define MOBILE_F32 0
#define MOBILE_BF16 1
#define MOBILE_F64 2

#define MOBILE_ACT_RELU 0   /* toymoe.py:203  relu(h W_in) W_out        */
#define MOBILE_ACT_SWIGLU 1 /* extension:     (silu(h W1) * h W3) W2    */

#define MOBILE_GATE_SELECTED_SOFTMAX 0 /* toymoe.py:201 softmax(logits[sel]) */
#define MOBILE_GATE_SOFTMAX_ALL 1      /* HF norm_topk_prob=False (extension) */

#define MOBILE_STATUS_HIT 0       /* memory.py:20 */
#define MOBILE_STATUS_IN_FLIGHT 1 /* memory.py:21 */
#define MOBILE_STATUS_ISSUED 2    /* memory.py:22 */

int mobile_version(void);
const char* mobile_last_error(void);
int mobile_num_sms(void);

/* ---- router ------------------------------------------------------------
 * Replaces toymoe.py:188-201 (h2 = LN(x); logits = h2 @ router; per-position
 * top_k with the stable lower-index tie rule; final-position replay of
 * recorded logits; gate softmax over the selected logits) for T tokens.
 *   x        (T, d) f32 residual stream (LN is applied in-kernel)
 *   h2_out   (T, d) f32 normalised activations (consumed by the experts)
 *   w_router (E + n_extra, d) out-major router weight, w_dtype; rows E.. are
 *            extra GEMV rows (e.g. Qwen's sigmoid shared-expert gate) whose
 *            logits go to extra_out (T, n_extra) and never enter top-k
 *   k_tok    (T,) int32 per-token width (little = k_little, big = k_big)
 *   replay   (T, E) f32 recorded logits, used where replay_mask[t] != 0
 *   logits_out (T, E) f32 own router logits (h_s rows)
 *   idx_out  (T, k_max) int32 selection (descending), -1 beyond k_tok[t]
 *   gates_out (T, k_max) f32 gate weights in selection order, 0 beyond k_tok
 *   flags    (1,) int32 device word; bit 0 set if any logit was non-finite,
 *            bit 1 if any k_tok[t] > E.  Caller zeroes it.
 *   perm_*   optional mobile_permute outputs (offsets, sorted_pairs, active):
 *            when given, the permute is fused into the router's leader CTA
 *            for decode-sized launches (T <= 4, T*k_max <= 32) and run as a
 *            separate kernel otherwise -- same results either way.
 */
int mobile_router_topk(const float* x, float* h2_out, const void* w_router, int w_dtype,
                       int T, int d, int E, int n_extra, int k_max, const int* k_tok,
                       const float* replay, const uint8_t* replay_mask, int reuse_gates,
                       int gate_norm, float* logits_out, float* extra_out, int* idx_out,
                       float* gates_out, int* flags, int* perm_offsets, int* perm_pairs,
                       int* perm_active, void* stream);
/* The same, and once the selection is known the launch also moves each
 * selected expert's first pf_bytes (at pf_base + e * pf_stride, resident
 * expert pool) toward L2 (cp.async.bulk.prefetch.L2: no result changes; the
 * routed gate-up launch that follows finds its first tiles in L2).
 * pf_base NULL = mobile_router_topk. */
int mobile_router_topk_pf(const float* x, float* h2_out, const void* w_router, int w_dtype,
                          int T, int d, int E, int n_extra, int k_max, const int* k_tok,
                          const float* replay, const uint8_t* replay_mask, int reuse_gates,
                          int gate_norm, float* logits_out, float* extra_out, int* idx_out,
                          float* gates_out, int* flags, int* perm_offsets, int* perm_pairs,
                          int* perm_active, const void* pf_base, long long pf_stride, long long pf_bytes,
                          void* stream);

/* Row-wise top-k (toymoe.py:80-88) over R rows of E logits (f32 or f64):
 * used by top_k(), build_mobile_plan (policy.py:98-103) and
 * selections_from_logits (engine.py:76-81). -0.0 ties +0.0; subnormals are
 * ordered (no FTZ). */
int mobile_topk_rows(const void* rows, int dtype, int R, int E, int k, int* idx_out, int* flags,
                     void* stream);

/* ---- head + confidence -------------------------------------------------
 * Replaces toymoe.py:209-210 + 273 and policy.py:69-79 for T rows:
 *   logits = LN(x[t]) @ head * logit_scale; conf[t] = max softmax(logits);
 *   argmax[t] = first maximiser; fallback[t] = conf[t] <= gamma (strict >
 *   accepts).  logits_out (T, V) may be NULL.  workspace >= head_ws_bytes.
 */
size_t mobile_head_ws_bytes(int T, int V);
int mobile_head_confidence(const float* x, const void* w_head, int w_dtype, int T, int d, int V,
                           float logit_scale, float gamma, float* logits_out, float* conf_out,
                           int* argmax_out, uint8_t* fallback_out, void* workspace, void* stream);

/* The head's outputs from precomputed raw logits rows (T, V) f32 (large-batch
 * decode, where LN(x) @ head runs as a tcgen05 GEMM): l = raw * logit_scale,
 * conf / argmax / fallback exactly as mobile_head_confidence. */
int mobile_logits_confidence(const float* logits, int T, int V, float logit_scale, float gamma,
                             float* conf_out, int* argmax_out, uint8_t* fallback_out, void* stream);

/* probs = softmax(logits) row-wise (toymoe.py:91-94), T rows of V; f32/f64
 * in, f32/f64 out (f64 accumulation when either side is f64). */
int mobile_softmax_rows(const void* logits, int in_dtype, void* probs, int out_dtype, int T, int V,
                        void* stream);

/* should_fallback on a caller-provided probability row (policy.py:69-79):
 * out[0] = sum (f64), out[1] = max (f64); fallback = max <= gamma. */
int mobile_probs_check(const void* probs, int dtype, int V, double* out, void* stream);

/* ---- permute ------------------------------------------------------------
 * Deterministic stable counting sort of (token, slot) pairs by expert
 * (replaces the implicit token-major loop toymoe.py:193-204).
 *   idx (T, k_max), k_tok (T,)
 *   offsets (E+1): pairs of expert e are sorted_pairs[offsets[e]:offsets[e+1]]
 *   sorted_pairs (T*k_max): pair id p = t*k_max + j, token-major within expert
 *   active (E+1): active[0] = number of experts with >= 1 pair, then their ids
 */
int mobile_permute(const int* idx, const int* k_tok, int T, int k_max, int E, int* offsets,
                   int* sorted_pairs, int* active, void* stream);

/* ---- bulk-copy streaming GEMV (decode engine) -----------------------------
 * One launch computes several groups of weight-row dot products, streaming
 * weights through shared memory with cp.async.bulk on an mbarrier ring.
 * Weights are row-major (out-major); rows are streamed in tiles of 16 rows x
 * 4 KB of K (one contiguous copy when the row fits, else one copy per row).
 * Group semantics (per pair p of expert e; pairs grouped by mobile_permute):
 *   epi 0 STORE : out[p, r] = (residual[p, r] +) x[p / x_div] . W_e[r]
 *   epi 1 RELU  : out[p, r] = max(x[p / x_div] . W_e[r], 0)
 *   epi 2 SWIGLU: rows in 16-row groups [8 gate | 8 up] ->
 *                 out[p, f] = silu(g_f) * u_f,  out_dim = rows / 2
 * active == NULL means one dense "expert" (weights at w_base) applied to
 * pairs 0..dense_T-1.  max_tokens bounds tokens per expert (1..4 fast path;
 * more are processed in chunks of 4).
 */
typedef struct {
  const void* w_base;
  long long stride;
  const int* slot;
  const float* x;
  int x_div;
  const int* offsets;
  const int* pairs;
  const int* active;
  int dense_T;
  int max_active;
  int K;
  int rows;
  float* out;
  const float* residual;
  int epi;
  int prefetch;  /* 1: weights AND expert lists do not depend on the previous kernel
                    (dense / shared experts): copies may start before the PDL wait */
} mobile_sg_group;
int mobile_stream_gemv(const mobile_sg_group* groups, int n_groups, int w_dtype, int max_tokens,
                       void* stream);
/* Output head + confidence on the same engine (toymoe.py:209-210, 273;
 * policy.py:69-79): logits = x_ln[t] . head_row * scale (x_ln already
 * layer-normalised), conf[t] = max softmax, first argmax, fallback =
 * conf <= gamma.  T <= 4.  workspace >= mobile_stream_head_ws_bytes(), zeroed
 * once (the kernel leaves it zeroed). */
size_t mobile_stream_head_ws_bytes(void);
int mobile_stream_head(const float* x_ln, int T, int d, const void* w_head, int w_dtype, int V,
                       float logit_scale, float gamma, float* logits_out, float* conf_out, int* argmax_out,
                       uint8_t* fallback_out, void* workspace, void* stream);

/* ---- grouped expert GEMM on tcgen05 (prefill / batched) -------------------
 * D_e = A_e . B_e^T, bf16 x bf16 -> f32 accumulate in TMEM, TMA-fed
 * (SWIZZLE_128B, 4-stage mbarrier ring), one 128 x 128 tile per CTA.
 *   A  (rows_a, K) bf16 row-major: expert-sorted activations; expert e owns
 *      rows offsets[e]..offsets[e+1] (active = [n, ids]); with offsets NULL,
 *      "dense" mode: each of dense_experts B experts sees rows 0..dense_rows.
 *   B  expert weights (N, K) bf16 row-major at B_base + slot[e]*b_expert_stride
 *      (n_slots experts addressable; slot NULL = identity).
 *   epi 0: out_f32[row_to_pair[r] * ldo + e*out_expert_stride + n] = D (f32)
 *   epi 1: SwiGLU on 16-column groups [8 gate | 8 up] -> bf16
 *          out_bf16[r * ldo + e*out_expert_stride + f]
 *   epi 2: bf16 store of D.
 *   epi 3: out_f32[r * ldo + e*out_expert_stride + n] += D (residual
 *          projections of the large-batch decode step: out holds x).
 * K % 64 == 0, N % 128 == 0; max_tiles bounds the number of 128x128 tiles
 * (surplus CTAs exit); the tile list is derived on the device. */
int mobile_grouped_gemm(const void* A, int rows_a, int K, const void* B_base, long long b_expert_stride,
                        int n_slots, int N, const int* offsets, const int* active, const int* slot, int max_tiles,
                        int dense_rows, int dense_experts, int epi, float* out_f32, void* out_bf16, int ldo,
                        int out_expert_stride, const int* row_to_pair, void* stream);
/* X[r, :] = bf16(src[pairs[r] / div, :]) (pairs NULL: row r) -- the expert-
 * sorted activation matrix for mobile_grouped_gemm. */
int mobile_gather_bf16(const float* src, const int* pairs, int div, int P, int d, void* X, void* stream);
/* the same gather from bf16 source rows (expert-parallel mailbox rows) */
int mobile_gather_rows_bf16(const void* src, const int* pairs, int div, int P, int d, void* X, void* stream);
/* X[r] = bf16(LN(src[pairs[r] / div])) (pairs NULL: row r): the pre-MoE
 * LayerNorm (toymoe.py:129-132, 188) with the router kernel's reduction
 * order, so X equals bf16 of the router's h2 rows bit for bit (the shared
 * experts of a batch start from the residual, concurrently with routing). */
int mobile_gather_ln_bf16(const float* src, const int* pairs, int div, int P, int d, void* X, void* stream);

/* ---- combine -------------------------------------------------------------
 * toymoe.py:192, 204, 207:  moe = sum_j gates[t,j] * Y[t*k_max + j] (selection
 * order), then + shared (optionally sigmoid(shared_logit[t,s]) * Ys[t][s]),
 * x_out[t] = x[t] + moe.  Y_shared is (T, n_shared, d) or NULL.  If ln_out is
 * non-NULL it also receives LN(x_out[t]) (the next layer's attention input).
 */
int mobile_combine(const float* x, const float* Y, const float* gates, const int* k_tok, int T,
                   int k_max, int d, const float* Y_shared, int n_shared,
                   const float* shared_logits, float* x_out, float* ln_out, void* stream);

/* ---- decode-step kernels around the layer --------------------------------
 * (toymoe.py:171-186 semantics, KV-cached, position read from device memory
 * so a whole decode step can be captured in one CUDA graph.)
 *   dense_gemv: y[t, r] = (residual ? residual[t, r] : 0) + (LN?(x[t])) . W[r]
 *               W (N, d) out-major, T <= 8 rows (attention q/k/v and o).
 *   attn_decode: qkv (B, 3d); writes k/v at pos[b] into k/v caches
 *               (B, H, max_len, d/H) f32 (head-major), out (B, d) = softmax(q k^T / sqrt(hd)) v.
 *   embed:      x[b] = embed[tok[b]] + pe[pos[b]]  (pe = sinusoidal table);
 *               ln_out (optional) = LN(x[b]).
 *   advance:    pos[b] += 1; tok[b] = next_tok[b] if next_tok.
 */
int mobile_dense_gemv(const float* x, int T, int d, int do_ln, const void* w, int w_dtype, int N,
                      const float* residual, float* y, void* stream);
int mobile_attn_decode(const float* qkv, float* k_cache, float* v_cache, const int* pos, int B, int d,
                       int H, int max_len, float* out, void* stream);
/* Split-KV variant (few (sequence, head) pairs on a long cache): positions are
 * split over ~2 x SMs CTAs, each writes its (m, s, o) partial into the CALLER-
 * OWNED workspace `ws` and takes a ticket; the (sequence, head)'s last split
 * merges the partials in split order (deterministic).  mobile_attn_split_ws
 * returns the sizes (0 = no split for this shape); tickets must be zeroed once
 * and are left zero by every launch.  One workspace per concurrently running
 * caller (stream / captured graph).  Without a workspace (or too small) the
 * kernel runs unsplit.  Grouped-query attention: Hkv key/value heads (H % Hkv
 * == 0), qkv rows (B, d + 2 Hkv hd) = [q | k | v], caches (B, Hkv, max_len,
 * hd); query head h reads key/value head h / (H / Hkv).  mobile_attn_decode
 * = mobile_attn_decode_ws with Hkv = H and no workspace. */
int mobile_attn_split_ws(int B, int d, int H, int max_len, int* ws_floats, int* n_tickets);
int mobile_attn_decode_ws(const float* qkv, float* k_cache, float* v_cache, const int* pos, int B, int d,
                          int H, int Hkv, int max_len, float* out, float* ws, unsigned* tickets, int ws_floats,
                          int n_tickets, void* stream);
int mobile_embed(const int* tok, const int* pos, const float* embed, const float* pe, int B, int d, float* x,
                 float* ln_out, void* stream);
int mobile_advance(int* pos, int B, int* tok, const int* next_tok, void* stream);
/* cudaMemcpyAsync(kind = default) on `stream` (graph-capturable H2D/D2H of
 * pinned slot tables and routing lists). */
int mobile_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---- expert parallelism over peer memory (ep_p2p.cu) ---------------------
 * Replaces the dispatch / combine all-to-alls of the expert-parallel layer
 * (ep.py) with direct peer stores on an NVSwitch node.  Every
 * rank owns a mailbox (mobile_ep_mailbox_create) whose CUDA IPC handle is
 * exchanged once (mobile_ep_ipc_handle / _open); peers_dev is a device array
 * of the G mailboxes as mapped in this process (this rank's own at [rank]).
 * Per layer, with an epoch that advances per exchange: the effective epoch is
 * `epoch` + *epoch_dev when epoch_dev is non-NULL -- a device counter bumped
 * by mobile_ep_advance at the start of each exchange, so a CUDA graph of the
 * exchange replays correctly (every rank runs every exchange, in lockstep):
 *   home : mobile_ep_dispatch  -- plan (stable per-owner positions, dest_pos
 *          (T*k_max) scratch, counts (G) scratch), row stores into the
 *          owners' mailboxes, counts + release flag (system scope)
 *   owner: mobile_ep_wait(which=0) -- acquire every source's flag, write
 *          k_tok_out (G*cap) = 1 for the received rows; run the experts on
 *          the mailbox rows; mobile_ep_return -- output rows back + flag
 *   home : mobile_ep_wait(which=1); mobile_ep_collect -- Y (T*k_max, d) in
 *          pair order (zero rows for unselected slots), then the combine.
 * rows_bf16 = 1: the dispatched rows are stored as bf16 (half the link bytes;
 * the owner's tcgen05 experts consume bf16 activations), packed at d * 2
 * bytes per row inside the mailbox's row area; 0: f32 rows.
 * cap = rows a source may send one owner (T_max * k_max covers the worst case;
 * overflow sets flags bit 0).  A wait that does not see its flags in 10 s
 * traps (flags bit 1).  G <= 8. */
size_t mobile_ep_mailbox_bytes(int G, int cap, int d);
int mobile_ep_mailbox_create(int G, int cap, int d, void** mailbox);
int mobile_ep_mailbox_destroy(void* mailbox);
int mobile_ep_ipc_handle(void* mailbox, void* handle64);
int mobile_ep_ipc_open(const void* handle64, void** ptr);
int mobile_ep_ipc_close(void* ptr);
int mobile_ep_dispatch(const float* rows, const int* idx, const int* k_tok, int T, int k_max, int d, const int* owner,
                       const int* local_id, void* const* peers_dev, int G, int rank, int cap, unsigned epoch,
                       const unsigned* epoch_dev, int rows_bf16, int* dest_pos, int* counts, int* flags,
                       void* stream);
int mobile_ep_wait(void* mailbox, int G, int cap, int d, int which, unsigned epoch, const unsigned* epoch_dev,
                   int* k_tok_out, int* flags, void* stream);
int mobile_ep_return(const float* out_rows, const void* mailbox, void* const* peers_dev, int G, int rank, int cap,
                     int d, unsigned epoch, const unsigned* epoch_dev, void* stream);
int mobile_ep_advance(unsigned* epoch_dev, void* stream);
int mobile_ep_collect(const void* mailbox, const int* dest_pos, int P, int G, int cap, int d, float* Y, void* stream);

/* ---- expert cache core (memory.py:65-181 semantics) ----------------------
 * LRU of (layer, expert) keys with pins, in-flight protection, speculative
 * deferral, CapacityDeadlock.  Each resident entry owns a physical slot
 * index in [0, slots).  Times are doubles: the simulator mirror passes the
 * reference's clock; the device runtime passes a logical clock.
 * If `channel` is non-NULL an issue completes at channel->issue(now)
 * (memory.py:38-43); otherwise at `ready_if_issued`.
 */
typedef struct mobile_cache mobile_cache;
typedef struct {
  double t_xfer;
  double busy_until;
  long long transfers_issued;
} mobile_channel;

mobile_cache* mobile_cache_create(int slots);
void mobile_cache_destroy(mobile_cache* c);
int mobile_cache_request(mobile_cache* c, int layer, int expert, double now, int speculative,
                         mobile_channel* channel, double ready_if_issued, int* status_out,
                         double* ready_out, int* slot_out);
int mobile_cache_pin(mobile_cache* c, int layer, int expert);
int mobile_cache_unpin(mobile_cache* c, int layer, int expert);
int mobile_cache_token_end(mobile_cache* c);
/* evict the n LRU unpinned entries with ready <= now (now = +inf: only pins
 * block); writes victims as (layer, expert) pairs; all-or-nothing. */
int mobile_cache_evict_lru(mobile_cache* c, int n, double now, int* victims_out, int* n_out);
int mobile_cache_size(const mobile_cache* c);
int mobile_cache_contains(const mobile_cache* c, int layer, int expert);
int mobile_cache_lookup(const mobile_cache* c, int layer, int expert, double* ready_out,
                        int* slot_out);
int mobile_cache_set_ready(mobile_cache* c, int layer, int expert, double ready);
/* entries in LRU -> MRU order as (layer, expert) pairs; cap = pairs room */
int mobile_cache_entries(const mobile_cache* c, int* out, int cap);
/* stats: hits, coalesced, issued, evictions, deferrals */
int mobile_cache_stats(const mobile_cache* c, long long* out5);

/* ---- device expert store + copy engine ------------------------------------
 * The engine.py:98-169 protocol on real hardware: an HBM slot pool, a pinned
 * host store of every (layer, expert) in device layout, cudaMemcpyAsync on a
 * side copy stream, one completion event per slot copy and one last-use event
 * per slot on the compute stream (a slot is never overwritten while a kernel
 * may still read it).  Cache decisions run through mobile_cache with a
 * logical clock: an issued entry stays "in flight" until the compute stream
 * has waited on it and the host has passed a sync point (mobile_offload_sync).
 */
typedef struct mobile_offload mobile_offload;
mobile_offload* mobile_offload_create(int slots, long long expert_bytes, void* slot_pool,
                                      const void* host_store, long long host_layer_stride,
                                      long long host_expert_stride, int num_layers,
                                      int num_experts, void* copy_stream);
void mobile_offload_destroy(mobile_offload* o);
/* Required loads for one layer (engine.py:137-145): request + pin each expert,
 * issue copies for misses, make `compute_stream` wait on every copy, write the
 * slot of each expert into slot_table_host[expert] (pinned, E ints). Counts
 * fresh transfers in *issued_out. */
int mobile_offload_require(mobile_offload* o, int layer, const int* experts, int n,
                           void* compute_stream, int* slot_table_host, int* issued_out);
/* Speculative prefetch (engine.py:98-119 _issue_window): returns DEFERRED
 * when no victim exists. */
int mobile_offload_prefetch(mobile_offload* o, int layer, int expert, int* status_out);
/* After the layer's kernels are enqueued: record each slot's last-use event
 * on compute_stream and unpin (engine.py:152-153). */
int mobile_offload_release(mobile_offload* o, int layer, const int* experts, int n,
                           void* compute_stream);
/* Host passed a synchronisation point with compute_stream: entries it waited
 * on are settled (logical clock advances). */
int mobile_offload_sync(mobile_offload* o);
int mobile_offload_token_end(mobile_offload* o);
mobile_cache* mobile_offload_cache(mobile_offload* o);
/* Drive one whole pass of L+1 captured graph segments (cudaGraphExec_t
 * handles) with the engine.py:121-169 protocol: planned = 1 replays a known
 * plan (targets (L, k), issue windows max(0, l - lookahead)); planned = 0 loads
 * on demand from the per-layer active lists the segments copy into
 * active_host ((L, E+1) pinned).  Slot tables go to slot_host ((L, E) pinned),
 * which the segments copy to the device. */
int mobile_offload_run_pass(mobile_offload* o, const unsigned long long* graph_execs, int L, void* stream,
                            int planned, const int* active_host, const int* targets, int k, int* slot_host,
                            const void* slot_dev_row, long long slot_row_bytes, int lookahead, int* fresh_out);
/* bytes copied H2D so far, transfers issued */
int mobile_offload_counters(const mobile_offload* o, long long* out2);
/* zero-sync mode (decode_pass.cu): per-slot copy tickets written by the copy
 * stream (cuStreamWriteValue32), slot reuse ordered after the kernel's
 * progress counter (cuStreamWaitValue32) */
int mobile_offload_zs_enable(mobile_offload* o, void** done_out, void** prog_out, void** prog_mirror_dev_out,
                             void** prog_mirror_host_out);
int mobile_offload_zs_require(mobile_offload* o, int layer, const int* experts, int n, int* out2, int* issued_out,
                              int (*wait_fn)(void*), void* wait_ctx);
int mobile_offload_zs_prefetch(mobile_offload* o, int layer, int expert, int* status_out);
int mobile_offload_zs_release(mobile_offload* o, int layer, const int* experts, int n, long long release_prog);
long long* mobile_offload_zs_base(mobile_offload* o); /* progress value at the next pass start (shared by all passes) */


/* ---- persistent decode pass (decode_pass.cu) -------------------------------
 * One launch runs a whole MoBiLE decode pass of B <= 4 sequences at one new
 * position each -- embed, per layer [LN + qkv, KV-cache attention, o +
 * residual, LN + router GEMV (+ shared-gate rows) + shared gate-up, stable
 * top-k / replay / gate softmax + permute, routed gate-up, shared and routed
 * down, weighted combine + residual], head + confidence -- i.e. one pass of
 * toymoe.little_forward / big_forward / full_forward (toymoe.py:143-236) with
 * a KV cache, on 148 persistent CTAs separated by grid barriers.  With
 * `offload` set the pass is cut into L+1 segments after each layer's routing
 * (the active expert list is published to active_out[l] for the host cache,
 * engine.py:121-169), routed experts are read through slot_table (L, E).
 * All pointers are device memory owned by the caller; the handle owns only
 * its program and a small workspace.  `replay` (L, B, E) non-NULL = big pass
 * (selection from the replayed logits, toymoe.py:194-200). */
typedef struct mobile_dp_model {
  int B, L, d, H, V, E, k, n_shared, n_gate, ffn, shared_ffn, activation, gate_norm, reuse_gates;
  int w_dtype, max_len, offload;
  int Hkv;                    /* key/value heads (0 = H; fewer = grouped-query attention) */
  float logit_scale, gamma;
  /* weights (out-major, row-major rows) */
  const void* qkv;            /* (L, d + 2 Hkv hd, d) */
  const void* o;              /* (L, d, d) */
  const void* router;         /* (L, E + n_gate, d) */
  const void* shared;         /* (L, S, shared_stride bytes) packed [W13 | W2] */
  long long shared_stride, shared_w2_offset;
  const void* experts;        /* resident (L, E, expert_stride) or the offload slot pool */
  long long expert_layer_stride, expert_stride, expert_w2_offset;
  const int* slot_table;      /* (L, E) slot of each expert (offload) or NULL */
  const void* head;           /* (V, d) */
  const float* embed;         /* (V, d) f32 */
  const float* pe;            /* (max_len, d) f32 positional rows */
  /* state */
  const int* tok;             /* (B,) input token */
  const int* pos;             /* (B,) position */
  float *kc, *vc;             /* (L, B, Hkv, max_len, d/H) head-major */
  float *x, *xa, *q, *att;    /* (B, d) */
  float *U, *Us, *Y, *Ys;     /* (B*k, ffn), (B*S, shared_ffn), (B*k, d), (B*S, d) */
  float* states;              /* (L, B, E) router logits of this pass */
  float* extra;               /* (L, B, max(n_gate,1)) shared-gate logits */
  const float* replay;        /* (L, B, E) or NULL */
  int* idx_out;               /* (L, B, k) selections */
  float* gates_out;           /* (L, B, k) */
  int* active_out;            /* (L, E + 1) [n, expert ids...] or NULL */
  float* head_logits;         /* (B, V) or NULL */
  float* conf;                /* (B,) max softmax prob */
  int* argmax;                /* (B,) */
  uint8_t* fallback;          /* (B,) conf <= gamma (policy.py:69-79) */
  int* flags;                 /* |= 1 non-finite router logits, 4/8 watchdog, 16 pos >= max_len */
} mobile_dp_model;
typedef struct mobile_dp mobile_dp;
int mobile_dp_create(const mobile_dp_model* m, mobile_dp** out);
void mobile_dp_destroy(mobile_dp* p);
int mobile_dp_num_segments(const mobile_dp* p);
int mobile_dp_info(const mobile_dp* p, int* out4); /* phases, stages, smem bytes, grid */
/* optional device buffer (phases x grid x 6 u64): per phase and CTA the
 * globaltimer at [inputs visible, inputs built, work done, arrival issued,
 * barrier observed, acquire fence done]; NULL = off */
int mobile_dp_set_trace(mobile_dp* p, unsigned long long* trace);
/* optional event log (grid x 2 roles x 1024 x 2 u64: globaltimer, code<<56 | phase<<32 | item); NULL = off */
int mobile_dp_set_events(mobile_dp* p, unsigned long long* evt);
/* watchdog diagnostics (host memory, readable after a trapped launch):
 * [0] 1 = producer stalled / 2 = grid barrier stalled, then CTA, phase, ... */
int mobile_dp_diag(const mobile_dp* p, int* out16);
/* segment = -1: the whole pass; else offload segment 0..L */
int mobile_dp_launch(mobile_dp* p, int segment, void* stream);
/* Zero-sync offloaded pass (one launch): the host runs the engine.py:121-169
 * cache protocol while the kernel runs -- demand passes read each layer's
 * selection from mapped host memory, planned passes (big, replay) use
 * `targets` (L x k); misses are copied on the runtime's copy stream and
 * announced to the kernel with per-slot tickets.  p must be created with
 * offload = 1. */
int mobile_dp_run_offload_pass(mobile_dp* p, mobile_offload* o, int planned, const int* targets, int k,
                               int lookahead, void* stream, int* fresh_out);

#ifdef __cplusplus
}
#endif
#endif /* MOBILE_H_ */
