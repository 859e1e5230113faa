// Device expert store + copy engine: the engine.py:98-169 protocol on real
// hardware (HBM slot pool, pinned host store, cudaMemcpyAsync side stream).
//
// Cache decisions go through mobile_cache (memory.py semantics) driven by a
// LOGICAL clock so that they are a deterministic function of the request
// sequence, independent of copy timing:
//   - a freshly issued entry is in flight (ready = +inf);
//   - when a layer requires it, the compute stream waits on its copy event;
//   - at the next host sync point with the compute stream (mobile_offload_sync)
//     every entry the compute stream waited on is complete, so it settles at
//     the current clock value, and the clock advances.
// A slot is never overwritten while a kernel may still read it: each slot has
// a last-use event recorded on the compute stream after the layer's expert
// kernels, and a new copy into the slot waits on it first.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <tuple>
#include <vector>

#include "../../include/mobile.h"

namespace mobile {
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
}  // namespace mobile

struct mobile_offload {
  mobile_cache* cache = nullptr;
  int slots = 0;
  long long expert_bytes = 0;
  char* pool = nullptr;
  const char* host = nullptr;
  long long layer_stride = 0, expert_stride = 0;
  int L = 0, E = 0;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> copy_done, last_use;
  std::vector<char> last_use_valid;
  std::vector<int> slot_layer, slot_expert;  // occupant of each slot (-1 = none)
  double clock = 0.0;
  std::vector<std::pair<int, int>> awaited;   // waited on since the last sync
  long long bytes = 0, transfers = 0;
  // ---- zero-sync mode (one persistent kernel per pass, see decode_pass.cu)
  unsigned* zs_done = nullptr;                // device: last copy ticket landed per slot (stream-written)
  unsigned* zs_prog = nullptr;                // device: layers whose experts the kernel has consumed
  std::vector<unsigned> zs_ticket;            // per slot: ticket of its latest copy
  std::vector<long long> zs_last_use;         // per slot: progress value that frees it (0 = free)
  long long zs_base = 0;                      // progress value at the start of the next pass
  unsigned* zs_prog_h = nullptr;              // mapped host mirror of zs_prog (the host polls it)
  unsigned* zs_prog_hd = nullptr;             // its device address
};

static const double kInf = std::numeric_limits<double>::infinity();

#define OFF_CUDA(call, where)                                         \
  do {                                                                \
    cudaError_t _e = (call);                                          \
    if (_e != cudaSuccess) return mobile::cuda_status(_e, where);     \
  } while (0)

static int issue_copy(mobile_offload* o, int layer, int expert, int slot) {
  if (o->last_use_valid[slot]) OFF_CUDA(cudaStreamWaitEvent(o->copy, o->last_use[slot], 0), "copy wait last-use");
  const char* src = o->host + (long long)layer * o->layer_stride + (long long)expert * o->expert_stride;
  char* dst = o->pool + (long long)slot * o->expert_bytes;
  OFF_CUDA(cudaMemcpyAsync(dst, src, (size_t)o->expert_bytes, cudaMemcpyHostToDevice, o->copy), "expert H2D");
  OFF_CUDA(cudaEventRecord(o->copy_done[slot], o->copy), "copy event");
  o->slot_layer[slot] = layer;
  o->slot_expert[slot] = expert;
  o->bytes += o->expert_bytes;
  o->transfers++;
  return MOBILE_OK;
}

extern "C" {

mobile_offload* mobile_offload_create(int slots, long long expert_bytes, void* slot_pool,
                                      const void* host_store, long long host_layer_stride,
                                      long long host_expert_stride, int num_layers, int num_experts,
                                      void* copy_stream) {
  if (slots < 1 || expert_bytes <= 0 || !slot_pool || !host_store) {
    mobile::set_error("offload: bad arguments (slots=%d bytes=%lld)", slots, expert_bytes);
    return nullptr;
  }
  auto* o = new mobile_offload();
  o->cache = mobile_cache_create(slots);
  o->slots = slots;
  o->expert_bytes = expert_bytes;
  o->pool = (char*)slot_pool;
  o->host = (const char*)host_store;
  o->layer_stride = host_layer_stride;
  o->expert_stride = host_expert_stride;
  o->L = num_layers;
  o->E = num_experts;
  o->copy = (cudaStream_t)copy_stream;
  o->copy_done.resize(slots);
  o->last_use.resize(slots);
  o->last_use_valid.assign(slots, 0);
  o->slot_layer.assign(slots, -1);
  o->slot_expert.assign(slots, -1);
  for (int s = 0; s < slots; ++s) {
    if (cudaEventCreateWithFlags(&o->copy_done[s], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&o->last_use[s], cudaEventDisableTiming) != cudaSuccess) {
      mobile::set_error("offload: cudaEventCreate failed");
      return nullptr;
    }
  }
  return o;
}

void mobile_offload_destroy(mobile_offload* o) {
  if (!o) return;
  if (o->zs_done) cudaFree(o->zs_done);
  if (o->zs_prog) cudaFree(o->zs_prog);
  if (o->zs_prog_h) cudaFreeHost(o->zs_prog_h);
  for (auto e : o->copy_done) cudaEventDestroy(e);
  for (auto e : o->last_use) cudaEventDestroy(e);
  mobile_cache_destroy(o->cache);
  delete o;
}

static int settle(mobile_offload* o) {
  o->clock += 1.0;
  for (auto& k : o->awaited) {
    double r;
    if (mobile_cache_lookup(o->cache, k.first, k.second, &r, nullptr) == MOBILE_OK && r == kInf)
      mobile_cache_set_ready(o->cache, k.first, k.second, o->clock);
  }
  o->awaited.clear();
  return MOBILE_OK;
}

// Every copy has landed (caller synchronised the copy stream): settle all
// in-flight entries at the next clock value.
static void settle_all(mobile_offload* o) {
  o->clock += 1.0;
  std::vector<int> buf(2 * (size_t)o->slots);
  const int n = mobile_cache_entries(o->cache, buf.data(), o->slots);
  for (int i = 0; i < n; ++i) {
    double r;
    if (mobile_cache_lookup(o->cache, buf[2 * i], buf[2 * i + 1], &r, nullptr) == MOBILE_OK && r == kInf)
      mobile_cache_set_ready(o->cache, buf[2 * i], buf[2 * i + 1], o->clock);
  }
  o->awaited.clear();
}

int mobile_offload_require(mobile_offload* o, int layer, const int* experts, int n,
                           void* compute_stream, int* slot_table_host, int* issued_out) {
  cudaStream_t cs = (cudaStream_t)compute_stream;
  int fresh = 0;
  for (int i = 0; i < n; ++i) {
    const int e = experts[i];
    int status = 0, slot = -1;
    double ready = 0;
    int st = mobile_cache_request(o->cache, layer, e, o->clock, 0, nullptr, kInf, &status, &ready, &slot);
    if (st == MOBILE_ERR_DEADLOCK) {
      // every slot is pinned or in flight: stall until the compute stream has
      // consumed what it waited on and every issued copy has landed, settle,
      // and retry (the simulator's stall); a second failure means every slot
      // is pinned by this layer -- a true CapacityDeadlock.
      OFF_CUDA(cudaStreamSynchronize(cs), "deadlock stall (compute)");
      OFF_CUDA(cudaStreamSynchronize(o->copy), "deadlock stall (copy)");
      settle_all(o);
      st = mobile_cache_request(o->cache, layer, e, o->clock, 0, nullptr, kInf, &status, &ready, &slot);
    }
    if (st != MOBILE_OK) return st;
    if (status == MOBILE_STATUS_ISSUED) {
      int r = issue_copy(o, layer, e, slot);
      if (r) return r;
      ++fresh;
    }
    mobile_cache_pin(o->cache, layer, e);
    if (ready == kInf) {
      OFF_CUDA(cudaStreamWaitEvent(cs, o->copy_done[slot], 0), "compute wait copy");
      o->awaited.emplace_back(layer, e);
    }
    if (slot_table_host) slot_table_host[e] = slot;
  }
  if (issued_out) *issued_out = fresh;
  return MOBILE_OK;
}

int mobile_offload_prefetch(mobile_offload* o, int layer, int expert, int* status_out) {
  int status = 0, slot = -1;
  double ready = 0;
  int st = mobile_cache_request(o->cache, layer, expert, o->clock, 1, nullptr, kInf, &status, &ready, &slot);
  if (st != MOBILE_OK) return st;  // DEFERRED: retry at the next boundary
  if (status == MOBILE_STATUS_ISSUED) {
    int r = issue_copy(o, layer, expert, slot);
    if (r) return r;
  }
  if (status_out) *status_out = status;
  return MOBILE_OK;
}

int mobile_offload_release(mobile_offload* o, int layer, const int* experts, int n, void* compute_stream) {
  cudaStream_t cs = (cudaStream_t)compute_stream;
  for (int i = 0; i < n; ++i) {
    int slot = -1;
    if (mobile_cache_lookup(o->cache, layer, experts[i], nullptr, &slot) == MOBILE_OK) {
      OFF_CUDA(cudaEventRecord(o->last_use[slot], cs), "last-use event");
      o->last_use_valid[slot] = 1;
    }
    mobile_cache_unpin(o->cache, layer, experts[i]);
  }
  return MOBILE_OK;
}

int mobile_offload_sync(mobile_offload* o) { return settle(o); }

int mobile_offload_token_end(mobile_offload* o) {
  // Prefetches never consumed by a layer are drained here so no entry stays
  // in flight across tokens (deterministic: the copy stream is synchronised).
  OFF_CUDA(cudaStreamSynchronize(o->copy), "token_end drain");
  settle_all(o);
  return mobile_cache_token_end(o->cache);
}

mobile_cache* mobile_offload_cache(mobile_offload* o) { return o->cache; }

// One whole pass of an offloaded decode step, driven from C++ so the per-layer
// host work is a few microseconds: graph segment l = [experts(l-1), attention
// + routing(l)], segment L = [experts(L-1), head] (runtime.py captures them).
// The order of operations is StreamSimulator.run_pass (engine.py:121-169):
//   planned pass: (1) speculative issue window at the layer boundary
//                 (engine.py:98-119: stale entries dropped, deferred retried)
//   both:         (2) attention/routing (segment l) ...
//   demand pass:  ... host reads layer l's active experts (the only sync)
//   both:         (3) request + pin, issue misses, (4) compute waits on copies,
//                 (5) experts run in segment l+1, (6) unpin after it is enqueued
int mobile_offload_run_pass(mobile_offload* o, const unsigned long long* graph_execs, int L, void* stream,
                            int planned, const int* active_host, const int* targets, int k, int* slot_host,
                            const void* slot_dev_row, long long slot_row_bytes, int lookahead, int* fresh_out) {
  cudaStream_t cs = (cudaStream_t)stream;
  const int E = o->E;
  int fresh = 0;
  // planned pass: entries sorted by (earliest_issue_layer, layer, expert) (policy.py:86-106)
  std::vector<std::tuple<int, int, int>> waiting;
  if (planned) {
    for (int l = 0; l < L; ++l)
      for (int j = 0; j < k; ++j) waiting.emplace_back(std::max(0, l - lookahead), l, targets[l * k + j]);
    std::sort(waiting.begin(), waiting.end());
  }
  std::vector<int> prev, cur;
  for (int l = 0; l < L; ++l) {
    OFF_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph_execs[l], cs), "segment launch");  // (5) of l-1, (2)
    if (l > 0) {  // (6) unpin layer l-1 before layer l's window, as engine.py:152-153 -> 131
      if (int rc = mobile_offload_release(o, l - 1, prev.data(), (int)prev.size(), stream)) return rc;
    }
    if (planned) {  // (1) issue window
      std::vector<std::tuple<int, int, int>> kept;
      size_t i = 0;
      for (; i < waiting.size(); ++i) {
        const auto& en = waiting[i];
        if (std::get<0>(en) > l) break;
        if (std::get<1>(en) < l) continue;  // stale: its layer already executed
        int st = 0;
        const int rc = mobile_offload_prefetch(o, std::get<1>(en), std::get<2>(en), &st);
        if (rc == MOBILE_ERR_DEFERRED) kept.push_back(en);
        else if (rc != MOBILE_OK) return rc;
      }
      kept.insert(kept.end(), waiting.begin() + i, waiting.end());
      waiting.swap(kept);
    }
    cur.clear();
    if (planned) {
      cur.assign(targets + l * k, targets + (l + 1) * k);
    } else {  // the layer's selection comes back to the host
      OFF_CUDA(cudaStreamSynchronize(cs), "routing sync");
      settle(o);
      const int* a = active_host + (size_t)l * (E + 1);
      cur.assign(a + 1, a + 1 + a[0]);
    }
    int issued = 0;  // (3) + (4)
    if (int rc = mobile_offload_require(o, l, cur.data(), (int)cur.size(), stream, slot_host + (size_t)l * E, &issued))
      return rc;
    fresh += issued;
    prev.swap(cur);
  }
  OFF_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph_execs[L], cs), "segment launch");  // (5) experts(L-1) + head
  if (int rc = mobile_offload_release(o, L - 1, prev.data(), (int)prev.size(), stream)) return rc;
  (void)slot_dev_row;
  (void)slot_row_bytes;
  if (fresh_out) *fresh_out = fresh;
  return MOBILE_OK;
}

// ---------------------------------------------------------------- zero-sync
// The copy for slot s is ordered after the kernel's release of the slot's
// previous occupant with cuStreamWaitValue32 on the kernel's progress counter,
// and announces completion with cuStreamWriteValue32(done[s], ticket): the
// kernel streams an expert's tiles once done[s] >= its ticket.  No host sync.
int mobile_offload_zs_enable(mobile_offload* o, void** done_out, void** prog_out, void** prog_mirror_dev_out,
                             void** prog_mirror_host_out) {
  if (!o->zs_done) {
    void* hd = nullptr;
    if (cudaMalloc(&o->zs_done, sizeof(unsigned) * o->slots) != cudaSuccess ||
        cudaMemset(o->zs_done, 0, sizeof(unsigned) * o->slots) != cudaSuccess ||
        cudaMalloc(&o->zs_prog, sizeof(unsigned) * 4) != cudaSuccess ||
        cudaMemset(o->zs_prog, 0, sizeof(unsigned) * 4) != cudaSuccess ||
        cudaHostAlloc((void**)&o->zs_prog_h, sizeof(unsigned) * 4, cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess ||
        cudaHostGetDevicePointer(&hd, o->zs_prog_h, 0) != cudaSuccess) {
      mobile::set_error("offload: zero-sync state allocation failed");
      return MOBILE_ERR_CUDA;
    }
    o->zs_prog_h[0] = 0u;
    o->zs_prog_hd = (unsigned*)hd;
    o->zs_ticket.assign(o->slots, 0u);
    o->zs_last_use.assign(o->slots, 0ll);
  }
  *done_out = o->zs_done;
  *prog_out = o->zs_prog;
  *prog_mirror_dev_out = o->zs_prog_hd;
  *prog_mirror_host_out = o->zs_prog_h;
  return MOBILE_OK;
}

// Stream memory operations come from the driver API; they are resolved at run
// time so libmobile.so does not link libcuda (it must import on GPU-less hosts).
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamValueFn driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (StreamValueFn)fn;
}
static StreamValueFn stream_wait_value() {
  static StreamValueFn f = driver_fn("cuStreamWaitValue32");
  return f;
}
static StreamValueFn stream_write_value() {
  static StreamValueFn f = driver_fn("cuStreamWriteValue32");
  return f;
}

static int zs_issue_copy(mobile_offload* o, int layer, int expert, int slot) {
  CUstream cs = (CUstream)o->copy;
  const long long need = o->zs_last_use[slot];
  if (!stream_wait_value() || !stream_write_value()) {
    mobile::set_error("offload: cuStreamWaitValue32 / cuStreamWriteValue32 unavailable");
    return MOBILE_ERR_UNSUPPORTED;
  }
  if (need > 0) {  // the slot's previous occupant must have been consumed
    if (stream_wait_value()(cs, (CUdeviceptr)o->zs_prog, (cuuint32_t)need, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
      mobile::set_error("offload: cuStreamWaitValue32 failed");
      return MOBILE_ERR_CUDA;
    }
  }
  const char* src = o->host + (long long)layer * o->layer_stride + (long long)expert * o->expert_stride;
  char* dst = o->pool + (long long)slot * o->expert_bytes;
  OFF_CUDA(cudaMemcpyAsync(dst, src, (size_t)o->expert_bytes, cudaMemcpyHostToDevice, o->copy), "expert H2D");
  const unsigned t = ++o->zs_ticket[slot];
  if (stream_write_value()(cs, (CUdeviceptr)(o->zs_done + slot), (cuuint32_t)t, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS) {
    mobile::set_error("offload: cuStreamWriteValue32 failed");
    return MOBILE_ERR_CUDA;
  }
  o->slot_layer[slot] = layer;
  o->slot_expert[slot] = expert;
  o->bytes += o->expert_bytes;
  o->transfers++;
  return MOBILE_OK;
}

// Required experts of `layer` (engine.py:137-145): request + pin; misses are
// issued; out2[2i] = slot, out2[2i+1] = ticket to wait for.  `now_prog` is the
// progress value the kernel has certainly reached (deadlock retry: the host
// waits for the kernel / copies through wait_fn).
int mobile_offload_zs_require(mobile_offload* o, int layer, const int* experts, int n, int* out2, int* issued_out,
                              int (*wait_fn)(void*), void* wait_ctx) {
  int fresh = 0;
  for (int i = 0; i < n; ++i) {
    const int e = experts[i];
    int status = 0, slot = -1;
    double ready = 0;
    int st = mobile_cache_request(o->cache, layer, e, o->clock, 0, nullptr, kInf, &status, &ready, &slot);
    if (st == MOBILE_ERR_DEADLOCK && wait_fn) {  // the simulator's stall: drain, settle, retry once
      if (int rc = wait_fn(wait_ctx)) return rc;
      OFF_CUDA(cudaStreamSynchronize(o->copy), "deadlock stall (copy)");
      settle_all(o);
      st = mobile_cache_request(o->cache, layer, e, o->clock, 0, nullptr, kInf, &status, &ready, &slot);
    }
    if (st != MOBILE_OK) return st;
    if (status == MOBILE_STATUS_ISSUED) {
      if (int r = zs_issue_copy(o, layer, e, slot)) return r;
      ++fresh;
    }
    mobile_cache_pin(o->cache, layer, e);
    if (ready == kInf) o->awaited.emplace_back(layer, e);
    out2[2 * i] = slot;
    out2[2 * i + 1] = (int)o->zs_ticket[slot];
  }
  if (issued_out) *issued_out = fresh;
  return MOBILE_OK;
}

long long* mobile_offload_zs_base(mobile_offload* o) { return &o->zs_base; }

int mobile_offload_zs_prefetch(mobile_offload* o, int layer, int expert, int* status_out) {
  int status = 0, slot = -1;
  double ready = 0;
  int st = mobile_cache_request(o->cache, layer, expert, o->clock, 1, nullptr, kInf, &status, &ready, &slot);
  if (st != MOBILE_OK) return st;
  if (status == MOBILE_STATUS_ISSUED)
    if (int r = zs_issue_copy(o, layer, expert, slot)) return r;
  if (status_out) *status_out = status;
  return MOBILE_OK;
}

// Unpin (engine.py:152-153); the slots stay busy until the kernel's progress
// counter reaches `release_prog` (it has consumed this layer).
int mobile_offload_zs_release(mobile_offload* o, int layer, const int* experts, int n, long long release_prog) {
  for (int i = 0; i < n; ++i) {
    int slot = -1;
    if (mobile_cache_lookup(o->cache, layer, experts[i], nullptr, &slot) == MOBILE_OK)
      o->zs_last_use[slot] = release_prog;
    mobile_cache_unpin(o->cache, layer, experts[i]);
  }
  return MOBILE_OK;
}

int mobile_offload_counters(const mobile_offload* o, long long* out2) {
  out2[0] = o->bytes;
  out2[1] = o->transfers;
  return MOBILE_OK;
}

}  // extern "C"
