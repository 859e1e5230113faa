// Expert cache core: the semantics of moesim.memory.HbmCache (memory.py:65-181)
// in C++, plus physical slot assignment for the device runtime.
//
// LRU order is a std::list (front = least recent) indexed by a hash map.  A
// resident entry is "settled" when ready <= now and "in flight" otherwise;
// pinned or in-flight entries are never victims.  Victim choice, deferral and
// deadlock follow memory.py:117-162 exactly; a fresh entry takes the slot the
// victim released (or the lowest never-used slot), so slot assignment is a
// deterministic function of the request sequence.
#include <cmath>
#include <cstdio>
#include <list>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/mobile.h"

namespace mobile {
void set_error(const char* fmt, ...);
}

struct CacheEntry {
  long long key;
  int layer, expert;
  double ready;
  int slot;
};

struct mobile_cache {
  int slots;
  std::list<CacheEntry> lru;
  std::unordered_map<long long, std::list<CacheEntry>::iterator> index;
  std::unordered_set<long long> pins;
  std::vector<int> free_slots;  // stack; top = lowest unused slot
  long long hits = 0, coalesced = 0, issued = 0, evictions = 0, deferrals = 0;
};

static inline long long cache_key(int layer, int expert) {
  return ((long long)layer << 32) | (unsigned int)expert;
}

static bool evict_one(mobile_cache* c, double now) {  // memory.py:150-157
  for (auto it = c->lru.begin(); it != c->lru.end(); ++it) {
    if (c->pins.count(it->key) || it->ready > now) continue;
    c->free_slots.push_back(it->slot);
    c->index.erase(it->key);
    c->lru.erase(it);
    c->evictions++;
    return true;
  }
  return false;
}

extern "C" {

mobile_cache* mobile_cache_create(int slots) {
  if (slots < 1) {
    mobile::set_error("cache needs at least 1 expert slot, got %d", slots);
    return nullptr;
  }
  auto* c = new mobile_cache();
  c->slots = slots;
  c->free_slots.reserve(slots);
  for (int s = slots - 1; s >= 0; --s) c->free_slots.push_back(s);
  return c;
}

void mobile_cache_destroy(mobile_cache* c) { delete c; }

int mobile_cache_request(mobile_cache* c, int layer, int expert, double now, int speculative,
                         mobile_channel* channel, double ready_if_issued, int* status_out,
                         double* ready_out, int* slot_out) {
  const long long k = cache_key(layer, expert);
  auto f = c->index.find(k);
  if (f != c->index.end()) {  // memory.py:129-135
    c->lru.splice(c->lru.end(), c->lru, f->second);  // move to MRU
    const CacheEntry& e = *f->second;
    if (ready_out) *ready_out = e.ready;
    if (slot_out) *slot_out = e.slot;
    if (e.ready <= now) {
      c->hits++;
      if (status_out) *status_out = MOBILE_STATUS_HIT;
    } else {
      c->coalesced++;
      if (status_out) *status_out = MOBILE_STATUS_IN_FLIGHT;
    }
    return MOBILE_OK;
  }
  if ((int)c->lru.size() >= c->slots && !evict_one(c, now)) {  // memory.py:136-144
    if (speculative) {
      c->deferrals++;
      return MOBILE_ERR_DEFERRED;
    }
    mobile::set_error("no evictable slot for L%dE%d: all %d slots are pinned or in flight at t=%.6f",
                      layer, expert, c->slots, now);
    return MOBILE_ERR_DEADLOCK;
  }
  double ready = ready_if_issued;
  if (channel) {  // memory.py:38-43
    const double start = now > channel->busy_until ? now : channel->busy_until;
    channel->busy_until = start + channel->t_xfer;
    channel->transfers_issued++;
    ready = channel->busy_until;
  }
  const int slot = c->free_slots.back();
  c->free_slots.pop_back();
  c->lru.push_back(CacheEntry{k, layer, expert, ready, slot});
  c->index[k] = std::prev(c->lru.end());
  c->issued++;
  if (status_out) *status_out = MOBILE_STATUS_ISSUED;
  if (ready_out) *ready_out = ready;
  if (slot_out) *slot_out = slot;
  return MOBILE_OK;
}

int mobile_cache_pin(mobile_cache* c, int layer, int expert) {
  c->pins.insert(cache_key(layer, expert));
  return MOBILE_OK;
}

int mobile_cache_unpin(mobile_cache* c, int layer, int expert) {
  c->pins.erase(cache_key(layer, expert));
  return MOBILE_OK;
}

int mobile_cache_token_end(mobile_cache* c) {
  c->pins.clear();
  return MOBILE_OK;
}

int mobile_cache_evict_lru(mobile_cache* c, int n, double now, int* victims_out, int* n_out) {
  // memory.py:159-181: all-or-nothing
  std::vector<std::list<CacheEntry>::iterator> victims;
  for (auto it = c->lru.begin(); it != c->lru.end() && (int)victims.size() < n; ++it) {
    if (c->pins.count(it->key) || it->ready > now) continue;
    victims.push_back(it);
  }
  if ((int)victims.size() < n) {
    mobile::set_error("asked to evict %d experts but only %d are unpinned", n, (int)victims.size());
    if (n_out) *n_out = (int)victims.size();
    return MOBILE_ERR_INVALID;
  }
  int i = 0;
  for (auto it : victims) {
    if (victims_out) {
      victims_out[2 * i] = it->layer;
      victims_out[2 * i + 1] = it->expert;
    }
    ++i;
    c->free_slots.push_back(it->slot);
    c->index.erase(it->key);
    c->lru.erase(it);
    c->evictions++;
  }
  if (n_out) *n_out = i;
  return MOBILE_OK;
}

int mobile_cache_size(const mobile_cache* c) { return (int)c->lru.size(); }

int mobile_cache_contains(const mobile_cache* c, int layer, int expert) {
  return c->index.count(cache_key(layer, expert)) ? 1 : 0;
}

int mobile_cache_lookup(const mobile_cache* c, int layer, int expert, double* ready_out, int* slot_out) {
  auto f = c->index.find(cache_key(layer, expert));
  if (f == c->index.end()) return MOBILE_ERR_NOT_FOUND;
  if (ready_out) *ready_out = f->second->ready;
  if (slot_out) *slot_out = f->second->slot;
  return MOBILE_OK;
}

int mobile_cache_set_ready(mobile_cache* c, int layer, int expert, double ready) {
  auto f = c->index.find(cache_key(layer, expert));
  if (f == c->index.end()) return MOBILE_ERR_NOT_FOUND;
  f->second->ready = ready;
  return MOBILE_OK;
}

int mobile_cache_entries(const mobile_cache* c, int* out, int cap) {
  int i = 0;
  for (const auto& e : c->lru) {
    if (i >= cap) break;
    out[2 * i] = e.layer;
    out[2 * i + 1] = e.expert;
    ++i;
  }
  return i;
}

int mobile_cache_stats(const mobile_cache* c, long long* out5) {
  out5[0] = c->hits;
  out5[1] = c->coalesced;
  out5[2] = c->issued;
  out5[3] = c->evictions;
  out5[4] = c->deferrals;
  return MOBILE_OK;
}

}  // extern "C"
