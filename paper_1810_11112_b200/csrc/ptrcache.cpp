// Pointer cache (PAPER §V-B; reference registry.py:52-151).
//
// Two backends behind one object:
//  * simulated: the reference's model verbatim — fake addresses from 0x1000,
//    lowest freed address reused first (registry.py:75-79), the "driver query"
//    is a ground-truth lookup that bumps a counter.
//  * real: allocations are real (cudaMalloc / cudaHostAlloc — the intercepted
//    allocation API), the driver query is cudaPointerGetAttributes and its wall
//    time is accumulated, and the intercept cache answers interior pointers of
//    registered allocations through an ordered range map (torch hands out
//    sub-allocations, so exact-address lookups are not enough on a GPU).
// Every operation takes the registry mutex (registry.py:52-56 serialises).
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "ptrcache.hpp"

using namespace cm;

namespace cm {

static const char* policy_name(int p) {
  switch (p) {
    case CM_NO_CACHE: return "no_cache";
    case CM_LAZY_CACHE: return "lazy_cache";
    case CM_INTERCEPT_CACHE: return "intercept_cache";
    default: return "?";
  }
}

static char hexbuf_[32];
static std::string hexaddr(uint64_t a) {
  char b[32];
  snprintf(b, sizeof b, "%#llx", (unsigned long long)a);
  (void)hexbuf_;
  return b;
}

// Real driver query: ONE cuPointerGetAttributes call for memory type, device
// ordinal, allocation range and buffer id (unregistered host memory is HOST).
typedef CUresult (*PtrAttrsFn)(unsigned, CUpointer_attribute*, void**, CUdeviceptr);

static PtrAttrsFn ptr_attrs_fn() {
  static PtrAttrsFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttributes", &f, cudaEnableDefault, &q) != cudaSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<PtrAttrsFn>(f);
  }();
  return fn;
}

int Registry::driver_query_real(uint64_t addr, Info* info, bool count) {
  PtrAttrsFn fn = ptr_attrs_fn();
  if (!fn) return fail(CM_ERR_UNSUPPORTED, "cuPointerGetAttributes unavailable");
  unsigned mtype = 0;
  int dev = -1;
  CUdeviceptr start = 0;
  size_t size = 0;
  unsigned long long bid = 0;
  unsigned managed = 0;
  CUpointer_attribute at[6] = {CU_POINTER_ATTRIBUTE_MEMORY_TYPE, CU_POINTER_ATTRIBUTE_DEVICE_ORDINAL,
                               CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, CU_POINTER_ATTRIBUTE_RANGE_SIZE,
                               CU_POINTER_ATTRIBUTE_BUFFER_ID, CU_POINTER_ATTRIBUTE_IS_MANAGED};
  void* val[6] = {&mtype, &dev, &start, &size, &bid, &managed};
  const auto t0 = std::chrono::steady_clock::now();
  CUresult r = fn(6, at, val, (CUdeviceptr)addr);
  const auto t1 = std::chrono::steady_clock::now();
  if (count) {
    st.driver_queries += 1;
    query_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  }
  if (r != CUDA_SUCCESS)
    return fail(CM_ERR_UNKNOWN_BUFFER, "driver query failed for " + hexaddr(addr) + " (CUresult " +
                                           std::to_string((int)r) + ")");
  info->kind = (mtype == CU_MEMORYTYPE_DEVICE || managed) ? CM_KIND_DEVICE : CM_KIND_HOST;
  info->device = mtype ? dev : -1;
  info->start = (uint64_t)start;
  info->size = (int64_t)size;
  info->buffer_id = bid;
  return CM_OK;
}

int Registry::driver_query_sim(uint64_t addr, int* kind) {
  st.driver_queries += 1;                                   // registry.py:125-131
  auto it = live.find(addr);
  if (it == live.end())
    return fail(CM_ERR_UNKNOWN_BUFFER, "classify of never-allocated address " + hexaddr(addr));
  *kind = it->second.kind;
  return CM_OK;
}

const Registry::Range* Registry::find_range(uint64_t addr) const {
  auto it = ranges.upper_bound(addr);
  if (it == ranges.begin()) return nullptr;
  --it;
  if (addr < it->first + (uint64_t)it->second.size) return &it->second;
  return nullptr;
}

int Registry::classify(uint64_t addr, int* kind, Info* info) {
  std::lock_guard<std::mutex> g(mu);
  Info tmp;
  Info* out = info ? info : &tmp;
  if (policy == CM_NO_CACHE) {
    int s;
    if (simulated) {
      s = driver_query_sim(addr, &out->kind);
    } else {
      s = driver_query_real(addr, out, true);
    }
    if (!s) *kind = out->kind;
    return s;
  }
  if (policy == CM_LAZY_CACHE) {                             // registry.py:110-117
    auto it = cache.find(addr);
    if (it != cache.end()) {
      st.cache_hits += 1;
      *out = it->second;
      *kind = it->second.kind;
      return CM_OK;
    }
    Info in;
    int s = simulated ? driver_query_sim(addr, &in.kind) : driver_query_real(addr, &in, true);
    if (s) return s;
    cache[addr] = in;
    st.inserts += 1;
    *out = in;
    *kind = in.kind;
    return CM_OK;
  }
  // intercept: the cache is authoritative, zero driver traffic (registry.py:118-123)
  if (simulated) {
    auto it = cache.find(addr);
    if (it == cache.end())
      return fail(CM_ERR_UNKNOWN_BUFFER, "classify of never-allocated address " + hexaddr(addr));
    st.cache_hits += 1;
    *out = it->second;
    *kind = it->second.kind;
    return CM_OK;
  }
  auto it = ranges.upper_bound(addr);
  if (it == ranges.begin())
    return fail(CM_ERR_UNKNOWN_BUFFER, "classify of never-registered address " + hexaddr(addr));
  --it;
  if (addr >= it->first + (uint64_t)it->second.size)
    return fail(CM_ERR_UNKNOWN_BUFFER, "classify of never-registered address " + hexaddr(addr));
  st.cache_hits += 1;
  out->kind = it->second.kind;
  out->start = it->first;
  out->size = it->second.size;
  *kind = it->second.kind;
  return CM_OK;
}

int Registry::insert_range(uint64_t addr, int64_t size, int kind) {
  ranges[addr] = Range{size, kind};
  st.inserts += 1;
  return CM_OK;
}

int Registry::alloc(int kind, int64_t size, uint64_t* out) {
  if (size <= 0) return fail(CM_ERR_VALUE, "allocation size must be positive, got " + std::to_string(size));
  if (kind != CM_KIND_HOST && kind != CM_KIND_DEVICE) return fail(CM_ERR_VALUE, "bad buffer kind");
  std::lock_guard<std::mutex> g(mu);
  uint64_t a;
  if (simulated) {                                          // registry.py:71-86
    if (!freed.empty()) { a = freed.top(); freed.pop(); }
    else a = next_address++;
  } else {
    void* p = nullptr;
    cudaError_t e = kind == CM_KIND_DEVICE ? cudaMalloc(&p, (size_t)size)
                                           : cudaHostAlloc(&p, (size_t)size, cudaHostAllocMapped);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(CM_ERR_CUDA, std::string("allocation failed: ") + cudaGetErrorString(e));
    }
    a = reinterpret_cast<uint64_t>(p);
  }
  live[a] = Live{size, kind};
  if (policy == CM_INTERCEPT_CACHE) {
    if (simulated) { Info in; in.kind = kind; cache[a] = in; st.inserts += 1; }
    else insert_range(a, size, kind);
  }
  *out = a;
  return CM_OK;
}

int Registry::free_(uint64_t addr) {
  std::lock_guard<std::mutex> g(mu);
  auto it = live.find(addr);
  if (it == live.end())
    return fail(CM_ERR_INVALID_HANDLE, "free of dead or unknown handle at address " + hexaddr(addr));
  const int kind = it->second.kind;
  live.erase(it);
  if (simulated) {
    freed.push(addr);
  } else {
    cudaError_t e = kind == CM_KIND_DEVICE ? cudaFree(reinterpret_cast<void*>(addr))
                                           : cudaFreeHost(reinterpret_cast<void*>(addr));
    if (e != cudaSuccess) cudaGetLastError();
  }
  if (policy == CM_INTERCEPT_CACHE) {                       // registry.py:97-99
    if (simulated) cache.erase(addr);
    else ranges.erase(addr);
    st.invalidations += 1;
  }
  // lazy_cache deliberately keeps its entry (the §V-B staleness flaw)
  return CM_OK;
}

int Registry::register_range(uint64_t addr, int64_t size, int kind) {
  if (size <= 0) return fail(CM_ERR_VALUE, "registered size must be positive");
  std::lock_guard<std::mutex> g(mu);
  if (simulated) {
    live[addr] = Live{size, kind};
    if (policy == CM_INTERCEPT_CACHE) { Info in; in.kind = kind; cache[addr] = in; st.inserts += 1; }
    return CM_OK;
  }
  if (policy == CM_INTERCEPT_CACHE) insert_range(addr, size, kind);
  external[addr] = Live{size, kind};
  return CM_OK;
}

int Registry::unregister_range(uint64_t addr) {
  std::lock_guard<std::mutex> g(mu);
  if (simulated) {
    if (!live.erase(addr)) return fail(CM_ERR_INVALID_HANDLE, "unregister of unknown address " + hexaddr(addr));
    if (policy == CM_INTERCEPT_CACHE) { cache.erase(addr); st.invalidations += 1; }
    return CM_OK;
  }
  if (!external.erase(addr)) return fail(CM_ERR_INVALID_HANDLE, "unregister of unknown address " + hexaddr(addr));
  if (policy == CM_INTERCEPT_CACHE) { ranges.erase(addr); st.invalidations += 1; }
  return CM_OK;
}

int Registry::ground_truth(uint64_t addr, int* kind) {
  std::lock_guard<std::mutex> g(mu);
  if (simulated) {
    auto it = live.find(addr);
    if (it == live.end()) return fail(CM_ERR_UNKNOWN_BUFFER, "no live allocation at address " + hexaddr(addr));
    *kind = it->second.kind;
    return CM_OK;
  }
  Info in;
  int s = driver_query_real(addr, &in, false);
  if (!s) *kind = in.kind;
  return s;
}

std::string Registry::stats_json() {
  std::lock_guard<std::mutex> g(mu);
  char b[256];
  snprintf(b, sizeof b,
           "{\"policy\": \"%s\", \"driver_queries\": %lld, \"cache_hits\": %lld, \"inserts\": %lld, "
           "\"invalidations\": %lld}",
           policy_name(policy), (long long)st.driver_queries, (long long)st.cache_hits,
           (long long)st.inserts, (long long)st.invalidations);
  return b;
}

Registry::~Registry() {
  if (simulated) return;
  for (auto& kv : live) {
    if (kv.second.kind == CM_KIND_DEVICE) cudaFree(reinterpret_cast<void*>(kv.first));
    else cudaFreeHost(reinterpret_cast<void*>(kv.first));
  }
  cudaGetLastError();
}

}  // namespace cm

extern "C" {

int cm_registry_create(int policy, int64_t query_delay_ns, int simulated, cm_registry_t** out) {
  if (policy < CM_NO_CACHE || policy > CM_INTERCEPT_CACHE) return fail(CM_ERR_VALUE, "unknown policy");
  auto* r = new Registry();
  r->policy = policy;
  r->delay_ns = query_delay_ns;
  r->simulated = simulated != 0;
  *out = reinterpret_cast<cm_registry_t*>(r);
  return CM_OK;
}

int cm_registry_destroy(cm_registry_t* reg) {
  delete reinterpret_cast<Registry*>(reg);
  return CM_OK;
}

#define REG(x) reinterpret_cast<Registry*>(x)

int cm_registry_alloc(cm_registry_t* reg, int kind, int64_t size, uint64_t* address) {
  return REG(reg)->alloc(kind, size, address);
}
int cm_registry_free(cm_registry_t* reg, uint64_t address) { return REG(reg)->free_(address); }
int cm_registry_register(cm_registry_t* reg, uint64_t address, int64_t size, int kind) {
  return REG(reg)->register_range(address, size, kind);
}
int cm_registry_unregister(cm_registry_t* reg, uint64_t address) {
  return REG(reg)->unregister_range(address);
}
int cm_registry_classify(cm_registry_t* reg, uint64_t address, int* kind) {
  return REG(reg)->classify(address, kind);
}
int cm_registry_info(cm_registry_t* reg, uint64_t address, cm_buffer_info_t* out) {
  Registry::Info in;
  int kind = 0;
  int s = REG(reg)->classify(address, &kind, &in);
  if (s) return s;
  out->kind = in.kind;
  out->device = in.device;
  out->range_start = in.start;
  out->range_size = in.size;
  out->buffer_id = in.buffer_id;
  return CM_OK;
}
int cm_registry_ground_truth(cm_registry_t* reg, uint64_t address, int* kind) {
  return REG(reg)->ground_truth(address, kind);
}
int cm_registry_stats(cm_registry_t* reg, cm_registry_stats_t* out) {
  std::lock_guard<std::mutex> g(REG(reg)->mu);
  *out = REG(reg)->st;
  return CM_OK;
}
int cm_registry_policy(cm_registry_t* reg, int* policy) {
  *policy = REG(reg)->policy;
  return CM_OK;
}
int cm_registry_query_time_ns(cm_registry_t* reg, int64_t* ns) {
  Registry* r = REG(reg);
  std::lock_guard<std::mutex> g(r->mu);
  *ns = r->simulated ? r->st.driver_queries * r->delay_ns : r->query_ns;   // registry.py:143-145
  return CM_OK;
}
int cm_registry_stats_json(cm_registry_t* reg, char* buf, size_t len) {
  std::string s = REG(reg)->stats_json();
  if (s.size() + 1 > len) return fail(CM_ERR_VALUE, "buffer too small");
  memcpy(buf, s.c_str(), s.size() + 1);
  return CM_OK;
}

}  // extern "C"
