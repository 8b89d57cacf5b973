// Pointer cache object shared by the C ABI (cm_registry_*) and the
// communicator's per-call send/recv classification.
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "cm.h"

namespace cm {

struct Registry {
  struct Live {
    int64_t size;
    int kind;
  };
  struct Range {
    int64_t size;
    int kind;
  };
  // what a cache entry records about an address (real backend: one
  // cuPointerGetAttributes call; sim backend: the kind only)
  struct Info {
    int kind = CM_KIND_HOST;
    int device = -1;
    uint64_t start = 0;       // allocation range holding the address
    int64_t size = 0;
    uint64_t buffer_id = 0;   // unique per allocation, never reused
  };

  int policy = CM_NO_CACHE;
  int64_t delay_ns = 1000;
  bool simulated = true;
  std::mutex mu;
  cm_registry_stats_t st{0, 0, 0, 0};
  int64_t query_ns = 0;

  // ground truth: allocations made through alloc() (and sim registrations)
  std::map<uint64_t, Live> live;
  // real backend: externally allocated, registered memory
  std::map<uint64_t, Live> external;
  // simulated caches are exact-address (registry.py:68); real intercept cache
  // is a range map; real lazy cache is exact-address like the reference
  std::unordered_map<uint64_t, Info> cache;
  std::map<uint64_t, Range> ranges;
  std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> freed;
  uint64_t next_address = 0x1000;                            // registry.py:20

  ~Registry();
  int alloc(int kind, int64_t size, uint64_t* out);
  int free_(uint64_t addr);
  int register_range(uint64_t addr, int64_t size, int kind);
  int unregister_range(uint64_t addr);
  int classify(uint64_t addr, int* kind, Info* info = nullptr);
  int ground_truth(uint64_t addr, int* kind);
  std::string stats_json();

 private:
  int driver_query_real(uint64_t addr, Info* info, bool count);
  int driver_query_sim(uint64_t addr, int* kind);
  int insert_range(uint64_t addr, int64_t size, int kind);
  const Range* find_range(uint64_t addr) const;
};

}  // namespace cm
