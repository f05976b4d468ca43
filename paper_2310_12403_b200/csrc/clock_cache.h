// Set-associative CLOCK feature cache (clock_cache.cu): the fast production
// cache mode; DeviceLru (cache.h) is the batch-exact LRU used for parity.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace cb {

struct ClockView {
  uint32_t* tags;     // [n_sets * ways] key or 0xffffffff
  uint8_t* ref;       // [n_sets * ways] CLOCK reference bits
  uint32_t* pinned;   // [n_sets * ways] batch epoch of the last hit / claim
  uint32_t* hand;     // [n_sets] CLOCK hands
  unsigned char* rows;  // [n_sets * ways * row_bytes]
  uint32_t n_sets, ways;
};

class ClockCache {
 public:
  ClockCache(int device, uint64_t capacity, uint32_t ways, uint64_t row_bytes);
  ~ClockCache();
  ClockCache(const ClockCache&) = delete;
  ClockCache& operator=(const ClockCache&) = delete;
  // rows of d_ids[0 .. min(*d_count, cap)) (distinct keys; d_count nullptr:
  // cap ids) into d_out requester-aligned: hits from the cache, misses from
  // table + row_map[v] * row_bytes (row_map nullptr: v); misses are inserted.
  void gather(const void* table, const uint32_t* row_map, const uint32_t* d_ids,
              const unsigned long long* d_count, uint64_t cap, void* d_out, cudaStream_t st);
  // per-batch scratch for up to cap ids, allocated now (before a capture)
  void reserve(uint64_t cap);
  // running totals (synchronises st)
  void counters(cudaStream_t st, uint64_t* hits, uint64_t* inserted);
  uint64_t capacity() const { return static_cast<uint64_t>(view_.n_sets) * view_.ways; }
  uint64_t row_bytes() const { return row_bytes_; }
  int device() const { return device_; }

 private:
  int device_;
  uint64_t row_bytes_;
  ClockView view_{};
  unsigned long long* ctr_ = nullptr;  // [0] hits, [1] inserted
  int32_t* slot_ = nullptr;
  uint64_t slot_cap_ = 0;
  uint32_t epoch_ = 0;
};

}  // namespace cb
