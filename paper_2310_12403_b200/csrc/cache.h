// Per-GPU feature-row cache with exact LRU semantics (LruCache, cache.hpp:17-42,
// cache.cpp:8-32), evaluated a whole minibatch at a time on the device.
//
// A batch is a list of DISTINCT keys accessed in a given order (the
// reference's feature traces are id sets: input_vertices(), cache.cpp:105 /
// 193). Key v at batch position i hits iff it was accessed before and fewer
// than C distinct other keys were accessed since:
//     rho(v) + i - X_i < C,
//   rho(v) = #keys whose last access is newer than v's (batch start),
//   X_i    = #{j < i : rho(a_j) < rho(v)}  (keys counted twice otherwise).
// rho comes from a bitmap over access times (bit t set iff access t is the
// latest of its key) and a popcount prefix; X_i by a bottom-up merge count
// (shared-memory levels, then global levels). Residency after the batch is
// the C most recent keys, which drives slot reuse of the row storage.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace cb {

struct CacheGatherSrc {
  const void* table = nullptr;      // backing rows (device or mapped host memory)
  const uint32_t* row_map = nullptr;  // row of v in table (nullptr = v)
  void* rows_out = nullptr;         // [kept] rows in kept-id order
  // instead of table/row_map: the address of each kept key's row on a miss
  // (device array by kept position; e.g. rows in peers' staging buffers)
  const void* const* miss_ptr = nullptr;
};

class DeviceLru {
 public:
  DeviceLru(int device, uint64_t n_keys, uint64_t capacity, uint64_t row_bytes);
  ~DeviceLru();
  DeviceLru(const DeviceLru&) = delete;
  DeviceLru& operator=(const DeviceLru&) = delete;

  // feature_load_sim / run_dependent_experiment step: the sorted unique ids
  // (device), optionally only those with owner[v] == part, accessed in
  // access_order(ids, order_key) (cache.cpp:74-84). With storage (row_bytes >
  // 0) and src.table, rows of the kept ids are produced in kept order: hits
  // from the cache, misses from the backing table. Returns the kept count;
  // hit / miss totals accumulate.
  uint64_t access_ids(const uint32_t* d_ids, uint64_t n, uint64_t order_key,
                      const uint32_t* d_owner, uint32_t part, const CacheGatherSrc& src,
                      cudaStream_t st);
  // Distinct keys (device) in access order; d_miss (optional) gets 1 per miss.
  void access_ordered(const uint32_t* d_keys, uint64_t B, uint8_t* d_miss, cudaStream_t st);
  // Arbitrary host trace (split into runs of distinct keys); miss[i] = 1/0.
  void access_trace(const uint32_t* keys, uint64_t n, uint8_t* miss, cudaStream_t st);

  void resident(std::vector<uint32_t>& out);  // most recent first
  uint64_t hits() const { return hits_; }
  uint64_t misses() const { return misses_; }
  uint64_t size() const;
  void reset_counters() { hits_ = misses_ = 0; }
  uint64_t capacity() const { return cap_; }
  uint64_t n_keys() const { return n_; }
  uint64_t row_bytes() const { return row_bytes_; }
  const void* storage() const { return rows_; }
  int device() const { return device_; }

 private:
  void ensure_batch(uint64_t B);
  void compact_time(cudaStream_t st);
  void prefix_time(cudaStream_t st);
  void run_batch(const uint32_t* keys_or_kept, const uint32_t* order, uint64_t B,
                 uint8_t* d_miss, const CacheGatherSrc* src, cudaStream_t st);

  int device_;
  uint64_t n_, cap_, row_bytes_;
  uint64_t T_ = 0;          // accesses so far (time of the newest access)
  uint64_t tbits_ = 0;      // time bitmap capacity (bits)
  uint64_t distinct_ = 0;   // keys ever seen
  uint64_t hits_ = 0, misses_ = 0;
  uint32_t* last_ = nullptr;    // [n] latest access time (0 = never)
  uint32_t* tmark_ = nullptr;   // [tbits/32]
  uint32_t* tpre_ = nullptr;    // [tbits/32 + 1] exclusive popcount prefix
  int32_t* slot_of_ = nullptr;  // [n] storage slot or -1
  uint32_t* slot_key_ = nullptr;  // [cap]
  unsigned char* rows_ = nullptr;  // [cap * row_bytes]
  unsigned long long* ctr_ = nullptr;  // [8] device counters
  // per-batch scratch
  uint64_t bcap_ = 0;
  uint32_t *kept_ = nullptr, *ord_ = nullptr, *ord2_ = nullptr, *rho_ = nullptr,
           *xcnt_ = nullptr, *mk_[2] = {nullptr, nullptr}, *mi_[2] = {nullptr, nullptr},
           *free_ = nullptr, *fill_slot_ = nullptr, *fill_row_ = nullptr;
  unsigned long long *hkey_ = nullptr, *hkey2_ = nullptr;
  const void** src_ptr_ = nullptr;
  void* cub_tmp_ = nullptr;
  size_t cub_bytes_ = 0;
};

}  // namespace cb
