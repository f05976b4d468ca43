// Fast per-GPU feature cache: set-associative with CLOCK (second chance)
// replacement -- the production mode next to DeviceLru's batch-exact LRU
// (cache.cu), which reproduces the reference's LruCache decisions
// (cache.cpp:8-32) for parity but needs sorts and merge passes per batch.
// "a fast set-associative/CLOCK mode that reports its own
// hit rate". Keys are vertex ids; a batch's ids are distinct (input vertices).
//
// One batch = three kernels, no sort and no host round trip:
//   lookup : key v -> set hash(v) % n_sets, compare its W tags; a hit marks
//            the way referenced and pinned for this batch
//   serve  : every row to the requester-aligned output: hits from the cache
//            rows, misses from the backing table (HBM or pinned host tier)
//   insert : each miss claims a way of its set (CLOCK hand, skipping ways
//            pinned this batch or already claimed, clearing reference bits)
//            and copies its row in from the output
// Rows read in serve are never written in the same batch (insert skips pinned
// ways), so a hit always reads a whole row.
#include <cuda_runtime.h>

#include <algorithm>

#include "cb_device.cuh"
#include "cb_internal.h"
#include "clock_cache.h"

namespace cb {
namespace {

using cbdev::lane_id;
constexpr uint32_t kEmpty = 0xffffffffu;

__device__ __forceinline__ uint32_t set_of(uint32_t v, uint32_t n_sets) {
  return static_cast<uint32_t>(cbdev::mix64(v ^ 0x636c6f636bULL) % n_sets);
}

__global__ void clock_lookup_kernel(ClockView c, const uint32_t* __restrict__ ids,
                                    const unsigned long long* __restrict__ count, uint64_t cap,
                                    int32_t* slot, uint32_t epoch,
                                    unsigned long long* hits) {
  cbdev::pdl_begin();
  const uint64_t n = count ? min(static_cast<uint64_t>(*count), cap) : cap;
  unsigned long long h = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = ids[i];
    const uint32_t s = set_of(v, c.n_sets);
    int32_t hit = -1;
    for (uint32_t w = 0; w < c.ways; ++w)
      if (c.tags[s * c.ways + w] == v) hit = static_cast<int32_t>(s * c.ways + w);
    if (hit >= 0) {
      c.ref[hit] = 1;
      c.pinned[hit] = epoch;
      ++h;
    }
    slot[i] = hit;
  }
  h = cbdev::warp_sum(h);
  if (lane_id() == 0 && h) atomicAdd(hits, h);
}

template <typename V>
__global__ void clock_serve_kernel(ClockView c, const V* __restrict__ table,
                                   const uint32_t* __restrict__ row_map,
                                   const uint32_t* __restrict__ ids,
                                   const unsigned long long* __restrict__ count, uint64_t cap,
                                   const int32_t* __restrict__ slot, uint32_t vpr,
                                   V* __restrict__ out) {
  cbdev::pdl_begin();
  const uint64_t n = count ? min(static_cast<uint64_t>(*count), cap) : cap;
  const uint64_t total = n * vpr;
  const V* rows = reinterpret_cast<const V*>(c.rows);
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = x / vpr, k = x - r * vpr;
    const int32_t sl = slot[r];
    const uint32_t v = ids[r];
    const V* src = sl >= 0 ? rows + static_cast<uint64_t>(sl) * vpr
                           : table + static_cast<uint64_t>(row_map ? row_map[v] : v) * vpr;
    __stcs(out + x, src[k]);
  }
}

// one warp per miss: lane 0 claims a way, the warp copies the row in
template <typename V>
__global__ void clock_insert_kernel(ClockView c, const uint32_t* __restrict__ ids,
                                    const unsigned long long* __restrict__ count, uint64_t cap,
                                    const int32_t* __restrict__ slot, uint32_t epoch,
                                    uint32_t vpr, const V* __restrict__ out,
                                    unsigned long long* inserted) {
  cbdev::pdl_begin();
  const uint64_t n = count ? min(static_cast<uint64_t>(*count), cap) : cap;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  V* rows = reinterpret_cast<V*>(c.rows);
  for (uint64_t i = warp; i < n; i += nw) {
    if (slot[i] >= 0) continue;
    const uint32_t v = ids[i];
    const uint32_t s = set_of(v, c.n_sets);
    int32_t way = -1;
    if (lane_id() == 0) {
      // second chance over at most two sweeps of the set
      for (uint32_t t = 0; t < 2 * c.ways && way < 0; ++t) {
        const uint32_t w = atomicAdd(&c.hand[s], 1u) % c.ways;
        const uint32_t e = s * c.ways + w;
        const uint32_t old = c.pinned[e];
        if (old == epoch) continue;  // hit (read) or claimed this batch
        if (c.tags[e] != kEmpty && c.ref[e]) {  // second chance
          c.ref[e] = 0;
          continue;
        }
        if (atomicCAS(&c.pinned[e], old, epoch) == old) way = static_cast<int32_t>(e);
      }
      if (way >= 0) {
        c.tags[way] = v;
        c.ref[way] = 0;
        atomicAdd(inserted, 1ULL);
      }
    }
    way = __shfl_sync(0xffffffffu, way, 0);
    if (way < 0) continue;
    for (uint32_t k = lane_id(); k < vpr; k += 32)
      rows[static_cast<uint64_t>(way) * vpr + k] = out[i * vpr + k];
  }
}

template <typename F>
void dispatch(uint64_t row_bytes, F&& f) {
  if (row_bytes % 16 == 0) f(uint4{});
  else if (row_bytes % 8 == 0) f(uint2{});
  else if (row_bytes % 4 == 0) f(uint32_t{});
  else f(static_cast<unsigned short>(0));
}

}  // namespace

ClockCache::ClockCache(int device, uint64_t capacity, uint32_t ways, uint64_t row_bytes)
    : device_(device), row_bytes_(row_bytes) {
  require(ways >= 1 && ways <= 32, "ClockCache: 1..32 ways");
  require(row_bytes % 2 == 0, "ClockCache: row bytes must be even");
  view_.ways = ways;
  view_.n_sets = static_cast<uint32_t>(std::max<uint64_t>(1, capacity / ways));
  const uint64_t slots = static_cast<uint64_t>(view_.n_sets) * ways;
  cuda_check(cudaMalloc(&view_.tags, slots * 4), "cudaMalloc");
  cuda_check(cudaMemset(view_.tags, 0xff, slots * 4), "cudaMemset");
  cuda_check(cudaMalloc(&view_.ref, slots), "cudaMalloc");
  cuda_check(cudaMemset(view_.ref, 0, slots), "cudaMemset");
  cuda_check(cudaMalloc(&view_.pinned, slots * 4), "cudaMalloc");
  cuda_check(cudaMemset(view_.pinned, 0, slots * 4), "cudaMemset");
  cuda_check(cudaMalloc(&view_.hand, view_.n_sets * 4ULL), "cudaMalloc");
  cuda_check(cudaMemset(view_.hand, 0, view_.n_sets * 4ULL), "cudaMemset");
  cuda_check(cudaMalloc(&view_.rows, slots * row_bytes), "cudaMalloc");
  cuda_check(cudaMalloc(&ctr_, 16), "cudaMalloc");
  cuda_check(cudaMemset(ctr_, 0, 16), "cudaMemset");
}

ClockCache::~ClockCache() {
  for (void* p : {static_cast<void*>(view_.tags), static_cast<void*>(view_.ref),
                  static_cast<void*>(view_.pinned), static_cast<void*>(view_.hand),
                  static_cast<void*>(view_.rows), static_cast<void*>(ctr_),
                  static_cast<void*>(slot_)})
    if (p) cudaFree(p);
}

void ClockCache::reserve(uint64_t cap) {
  if (slot_cap_ >= cap) return;
  if (slot_) cuda_check(cudaFree(slot_), "cudaFree");
  slot_cap_ = cap;
  cuda_check(cudaMalloc(&slot_, cap * 4), "cudaMalloc");
}

void ClockCache::gather(const void* table, const uint32_t* row_map, const uint32_t* d_ids,
                        const unsigned long long* d_count, uint64_t cap, void* d_out,
                        cudaStream_t st) {
  if (cap == 0) return;
  reserve(cap);
  ++epoch_;
  const unsigned grid = cbdev::kNumSMs * 8;
  launch_k(clock_lookup_kernel, grid, 256, st, view_, d_ids, d_count, cap, slot_, epoch_, ctr_);
  CB_LAUNCH("clock_lookup");
  dispatch(row_bytes_, [&](auto v) {
    using V = decltype(v);
    const uint32_t vpr = static_cast<uint32_t>(row_bytes_ / sizeof(V));
    launch_k(clock_serve_kernel<V>, grid, 256, st, view_, static_cast<const V*>(table), row_map,
             d_ids, d_count, cap, slot_, vpr, static_cast<V*>(d_out));
    CB_LAUNCH("clock_serve");
    launch_k(clock_insert_kernel<V>, grid, 256, st, view_, d_ids, d_count, cap, slot_, epoch_,
             vpr, static_cast<const V*>(d_out), ctr_ + 1);
    CB_LAUNCH("clock_insert");
  });
}

void ClockCache::counters(cudaStream_t st, uint64_t* hits, uint64_t* inserted) {
  unsigned long long h[2];
  cuda_check(cudaMemcpyAsync(h, ctr_, 16, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (hits) *hits = h[0];
  if (inserted) *inserted = h[1];
}

}  // namespace cb
