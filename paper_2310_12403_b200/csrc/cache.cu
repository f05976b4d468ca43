// Batch-exact LRU feature cache on the device (see cache.h for the model).
// Reference semantics: LruCache::access (cache.cpp:12-27) applied key by key
// in access_order (cache.cpp:74-84); feature_load_sim (cache.cpp:88-119) and
// run_dependent_experiment (cache.cpp:137-208) feed it one id set per step.
//
// Per batch of B distinct keys (all on the plan/cache stream):
//   order     : h = mix64(v ^ key), stable radix sort of (h, kept index)
//   lookup    : rho_i = #keys newer than the key's last access (time bitmap
//               popcount against the exclusive word prefix), INF if unseen
//   merge     : X_i = #{j < i : rho_j < rho_i}, bottom-up merge count
//               (1024-element shared-memory tiles, then global levels)
//   decide    : hit_i = rho_i + i - X_i < C; row source = cache slot / table
//   gather    : rows of the kept ids, kept order (before any slot changes)
//   update    : clear old time bits, set the batch's, last[v] = T + 1 + i
//   evict     : slots whose key is no longer among the C newest are freed
//   assign    : keys resident at the end without a slot take freed / new
//               slots; their rows are copied into the storage (fill)
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstring>

#include "cache.h"
#include "cb_internal.h"

namespace cb {
using namespace cbdev;

namespace {

constexpr uint32_t kInf = 0xffffffffu;
constexpr int kMT = 1024;  // merge tile = threads of the tile kernel
enum { kHits = 0, kFree = 1, kNeed = 2, kUsed = 3, kKept = 4, kDistinct = 5, kNCtr = 8 };

// #keys whose latest access is newer than t (bits above t in the time bitmap)
__device__ __forceinline__ uint32_t newer_than(const uint32_t* __restrict__ M,
                                               const uint32_t* __restrict__ P, uint32_t total,
                                               uint32_t t) {
  const uint32_t w = t >> 5, b = t & 31u;
  return total - (P[w] + __popc(M[w] & ((2u << b) - 1u)));
}

struct OwnedBy {
  const uint32_t* owner;
  uint32_t part;
  __device__ __forceinline__ bool operator()(const uint32_t v) const { return owner[v] == part; }
};

struct PopcOp {
  __device__ __forceinline__ uint32_t operator()(const uint32_t w) const { return __popc(w); }
};

__global__ void order_keys_kernel(const uint32_t* __restrict__ kept, uint64_t B, uint64_t key,
                                  unsigned long long* h, uint32_t* val) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < B;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    h[j] = mix64(static_cast<uint64_t>(kept[j]) ^ key);
    val[j] = static_cast<uint32_t>(j);
  }
}

__global__ void lookup_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ord,
                              uint64_t B, const uint32_t* __restrict__ last,
                              const uint32_t* __restrict__ M, const uint32_t* __restrict__ P,
                              uint32_t W, uint32_t* rho, uint32_t* mk, uint32_t* mi,
                              uint32_t* xcnt) {
  const uint32_t total = P[W];
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < B;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = keys[ord ? ord[i] : i];
    const uint32_t t = last[v];
    const uint32_t r = t ? newer_than(M, P, total, t) : kInf;
    rho[i] = r;
    mk[i] = r;
    mi[i] = static_cast<uint32_t>(i);
    xcnt[i] = 0;
  }
}

// #elements < key (LT) or <= key (!LT) in the sorted run a[0..n)
template <bool LT>
__device__ __forceinline__ uint32_t rank_in(const uint32_t* a, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (LT ? a[mid] < key : a[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Stable merge of sorted halves; right-half elements add #left < key to X.
__device__ __forceinline__ void merge_step(const uint32_t* k, uint32_t p, uint32_t w, uint32_t n,
                                           uint32_t key, uint32_t& dst, uint32_t& x_add) {
  const uint32_t blk = p / w, lo = blk * w, pair_lo = (blk & ~1u) * w;
  x_add = 0;
  if ((blk & 1u) == 0) {
    const uint32_t o0 = lo + w;
    const uint32_t o1 = min(lo + 2 * w, n);
    const uint32_t c = o0 < o1 ? rank_in<true>(k + o0, o1 - o0, key) : 0u;
    dst = pair_lo + (p - lo) + c;
  } else {
    const uint32_t o0 = lo - w;
    x_add = rank_in<true>(k + o0, w, key);
    dst = pair_lo + (p - lo) + rank_in<false>(k + o0, w, key);
  }
}

__global__ void __launch_bounds__(kMT) merge_tile_kernel(uint32_t* mk, uint32_t* mi,
                                                         uint32_t* xcnt, uint64_t B) {
  __shared__ uint32_t sk[2][kMT], si[2][kMT], sx[2][kMT];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kMT;
  const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kMT), B - base));
  const uint32_t p = threadIdx.x;
  if (p < n) {
    sk[0][p] = mk[base + p];
    si[0][p] = mi[base + p];
    sx[0][p] = 0;
  }
  __syncthreads();
  int c = 0;
  for (uint32_t w = 1; w < n; w <<= 1) {
    if (p < n) {
      uint32_t dst, xa;
      merge_step(sk[c], p, w, n, sk[c][p], dst, xa);
      sk[c ^ 1][dst] = sk[c][p];
      si[c ^ 1][dst] = si[c][p];
      sx[c ^ 1][dst] = sx[c][p] + xa;
    }
    __syncthreads();
    c ^= 1;
  }
  if (p < n) {
    mk[base + p] = sk[c][p];
    mi[base + p] = si[c][p];
    xcnt[si[c][p]] = sx[c][p];
  }
}

__global__ void merge_level_kernel(const uint32_t* __restrict__ ik, const uint32_t* __restrict__ ii,
                                   uint32_t* ok, uint32_t* oi, uint32_t* xcnt, uint32_t w,
                                   uint32_t B) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < B; p += gridDim.x * blockDim.x) {
    const uint32_t key = ik[p], idx = ii[p];
    uint32_t dst, xa;
    merge_step(ik, p, w, B, key, dst, xa);
    ok[dst] = key;
    oi[dst] = idx;
    if (xa) xcnt[idx] += xa;
  }
}

__global__ void decide_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ord,
                              uint64_t B, const uint32_t* __restrict__ rho,
                              const uint32_t* __restrict__ xcnt, uint64_t cap, uint8_t* miss,
                              const int32_t* __restrict__ slot_of, const unsigned char* rows,
                              const unsigned char* table, const uint32_t* __restrict__ row_map,
                              const void* const* __restrict__ miss_ptr,
                              uint64_t row_bytes, const void** src_ptr,
                              unsigned long long* ctr) {
  unsigned long long h = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < B;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = rho[i];
    const bool hit = r != kInf && static_cast<uint64_t>(r) + i - xcnt[i] < cap;
    h += hit;
    if (miss) miss[i] = hit ? 0 : 1;
    if (src_ptr) {
      const uint32_t j = ord ? ord[i] : static_cast<uint32_t>(i);
      const uint32_t v = keys[j];
      src_ptr[j] = hit ? static_cast<const void*>(rows + static_cast<uint64_t>(slot_of[v]) * row_bytes)
                   : miss_ptr ? miss_ptr[j]
                              : static_cast<const void*>(table + static_cast<uint64_t>(
                                                                     row_map ? row_map[v] : v) *
                                                                     row_bytes);
    }
  }
  h = warp_sum(h);
  if (lane_id() == 0 && h) atomicAdd(&ctr[kHits], h);
}

// out[x] = src_ptr[row][vec] over the flattened (row, vector) space
template <typename V>
__global__ void copy_rows_kernel(const void* const* __restrict__ src_ptr, uint64_t rows,
                                 uint32_t vpr, V* __restrict__ out) {
  const uint64_t total = rows * vpr;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = x / vpr, c = x - r * vpr;
    out[x] = static_cast<const V*>(src_ptr[r])[c];
  }
}

__global__ void update_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ord,
                              uint64_t B, uint32_t T, uint32_t* last, uint32_t* M,
                              unsigned long long* ctr) {
  unsigned long long fresh = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < B;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = keys[ord ? ord[i] : i];
    const uint32_t t = last[v];
    if (t) atomicAnd(&M[t >> 5], ~(1u << (t & 31u)));
    else ++fresh;
    const uint32_t nt = T + 1u + static_cast<uint32_t>(i);
    atomicOr(&M[nt >> 5], 1u << (nt & 31u));
    last[v] = nt;
  }
  fresh = warp_sum(fresh);
  if (lane_id() == 0 && fresh) atomicAdd(&ctr[kDistinct], fresh);
}

__global__ void evict_kernel(const uint32_t* __restrict__ slot_key, uint64_t cap,
                             const uint32_t* __restrict__ last, const uint32_t* __restrict__ M,
                             const uint32_t* __restrict__ P, uint32_t W, int32_t* slot_of,
                             uint32_t* free_list, unsigned long long* ctr) {
  const uint32_t total = P[W];
  const uint64_t used = ctr[kUsed];
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < used;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = slot_key[s];
    if (newer_than(M, P, total, last[k]) >= cap) {
      slot_of[k] = -1;
      free_list[atomicAdd(&ctr[kFree], 1ULL)] = static_cast<uint32_t>(s);
    }
  }
}

__global__ void assign_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ord,
                              uint64_t B, uint64_t cap, int32_t* slot_of, uint32_t* slot_key,
                              const uint32_t* __restrict__ free_list, uint32_t* fill_slot,
                              uint32_t* fill_row, unsigned long long* ctr) {
  const uint64_t nfree = ctr[kFree], used = ctr[kUsed];
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < B;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (B - 1 - i >= cap) continue;  // evicted again within this batch
    const uint32_t j = ord ? ord[i] : static_cast<uint32_t>(i);
    const uint32_t v = keys[j];
    if (slot_of[v] >= 0) continue;
    const uint64_t r = atomicAdd(&ctr[kNeed], 1ULL);
    const uint64_t s = r < nfree ? free_list[r] : used + (r - nfree);
    slot_of[v] = static_cast<int32_t>(s);
    slot_key[s] = v;
    if (fill_slot) {
      fill_slot[r] = static_cast<uint32_t>(s);
      fill_row[r] = j;
    }
  }
}

__global__ void finalize_kernel(unsigned long long* ctr) {
  if (ctr[kNeed] > ctr[kFree]) ctr[kUsed] += ctr[kNeed] - ctr[kFree];
}

template <typename V>
__global__ void fill_kernel(const uint32_t* __restrict__ fill_slot,
                            const uint32_t* __restrict__ fill_row, const unsigned long long* ctr,
                            uint32_t vpr, const V* __restrict__ rows_out, V* storage) {
  const uint64_t total = ctr[kNeed] * vpr;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = x / vpr, c = x - r * vpr;
    storage[static_cast<uint64_t>(fill_slot[r]) * vpr + c] =
        rows_out[static_cast<uint64_t>(fill_row[r]) * vpr + c];
  }
}

__global__ void compact_kernel(uint64_t n, uint32_t* last, const uint32_t* __restrict__ M,
                               const uint32_t* __restrict__ P) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = last[v];
    if (t) {
      const uint32_t w = t >> 5, b = t & 31u;
      last[v] = 1u + P[w] + __popc(M[w] & ((1u << b) - 1u));
    }
  }
}

__global__ void set_prefix_bits_kernel(uint32_t* M, uint64_t words, uint64_t K) {
  // bits 1..K set, everything else clear
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b0 = w * 32, b1 = b0 + 32;
    uint32_t m = 0;
    for (uint64_t b = max(b0, static_cast<uint64_t>(1)); b < b1 && b <= K; ++b)
      m |= 1u << (b - b0);
    M[w] = m;
  }
}

int grid_of(uint64_t n, int per = 256, int max_per_sm = 8) {
  return static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>((n + per - 1) / per, static_cast<uint64_t>(kNumSMs) * max_per_sm)));
}

int vec_of(uint64_t row_bytes) {
  for (int v : {16, 8, 4, 2})
    if (row_bytes % v == 0) return v;
  return 1;
}

template <typename F>
void dispatch_vec(int vb, F&& f) {
  switch (vb) {
    case 16: f(uint4{}); break;
    case 8: f(uint2{}); break;
    case 4: f(uint32_t{}); break;
    case 2: f(static_cast<unsigned short>(0)); break;
    default: f(static_cast<unsigned char>(0));
  }
}

}  // namespace

DeviceLru::DeviceLru(int device, uint64_t n_keys, uint64_t capacity, uint64_t row_bytes)
    : device_(device), n_(n_keys), cap_(capacity), row_bytes_(row_bytes) {
  require(capacity >= 1, "LruCache: capacity must be >= 1");
  require(n_keys >= 1 && n_keys < 0x7fffffffULL, "LruCache: key space must be in [1, 2^31)");
  tbits_ = ((std::max<uint64_t>(2 * n_keys + 64, 1 << 16) + 31) / 32) * 32;
  const uint64_t W = tbits_ / 32;
  CB_CUDA(cudaMalloc(&last_, n_ * 4));
  CB_CUDA(cudaMalloc(&tmark_, (W + 1) * 4));
  CB_CUDA(cudaMalloc(&tpre_, (W + 1) * 4));
  CB_CUDA(cudaMalloc(&slot_of_, n_ * 4));
  CB_CUDA(cudaMalloc(&slot_key_, std::min(cap_, n_) * 4));
  CB_CUDA(cudaMalloc(&ctr_, kNCtr * 8));
  CB_CUDA(cudaMemset(last_, 0, n_ * 4));
  CB_CUDA(cudaMemset(tmark_, 0, (W + 1) * 4));
  CB_CUDA(cudaMemset(tpre_, 0, (W + 1) * 4));
  CB_CUDA(cudaMemset(slot_of_, 0xff, n_ * 4));
  CB_CUDA(cudaMemset(ctr_, 0, kNCtr * 8));
  if (row_bytes_) CB_CUDA(cudaMalloc(&rows_, std::min(cap_, n_) * row_bytes_ + 16));
}

DeviceLru::~DeviceLru() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  for (void* p : {(void*)last_, (void*)tmark_, (void*)tpre_, (void*)slot_of_, (void*)slot_key_,
                  (void*)rows_, (void*)ctr_, (void*)kept_, (void*)ord_, (void*)ord2_,
                  (void*)rho_, (void*)xcnt_, (void*)mk_[0], (void*)mk_[1], (void*)mi_[0],
                  (void*)mi_[1], (void*)free_, (void*)fill_slot_, (void*)fill_row_,
                  (void*)hkey_, (void*)hkey2_, (void*)src_ptr_, cub_tmp_})
    if (p) cudaFree(p);
  cudaSetDevice(prev);
}

void DeviceLru::ensure_batch(uint64_t B) {
  if (B <= bcap_) return;
  const uint64_t c = std::max<uint64_t>(B, 2 * bcap_);
  for (void* p : {(void*)kept_, (void*)ord_, (void*)ord2_, (void*)rho_, (void*)xcnt_,
                  (void*)mk_[0], (void*)mk_[1], (void*)mi_[0], (void*)mi_[1],
                  (void*)fill_slot_, (void*)fill_row_, (void*)hkey_, (void*)hkey2_,
                  (void*)src_ptr_, cub_tmp_})
    if (p) CB_CUDA(cudaFree(p));
  for (uint32_t** p : {&kept_, &ord_, &ord2_, &rho_, &xcnt_, &mk_[0], &mk_[1], &mi_[0], &mi_[1],
                       &fill_slot_, &fill_row_})
    CB_CUDA(cudaMalloc(p, c * 4 + 16));
  CB_CUDA(cudaMalloc(&hkey_, c * 8 + 16));
  CB_CUDA(cudaMalloc(&hkey2_, c * 8 + 16));
  CB_CUDA(cudaMalloc(&src_ptr_, c * 8 + 16));
  if (!free_) CB_CUDA(cudaMalloc(&free_, std::min(cap_, n_) * 4 + 16));
  // CUB scratch: radix sort of c pairs, select of c ids, scan of the time words
  size_t a = 0, b = 0, d = 0;
  cub::DoubleBuffer<unsigned long long> kb(hkey_, hkey2_);
  cub::DoubleBuffer<uint32_t> vb(ord2_, ord_);
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, static_cast<int64_t>(c)));
  CB_CUDA(cub::DeviceSelect::If(nullptr, b, kept_, kept_, ctr_ + kKept,
                                static_cast<int64_t>(c), OwnedBy{nullptr, 0}));
  auto it = thrust::make_transform_iterator(static_cast<const uint32_t*>(tmark_), PopcOp{});
  CB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, d, it, tpre_,
                                        static_cast<int64_t>(tbits_ / 32 + 1)));
  cub_bytes_ = std::max({a, b, d}) + 256;
  CB_CUDA(cudaMalloc(&cub_tmp_, cub_bytes_));
  bcap_ = c;
}

void DeviceLru::prefix_time(cudaStream_t st) {
  // exclusive popcount prefix over words [0, W]; tpre_[W] = set bits in [0, W)
  const uint64_t W = (T_ >> 5) + 1;
  size_t bytes = cub_bytes_;
  auto it = thrust::make_transform_iterator(static_cast<const uint32_t*>(tmark_), PopcOp{});
  CB_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp_, bytes, it, tpre_, static_cast<int64_t>(W + 1),
                                        st));
}

void DeviceLru::compact_time(cudaStream_t st) {
  prefix_time(st);
  const uint64_t W = (T_ >> 5) + 1;
  compact_kernel<<<grid_of(n_), 256, 0, st>>>(n_, last_, tmark_, tpre_);
  CB_LAUNCH("cache_compact");
  uint32_t K = 0;
  CB_CUDA(cudaMemcpyAsync(&K, tpre_ + W, 4, cudaMemcpyDeviceToHost, st));
  CB_CUDA(cudaStreamSynchronize(st));
  set_prefix_bits_kernel<<<grid_of(W), 256, 0, st>>>(tmark_, W, K);
  CB_LAUNCH("cache_compact_bits");
  T_ = K;
}

void DeviceLru::run_batch(const uint32_t* keys, const uint32_t* ord, uint64_t B, uint8_t* d_miss,
                          const CacheGatherSrc* src, cudaStream_t st) {
  if (B == 0) return;
  require(B <= n_, "cache batch larger than the key space");
  ensure_batch(B);
  if (T_ + B + 1 >= tbits_) compact_time(st);
  CB_CUDA(cudaMemsetAsync(ctr_ + kHits, 0, 3 * 8, st));  // hits, free, need
  prefix_time(st);
  const uint32_t W0 = static_cast<uint32_t>((T_ >> 5) + 1);
  lookup_kernel<<<grid_of(B), 256, 0, st>>>(keys, ord, B, last_, tmark_, tpre_, W0, rho_,
                                            mk_[0], mi_[0], xcnt_);
  CB_LAUNCH("cache_lookup");
  merge_tile_kernel<<<static_cast<unsigned>((B + kMT - 1) / kMT), kMT, 0, st>>>(mk_[0], mi_[0],
                                                                                 xcnt_, B);
  CB_LAUNCH("cache_merge_tile");
  int c = 0;
  for (uint64_t w = kMT; w < B; w <<= 1) {
    merge_level_kernel<<<grid_of(B), 256, 0, st>>>(mk_[c], mi_[c], mk_[c ^ 1], mi_[c ^ 1], xcnt_,
                                                   static_cast<uint32_t>(w),
                                                   static_cast<uint32_t>(B));
    CB_LAUNCH("cache_merge_level");
    c ^= 1;
  }
  const bool gather = src && src->rows_out && (src->table || src->miss_ptr);
  const int vb = vec_of(row_bytes_);
  decide_kernel<<<grid_of(B), 256, 0, st>>>(
      keys, ord, B, rho_, xcnt_, cap_, d_miss, slot_of_, rows_,
      gather ? static_cast<const unsigned char*>(src->table) : nullptr,
      gather ? src->row_map : nullptr, gather ? src->miss_ptr : nullptr, row_bytes_,
      gather ? src_ptr_ : nullptr, ctr_);
  CB_LAUNCH("cache_decide");
  if (gather) {
    const uint32_t vpr = static_cast<uint32_t>(row_bytes_ / vb);
    dispatch_vec(vb, [&](auto v) {
      using V = decltype(v);
      copy_rows_kernel<V><<<grid_of(B * vpr), 256, 0, st>>>(src_ptr_, B, vpr,
                                                            static_cast<V*>(src->rows_out));
    });
    CB_LAUNCH("cache_gather");
  }
  update_kernel<<<grid_of(B), 256, 0, st>>>(keys, ord, B, static_cast<uint32_t>(T_), last_,
                                            tmark_, ctr_);
  CB_LAUNCH("cache_update");
  T_ += B;
  prefix_time(st);
  const uint32_t W1 = static_cast<uint32_t>((T_ >> 5) + 1);
  const uint64_t slots = std::min(cap_, n_);
  evict_kernel<<<grid_of(slots), 256, 0, st>>>(slot_key_, cap_, last_, tmark_, tpre_, W1,
                                               slot_of_, free_, ctr_);
  CB_LAUNCH("cache_evict");
  const bool fill = gather && rows_;
  assign_kernel<<<grid_of(B), 256, 0, st>>>(keys, ord, B, cap_, slot_of_, slot_key_, free_,
                                            fill ? fill_slot_ : nullptr, fill_row_, ctr_);
  CB_LAUNCH("cache_assign");
  if (fill) {
    const uint32_t vpr = static_cast<uint32_t>(row_bytes_ / vb);
    dispatch_vec(vb, [&](auto v) {
      using V = decltype(v);
      fill_kernel<V><<<grid_of(B * vpr), 256, 0, st>>>(fill_slot_, fill_row_, ctr_, vpr,
                                                       static_cast<const V*>(src->rows_out),
                                                       reinterpret_cast<V*>(rows_));
    });
    CB_LAUNCH("cache_fill");
  }
  finalize_kernel<<<1, 1, 0, st>>>(ctr_);
  CB_LAUNCH("cache_finalize");
  unsigned long long h[kNCtr];
  CB_CUDA(cudaMemcpyAsync(h, ctr_, sizeof(h), cudaMemcpyDeviceToHost, st));
  CB_CUDA(cudaStreamSynchronize(st));
  hits_ += h[kHits];
  misses_ += B - h[kHits];
  distinct_ = h[kDistinct];
}

uint64_t DeviceLru::access_ids(const uint32_t* d_ids, uint64_t n, uint64_t order_key,
                               const uint32_t* d_owner, uint32_t part,
                               const CacheGatherSrc& src, cudaStream_t st) {
  if (n == 0) return 0;
  ensure_batch(n);
  const uint32_t* kept = d_ids;
  uint64_t B = n;
  if (d_owner) {
    size_t bytes = cub_bytes_;
    CB_CUDA(cub::DeviceSelect::If(cub_tmp_, bytes, d_ids, kept_, ctr_ + kKept,
                                  static_cast<int64_t>(n), OwnedBy{d_owner, part}, st));
    unsigned long long k = 0;
    CB_CUDA(cudaMemcpyAsync(&k, ctr_ + kKept, 8, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
    kept = kept_;
    B = k;
    if (B == 0) return 0;
  }
  order_keys_kernel<<<grid_of(B), 256, 0, st>>>(kept, B, order_key, hkey_, ord2_);
  CB_LAUNCH("cache_order_keys");
  cub::DoubleBuffer<unsigned long long> kb(hkey_, hkey2_);
  cub::DoubleBuffer<uint32_t> vb(ord2_, ord_);
  size_t bytes = cub_bytes_;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp_, bytes, kb, vb, static_cast<int64_t>(B), 0, 64,
                                          st));
  run_batch(kept, vb.Current(), B, nullptr, &src, st);
  return B;
}

void DeviceLru::access_ordered(const uint32_t* d_keys, uint64_t B, uint8_t* d_miss,
                               cudaStream_t st) {
  run_batch(d_keys, nullptr, B, d_miss, nullptr, st);
}

void DeviceLru::access_trace(const uint32_t* keys, uint64_t n, uint8_t* miss, cudaStream_t st) {
  for (uint64_t i = 0; i < n; ++i) require(keys[i] < n_, "LruCache: key outside the key space");
  DevBuf b_keys(n * 4 + 16), b_miss(n + 16);
  uint32_t* d_keys = b_keys.as<uint32_t>();
  uint8_t* d_miss = b_miss.as<uint8_t>();
  CB_CUDA(cudaMemcpyAsync(d_keys, keys, n * 4, cudaMemcpyHostToDevice, st));
  std::vector<uint8_t> in_run;
  in_run.assign(n_, 0);
  uint64_t start = 0;
  while (start < n) {
    uint64_t end = start;
    while (end < n && !in_run[keys[end]]) in_run[keys[end++]] = 1;
    run_batch(d_keys + start, nullptr, end - start, d_miss + start, nullptr, st);
    for (uint64_t i = start; i < end; ++i) in_run[keys[i]] = 0;
    start = end;
  }
  CB_CUDA(cudaMemcpyAsync(miss, d_miss, n, cudaMemcpyDeviceToHost, st));
  CB_CUDA(cudaStreamSynchronize(st));
}

uint64_t DeviceLru::size() const { return std::min(cap_, distinct_); }

void DeviceLru::resident(std::vector<uint32_t>& out) {
  std::vector<uint32_t> last(n_);
  CB_CUDA(cudaMemcpy(last.data(), last_, n_ * 4, cudaMemcpyDeviceToHost));
  std::vector<std::pair<uint32_t, uint32_t>> tv;
  for (uint64_t v = 0; v < n_; ++v)
    if (last[v]) tv.push_back({last[v], static_cast<uint32_t>(v)});
  std::sort(tv.begin(), tv.end(), [](auto& a, auto& b) { return a.first > b.first; });
  out.clear();
  for (uint64_t i = 0; i < tv.size() && i < cap_; ++i) out.push_back(tv[i].second);
}

}  // namespace cb
