// C-ABI: per-GPU LRU feature cache, fingerprints, training order, storage tier,
// async meta copies, launch counters, CBCS helpers (see coopbatch_cuda.h).
#include "capi_internal.h"

extern "C" {

// ------------------------------------------------------------- LRU cache --
int cb_cache_create(int device, uint64_t n_keys, uint64_t capacity, uint64_t row_bytes,
                    cb_cache** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(capacity >= 1, "LruCache: capacity must be >= 1");
    DeviceGuard dg(device);
    auto c = std::make_unique<cb_cache>();
    c->lru = std::make_unique<DeviceLru>(device, n_keys, capacity, row_bytes);
    CB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c.release();
  });
}

void cb_cache_destroy(cb_cache* c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->lru->device());
  delete c;
  cudaSetDevice(prev);
}

int cb_cache_access_trace(cb_cache* c, const uint32_t* keys, uint64_t n, uint8_t* miss) {
  return guard([&] {
    require(c != nullptr && (n == 0 || (keys != nullptr && miss != nullptr)), "null argument");
    DeviceGuard dg(c->lru->device());
    c->lru->access_trace(keys, n, miss, c->stream);
  });
}

int cb_cache_access_ids(cb_cache* c, const uint32_t* d_ids, uint64_t n, uint64_t order_key,
                        const cb_partition* pm, uint32_t part, const cb_features* backing,
                        void* d_rows_out, uint64_t* kept, void* stream) {
  NvtxRange nvtx_("cb.cache_access");
  return guard([&] {
    require(c != nullptr, "null cache");
    require(pm == nullptr || part < pm->parts, "part index out of range");
    require(d_rows_out == nullptr || backing != nullptr, "rows requested without a table");
    if (backing) require_full_table(backing);
    require(backing == nullptr || c->lru->row_bytes() == 0 ||
                backing->row_bytes == c->lru->row_bytes(),
            "cache row size does not match the feature table");
    DeviceGuard dg(c->lru->device());
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    CacheGatherSrc src;
    if (backing && d_rows_out) {
      src.table = backing->table;
      src.row_map = backing->row_map;
      src.rows_out = d_rows_out;
    }
    const uint64_t k = c->lru->access_ids(d_ids, n, order_key, pm ? pm->owner : nullptr,
                                          part, src, st);
    if (kept) *kept = k;
  });
}

int cb_cache_access_plan(cb_cache* c, cb_plan* plan, uint32_t part, uint64_t order_key,
                         const cb_partition* pm, uint32_t owner_part,
                         const cb_features* backing, void* d_rows_out, uint64_t* kept) {
  NvtxRange nvtx_("cb.cache_access_plan");
  return guard([&] {
    require(c != nullptr && plan != nullptr, "null argument");
    require_batch(plan, part, plan->L - 1);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const uint64_t n = host_meta(plan, part, plan->L - 1).n_src;
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    const uint32_t* ids = plan->pe[part].L[plan->L - 1].src;
    if (backing && !d_rows_out) {  // rows land in the plan's own row buffer
      require(pm == nullptr, "plan row buffer holds all input rows: no owner filter");
      prepare_rows(plan, backing);
      d_rows_out = plan->pe[part].rows;
      plan->have_rows = true;
    }
    CacheGatherSrc src;
    if (backing) require_full_table(backing);
    if (backing && d_rows_out) {
      require(c->lru->row_bytes() == 0 || backing->row_bytes == c->lru->row_bytes(),
              "cache row size does not match the feature table");
      src.table = backing->table;
      src.row_map = backing->row_map;
      src.rows_out = d_rows_out;
    }
    const uint64_t k = c->lru->access_ids(ids, n, order_key, pm ? pm->owner : nullptr,
                                          owner_part, src, plan->stream);
    if (kept) *kept = k;
  });
}

int cb_cache_access_host_ids(cb_cache* c, const uint32_t* ids, uint64_t n, uint64_t order_key,
                             const cb_partition* pm, uint32_t part, uint64_t* kept) {
  return guard([&] {
    require(c != nullptr && (n == 0 || ids != nullptr), "null argument");
    require(pm == nullptr || part < pm->parts, "part index out of range");
    DeviceGuard dg(c->lru->device());
    DevBuf buf(n * 4 + 16);
    uint32_t* d = buf.as<uint32_t>();
    // the batch-exact LRU assumes distinct keys inside the key space
    // (LruCache::access would count a repeat as a hit; that is a trace, see
    // cb_cache_access_trace)
    {
      std::vector<uint32_t> sorted(ids, ids + n);
      std::sort(sorted.begin(), sorted.end());
      require(n == 0 || sorted.back() < c->lru->n_keys(), "cache access: id outside the key space");
      require(std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end(),
              "cache access: ids of one access set must be distinct");
    }
    CB_CUDA(cudaMemcpyAsync(d, ids, n * 4, cudaMemcpyHostToDevice, c->stream));
    const uint64_t k = c->lru->access_ids(d, n, order_key, pm ? pm->owner : nullptr, part,
                                          CacheGatherSrc{}, c->stream);
    if (kept) *kept = k;
  });
}

int cb_cache_stats(const cb_cache* c, uint64_t* hits, uint64_t* misses, uint64_t* size) {
  return guard([&] {
    require(c != nullptr, "null cache");
    if (hits) *hits = c->lru->hits();
    if (misses) *misses = c->lru->misses();
    if (size) *size = c->lru->size();
  });
}

int cb_cache_reset_counters(cb_cache* c) {
  return guard([&] {
    require(c != nullptr, "null cache");
    c->lru->reset_counters();
  });
}

int cb_cache_resident(cb_cache* c, uint32_t* out, uint64_t cap_out, uint64_t* n) {
  return guard([&] {
    require(c != nullptr && n != nullptr, "null argument");
    DeviceGuard dg(c->lru->device());
    std::vector<uint32_t> r;
    c->lru->resident(r);
    require(out == nullptr || cap_out >= r.size(), "output buffer too small");
    if (out) std::memcpy(out, r.data(), r.size() * 4);
    *n = r.size();
  });
}

int cb_cache_storage(const cb_cache* c, const void** d_rows) {
  return guard([&] {
    require(c != nullptr && d_rows != nullptr, "null argument");
    *d_rows = c->lru->storage();
  });
}

// stack_fingerprint (cache.cpp:123-133): sequential mix64 fold over the
// downloaded blocks of part p, computed on the host.
int cb_stack_fingerprint(cb_plan* plan, uint32_t part, uint64_t* out) {
  return guard([&] {
    require(plan != nullptr && out != nullptr, "null argument");
    require_batch(plan, part, 0);
    uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int l = 0; l < plan->L; ++l) {
      uint64_t sz[6];
      if (cb_layer_sizes(plan, part, l, sz) != CB_OK) throw Error(kCuda, g_err);
      std::vector<uint32_t> dst(sz[0]), src(sz[1]), edges(2 * sz[2]);
      if (cb_download_block(plan, part, l, dst.data(), src.data(), edges.data(), nullptr) !=
          CB_OK)
        throw Error(kCuda, g_err);
      h = cbdev::mix64(h ^ static_cast<uint64_t>(l));
      for (uint32_t v : dst) h = cbdev::mix64(h ^ v);
      for (uint32_t v : src) h = cbdev::mix64(h ^ (0x100000000ULL | v));
      for (uint64_t e = 0; e < sz[2]; ++e)
        h = cbdev::mix64(h ^ ((static_cast<uint64_t>(edges[2 * e]) << 32) | edges[2 * e + 1]));
    }
    *out = h;
  });
}

// Fixed training order of run_dependent_experiment (cache.cpp:155-162):
// Fisher-Yates with j = (u64)(hash_uniform(seed, {kStreamSeedDraw, i}) * i).
int cb_shuffled_order(uint64_t n, uint64_t seed, uint32_t* out) {
  return guard([&] {
    require(out != nullptr || n == 0, "null argument");
    for (uint64_t v = 0; v < n; ++v) out[v] = static_cast<uint32_t>(v);
    const uint64_t pfx = cbdev::hstep(cbdev::hinit(seed), 8ULL);
    for (uint64_t i = n; i > 1; --i) {
      const double u = cbdev::ufb(cbdev::hstep(pfx, i));
      const uint64_t j = static_cast<uint64_t>(u * static_cast<double>(i));
      std::swap(out[i - 1], out[std::min(j, i - 1)]);
    }
  });
}

// Storage tier of a feature table: 1 = pinned host memory mapped into the
// device address space (rows then cross the host link on every miss),
// 0 = HBM. The row layout is unchanged.
int cb_features_set_tier(cb_features* f, int host) {
  return guard([&] {
    require(f != nullptr, "null features");
    DeviceGuard dg(f->device);
    // a single-part shard holds shard_rows rows behind a virtual base
    // (table + shard_r0 rows is the allocation); the tier moves those rows
    const uint64_t rows = f->shard_rows ? f->shard_rows : f->n_rows;
    const uint64_t off = f->shard_rows ? f->shard_r0 * f->row_bytes : 0;
    const uint64_t bytes = rows * f->row_bytes;
    const bool on_host = f->host_base != nullptr;
    if (static_cast<bool>(host) == on_host) return;
    CB_CUDA(cudaDeviceSynchronize());
    if (host) {
      void* h = nullptr;
      CB_CUDA(cudaHostAlloc(&h, bytes + 64, cudaHostAllocMapped | cudaHostAllocPortable));
      CB_CUDA(cudaMemcpy(h, static_cast<unsigned char*>(f->table) + off, bytes,
                         cudaMemcpyDeviceToHost));
      void* d = nullptr;
      CB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
      f->hbm_table = f->table;
      f->host_base = h;
      f->table = static_cast<unsigned char*>(d) - off;
    } else {
      h2d_sync(static_cast<unsigned char*>(f->hbm_table) + off, f->host_base, bytes);
      CB_CUDA(cudaFreeHost(f->host_base));
      f->host_base = nullptr;
      f->table = f->hbm_table;
      f->hbm_table = nullptr;
    }
  });
}

int cb_plan_set_rw(cb_plan* plan, uint32_t rw_length, double rw_restart, uint32_t rw_walks) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(rw_length >= 1 && rw_walks >= 1, "sample_rw: rw_length and rw_walks must be >= 1");
    require(rw_restart >= 0.0 && rw_restart < 1.0, "sample_rw: rw_restart must be in [0, 1)");
    require(static_cast<uint64_t>(rw_length) * rw_walks <= kRwMaxVisits,
            "rw_walks * rw_length must be <= 512 on the device");
    plan->rw_length = rw_length;
    plan->rw_restart = rw_restart;
    plan->rw_walks = rw_walks;
    plan->drop_graphs();
  });
}

int cb_plan_meta_async(cb_plan* plan, void* host_dst, uint64_t* bytes) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    const uint64_t nb = sizeof(LayerMeta) * plan->P * (plan->L + 1);
    if (bytes) *bytes = nb;
    if (!host_dst) return;
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaMemcpyAsync(host_dst, plan->meta, nb, cudaMemcpyDeviceToHost, plan->stream));
  });
}

int cb_kernel_launches(uint64_t* n) {
  return guard([&] {
    require(n != nullptr, "null argument");
    *n = g_kernel_launches.load();
  });
}

int cb_plan_input_ids(cb_plan* plan, uint32_t part, const uint32_t** d_ids, uint64_t* n) {
  return guard([&] {
    require(plan != nullptr && d_ids != nullptr && n != nullptr, "null argument");
    require_batch(plan, part, plan->L - 1);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    *n = host_meta(plan, part, plan->L - 1).n_src;
    *d_ids = plan->pe[part].L[plan->L - 1].src;
  });
}

}  // extern "C"

// ---- set-associative CLOCK cache (the fast production mode) -----------------
extern "C" {

int cb_ccache_create(int device, uint64_t capacity, uint32_t ways, uint64_t row_bytes,
                     cb_ccache** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(capacity >= 1 && row_bytes >= 2, "ClockCache: capacity and row bytes must be > 0");
    DeviceGuard dg(device);
    auto c = std::make_unique<cb_ccache>();
    c->cc = std::make_unique<ClockCache>(device, capacity, ways, row_bytes);
    CB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c.release();
  });
}

void cb_ccache_destroy(cb_ccache* c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->cc->device());
  delete c;
  cudaSetDevice(prev);
}

int cb_ccache_gather_plan(cb_ccache* c, cb_plan* plan, uint32_t part, const cb_features* backing) {
  NvtxRange nvtx_("cb.ccache_gather_plan");
  return guard([&] {
    require(c != nullptr && plan != nullptr && backing != nullptr, "null argument");
    require_batch(plan, part, plan->L - 1);
    require(backing->row_bytes == c->cc->row_bytes(), "cache row size does not match the table");
    require_full_table(backing);
    DeviceGuard dg(plan->device);
    prepare_rows(plan, backing);
    PeWork& w = plan->pe[part];
    const LayerBufs& b = w.L[plan->L - 1];
    // device count, on the plan stream: no host round trip
    c->cc->gather(backing->table, backing->row_map, b.src, &plan->meta_at(part, plan->L - 1)->n_src,
                  w.cap_rows, w.rows, plan->stream);
    plan->have_rows = true;
  });
}

int cb_ccache_stats(cb_ccache* c, uint64_t* hits, uint64_t* inserted, uint64_t* capacity) {
  return guard([&] {
    require(c != nullptr, "null cache");
    DeviceGuard dg(c->cc->device());
    CB_CUDA(cudaDeviceSynchronize());
    c->cc->counters(c->stream, hits, inserted);
    if (capacity) *capacity = c->cc->capacity();
  });
}

}  // extern "C"
