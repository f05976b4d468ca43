// Drop-in replacement of the reference's src/cache.cpp: the functions declared
// in include/coopbatch/cache.hpp (unchanged).
//
//   LruCache               cache.cpp:8-32    -> host (a per-key host API whose
//                                               state is the header's own
//                                               std::list / unordered_map)
//   nested_batches         cache.cpp:34-66   -> the super batch and the kappa
//                                               sub-batches as one device batch
//   feature_load_sim       cache.cpp:88-119  -> the batch-exact LRU on the device
//                                               (csrc/cache.cu), one id set per
//                                               step and part; the callers' caches
//                                               end in the state the sequential
//                                               LRU leaves
//   run_dependent_experiment cache.cpp:137-208 -> device expansion, fingerprint
//                                               and LRU per step
#include <unordered_set>

#include "ctx.hpp"

namespace coopbatch {

// ---- LruCache state access ----------------------------------------------------
// feature_load_sim runs the accesses on the device and must then leave every
// caller-owned LruCache in the state the sequential accesses would have left
// (recency list, index, counters). The header is the reference's, unchanged,
// and declares no member for that; explicit template instantiation may name
// private members ([temp.spec.general]/6), which this uses to reach them.
namespace {

template <typename Tag, typename Tag::type M>
struct Grant {
  friend typename Tag::type get(Tag) { return M; }
};
struct RecencyTag {
  using type = std::list<VertexId> LruCache::*;
  friend type get(RecencyTag);
};
struct IndexTag {
  using type = std::unordered_map<VertexId, std::list<VertexId>::iterator> LruCache::*;
  friend type get(IndexTag);
};
struct HitsTag {
  using type = std::uint64_t LruCache::*;
  friend type get(HitsTag);
};
struct MissesTag {
  using type = std::uint64_t LruCache::*;
  friend type get(MissesTag);
};
template struct Grant<RecencyTag, &LruCache::recency_>;
template struct Grant<IndexTag, &LruCache::index_>;
template struct Grant<HitsTag, &LruCache::hits_>;
template struct Grant<MissesTag, &LruCache::misses_>;

// Replace c's contents by `resident` (most recent first) and add to its counters.
void set_state(LruCache& c, const std::vector<VertexId>& resident, std::uint64_t add_hits,
               std::uint64_t add_misses) {
  auto& rec = c.*get(RecencyTag{});
  auto& idx = c.*get(IndexTag{});
  rec.assign(resident.begin(), resident.end());
  idx.clear();
  for (auto it = rec.begin(); it != rec.end(); ++it) idx[*it] = it;
  c.*get(HitsTag{}) += add_hits;
  c.*get(MissesTag{}) += add_misses;
}

using namespace b200;

struct DeviceCache {
  cb_cache* h = nullptr;
  DeviceCache(std::uint64_t n_keys, std::uint64_t capacity) {
    check(cb_cache_create(device(), std::max<std::uint64_t>(n_keys, 1), capacity, 0, &h));
  }
  ~DeviceCache() { cb_cache_destroy(h); }
  void stats(std::uint64_t& hits, std::uint64_t& misses) const {
    check(cb_cache_stats(h, &hits, &misses, nullptr));
  }
  std::vector<VertexId> resident() const {
    std::uint64_t n = 0;
    check(cb_cache_resident(h, nullptr, 0, &n));
    std::vector<VertexId> r(n);
    if (n) check(cb_cache_resident(h, r.data(), n, &n));
    return r;
  }
};

std::uint64_t fingerprint(cb_plan* pl) {
  std::uint64_t fp = 0;
  check(cb_stack_fingerprint(pl, 0, &fp));
  return fp;
}

}  // namespace

LruCache::LruCache(std::uint64_t capacity) : capacity_(capacity) {
  if (capacity == 0) throw InputError("LruCache: capacity must be >= 1");
  index_.reserve(std::min<std::uint64_t>(capacity, 1ULL << 20));
}

CacheOutcome LruCache::access(VertexId key) {
  if (auto it = index_.find(key); it != index_.end()) {
    if (it->second != recency_.begin()) recency_.splice(recency_.begin(), recency_, it->second);
    ++hits_;
    return CacheOutcome::kHit;
  }
  ++misses_;
  if (recency_.size() == capacity_) {
    index_.erase(recency_.back());
    recency_.pop_back();
  }
  recency_.push_front(key);
  index_.emplace(key, recency_.begin());
  return CacheOutcome::kMiss;
}

std::vector<VertexId> LruCache::resident() const { return {recency_.begin(), recency_.end()}; }

std::vector<LayerStack> nested_batches(const Graph& g, std::span<const VertexId> super_seeds,
                                       std::uint64_t kappa, std::uint64_t b, int num_layers,
                                       const SamplerConfig& cfg, std::uint64_t epoch_seed) {
  if (kappa == 0 || b == 0) throw InputError("nested_batches: kappa and b must be >= 1");
  if (super_seeds.size() != kappa * b)
    throw InputError("nested_batches: super batch must hold exactly kappa*b seeds");
  // part 0: the super batch; parts 1..kappa: its slices, all under the
  // super batch's plain stream
  std::vector<std::vector<VertexId>> parts;
  parts.emplace_back(super_seeds.begin(), super_seeds.end());
  for (std::uint64_t i = 0; i < kappa; ++i)
    parts.emplace_back(super_seeds.begin() + i * b, super_seeds.begin() + (i + 1) * b);
  SeedSchedule plain;
  plain.z1 = plain.z2 = epoch_seed;
  const std::vector<LayerStack> all = indep_sample(g, parts, num_layers, cfg, plain);
  // containment, layer by layer: both lists are sorted, so a merge walk
  for (int l = 0; l < num_layers; ++l) {
    const auto& sup = all[0].blocks[l].src_vertices;
    for (std::uint64_t i = 1; i <= kappa; ++i) {
      const auto& sub = all[i].blocks[l].src_vertices;
      if (!std::includes(sup.begin(), sup.end(), sub.begin(), sub.end()))
        throw InputError("nested_batches: containment violated at layer " + std::to_string(l));
    }
  }
  return {all.begin() + 1, all.end()};
}

std::vector<CacheStats> feature_load_sim(const std::vector<std::vector<LayerStack>>& steps,
                                         std::vector<LruCache>& caches, const PartitionMap* pm,
                                         std::uint32_t dim, std::uint32_t bytes_per_scalar) {
  Lock lk(api_mutex());
  const std::size_t parts = caches.size();
  for (const auto& step : steps)
    if (step.size() != parts) throw InputError("feature_load_sim: stack/cache count mismatch");
  std::vector<CacheStats> stats(parts);
  for (std::size_t p = 0; p < parts; ++p) {
    // key space: every id this cache will see
    std::uint64_t n_keys = 1;
    for (const VertexId v : caches[p].resident()) n_keys = std::max<std::uint64_t>(n_keys, v + 1ULL);
    for (const auto& step : steps)
      if (!step[p].input_vertices().empty())
        n_keys = std::max<std::uint64_t>(n_keys, step[p].input_vertices().back() + 1ULL);
    DeviceCache dc(n_keys, caches[p].capacity());
    // start from the caller's cache: its residents accessed oldest first
    const std::vector<VertexId> start = caches[p].resident();
    if (!start.empty()) {
      std::vector<VertexId> oldest_first(start.rbegin(), start.rend());
      std::vector<std::uint8_t> miss(oldest_first.size());
      check(cb_cache_access_trace(dc.h, oldest_first.data(), oldest_first.size(), miss.data()));
      check(cb_cache_reset_counters(dc.h));
    }
    std::vector<VertexId> owned;
    for (std::size_t s = 0; s < steps.size(); ++s) {
      const auto& in = steps[s][p].input_vertices();
      const VertexId* ids = in.data();
      std::uint64_t n = in.size();
      if (pm) {  // cooperative: this part's rows only (cache.cpp:105)
        owned.clear();
        for (const VertexId v : in)
          if (pm->owner.at(v) == p) owned.push_back(v);
        ids = owned.data();
        n = owned.size();
      }
      // access_order(ids, hash_bits(step_index, {p})), cache.cpp:74-84, 100-101
      const std::uint64_t key = hash_bits(s + 1, {static_cast<std::uint64_t>(p)});
      check(cb_cache_access_host_ids(dc.h, ids, n, key, nullptr, 0, nullptr));
    }
    std::uint64_t h = 0, m = 0;
    dc.stats(h, m);
    stats[p].hits = h;
    stats[p].misses = m;
    stats[p].accesses = h + m;
    set_state(caches[p], dc.resident(), h, m);
  }
  for (auto& s : stats) {
    s.miss_rate = s.accesses == 0 ? 0.0
                                  : static_cast<double>(s.misses) / static_cast<double>(s.accesses);
    s.bytes = s.misses * static_cast<std::uint64_t>(dim) * bytes_per_scalar;
  }
  return stats;
}

DependentExperimentResult run_dependent_experiment(
    const Graph& g, const MinibatchSchedule& schedule, std::uint64_t steps,
    std::uint64_t cache_capacity, const SamplerConfig& cfg, int num_layers,
    std::uint32_t feature_dim, std::uint32_t bytes_per_scalar, std::uint64_t seed) {
  Lock lk(api_mutex());
  const std::uint64_t n = g.num_vertices;
  const std::uint64_t b = std::min<std::uint64_t>(schedule.batch_size, n);
  if (b == 0) throw InputError("run_dependent_experiment: empty batches");
  if (cache_capacity == 0) throw InputError("LruCache: capacity must be >= 1");
  if (num_layers < 1) throw InputError("expand: num_layers must be >= 1");
  // the fixed training order (cache.cpp:155-162)
  std::vector<VertexId> order(n);
  check(cb_shuffled_order(n, seed, order.data()));
  const std::uint64_t per_epoch = std::max<std::uint64_t>(1, n / b);

  DependentExperimentResult res;
  res.steps_per_epoch = per_epoch;
  res.warmup_steps = std::min(per_epoch, steps / 2);
  res.rows.reserve(steps);

  const bool nested = schedule.mode == BatchMode::kNested;
  SeedSchedule sched = SeedSchedule::make(nested ? 1 : schedule.kappa, seed);
  cb_plan* pl = plan_for({&g, nullptr, 1, num_layers, &cfg, b});
  DeviceCache dc(n, cache_capacity);
  std::uint64_t steady_hits = 0, steady_misses = 0;
  const std::uint64_t off[2] = {0, b};
  for (std::uint64_t step = 0; step < steps; ++step) {
    const VertexId* batch = order.data() + (step % per_epoch) * b;
    cb_sched cs;
    if (nested) {  // groups of kappa steps share one epoch seed
      const std::uint64_t group = schedule.kappa == kKappaInfinity ? 0 : step / schedule.kappa;
      const std::uint64_t z = hash_bits(seed, {kStreamFresh, group});
      cs = {1, z, z, 0};
    } else {
      cs = to_sched(sched);
      sched = schedule_advance(sched);
    }
    check(cb_sample_sync(pl, CB_MODE_INDEP, batch, off, &cs));
    DependentStepRow row;
    row.step = step;
    row.fingerprint = fingerprint(pl);
    std::uint64_t h0 = 0, m0 = 0, h1 = 0, m1 = 0, kept = 0;
    dc.stats(h0, m0);
    // access_order(inputs, hash_bits(seed, {step, 0xACCE55})), cache.cpp:187-188
    check(cb_cache_access_plan(dc.h, pl, 0, hash_bits(seed, {step, 0xACCE55}), nullptr, 0,
                               nullptr, nullptr, &kept));
    dc.stats(h1, m1);
    const std::uint64_t miss = m1 - m0;
    row.s_l = kept;
    row.miss_rate = kept == 0 ? 0.0 : static_cast<double>(miss) / static_cast<double>(kept);
    row.bytes = miss * static_cast<std::uint64_t>(feature_dim) * bytes_per_scalar;
    if (step >= res.warmup_steps) {
      steady_misses += miss;
      steady_hits += kept - miss;
    }
    res.rows.push_back(row);
  }
  const std::uint64_t total = steady_hits + steady_misses;
  res.steady_miss_rate =
      total == 0 ? 0.0 : static_cast<double>(steady_misses) / static_cast<double>(total);
  return res;
}

}  // namespace coopbatch
