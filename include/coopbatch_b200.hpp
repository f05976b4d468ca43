// coopbatch_b200.hpp — header-only C++17 drop-in for the reference's sampler /
// minibatch API (/root/reference/proj/include/coopbatch/{graph,rng,samplers,
// partition,coop}.hpp) over the C-ABI of libcoopbatch_b200.so.
//
// Same names, argument meaning, value-type results and exception behaviour
// (InputError for contract violations, common.hpp:12-15); the work runs in
// the sm_100a kernels. Link with -lcoopbatch_b200 (paper_2310_12403_b200/).
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "coopbatch_cuda.h"

namespace coopbatch_b200 {

using VertexId = std::uint32_t;

struct InputError : std::invalid_argument {  // common.hpp:12-15
  using std::invalid_argument::invalid_argument;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == CB_OK) return;
  const std::string msg = cb_last_error();
  if (rc == CB_INPUT) throw InputError(msg);
  throw DeviceError(msg);
}

enum class SamplerKind { kFull = CB_FULL, kNs = CB_NS, kLabor0 = CB_LABOR0, kRw = CB_RW };

struct SamplerConfig {  // samplers.hpp:17-23 (+ per-layer fanouts extension)
  SamplerKind kind = SamplerKind::kNs;
  std::uint32_t fanout = 10;
  std::vector<std::uint32_t> fanouts;  // empty -> fanout at every layer
  std::uint32_t rw_length = 3;  // o
  double rw_restart = 0.5;      // p
  std::uint32_t rw_walks = 100; // a

  std::vector<std::uint32_t> per_layer(int L) const {
    if (!fanouts.empty()) {
      if (static_cast<int>(fanouts.size()) != L)
        throw InputError("fanouts must list one fanout per layer");
      return fanouts;
    }
    return std::vector<std::uint32_t>(L, fanout);
  }
};

inline constexpr std::uint64_t kKappaInfinity = std::numeric_limits<std::uint64_t>::max();

struct SeedSchedule {  // rng.hpp:93-111 (value type; make/advance as rng.cpp:69-86)
  std::uint64_t kappa = 1, z1 = 0, z2 = 0, iteration = 0;
  cb_sched c() const { return {kappa, z1, z2, iteration}; }
};

struct BipartiteBlock {  // samplers.hpp:30-38
  std::vector<VertexId> dst_vertices;
  std::vector<VertexId> src_vertices;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;
  std::vector<std::uint32_t> dst_pos_in_src;
  int layer = 0;
  std::uint64_t num_edges() const { return edges.size(); }
};

struct LayerStack {  // samplers.hpp:42-49
  std::vector<BipartiteBlock> blocks;
  const std::vector<VertexId>& input_vertices() const { return blocks.back().src_vertices; }
};

struct RemoteRef {  // coop.hpp:14-17
  std::uint32_t part = 0;
  std::uint64_t row = 0;
};

struct ExchangeRecord {  // coop.hpp:25-37
  int layer = 0;
  std::vector<std::vector<std::uint64_t>> send_counts;
  std::vector<std::vector<RemoteRef>> src_location;
  std::vector<std::uint64_t> owner_row_counts;
  std::uint32_t num_parts() const { return static_cast<std::uint32_t>(send_counts.size()); }
  std::uint64_t communicated(std::uint32_t p) const {
    std::uint64_t t = 0;
    for (std::uint32_t q = 0; q < num_parts(); ++q)
      if (q != p) t += send_counts[p][q];
    return t;
  }
};

struct CoopSampleResult {  // coop.hpp:39-43
  std::vector<LayerStack> stacks;
  std::vector<ExchangeRecord> exchanges;
  std::vector<std::vector<VertexId>> owner_sets;
};

// ---- device handles ---------------------------------------------------------
class Graph {  // graph.hpp:21-53, resident in HBM
 public:
  static Graph from_csr(const std::vector<std::uint64_t>& indptr,
                        const std::vector<VertexId>& indices, int device = 0) {
    cb_graph* g = nullptr;
    check(cb_graph_create_from_csr(indptr.data(), indices.data(), indptr.size() - 1,
                                   indices.size(), device, &g));
    return Graph(g);
  }
  static Graph generate_rmat(std::uint64_t n, std::uint64_t m, std::uint64_t seed,
                             int device = 0) {
    cb_graph* g = nullptr;
    check(cb_graph_generate_rmat(n, m, seed, device, &g));
    return Graph(g);
  }
  // load_csr / save_csr (graph.cpp:216-252): CBCS straight into / out of HBM
  static Graph load_csr(const std::string& path, int device = 0) {
    cb_graph* g = nullptr;
    check(cb_graph_load_cbcs(path.c_str(), device, &g));
    return Graph(g);
  }
  void save_csr(const std::string& path) const { check(cb_graph_save_cbcs(h_.get(), path.c_str())); }
  std::uint64_t num_vertices() const {
    std::uint64_t n = 0;
    check(cb_graph_info(h_.get(), &n, nullptr, nullptr));
    return n;
  }
  cb_graph* get() const { return h_.get(); }

 private:
  explicit Graph(cb_graph* g) : h_(g, cb_graph_destroy) {}
  std::shared_ptr<cb_graph> h_;
};

class PartitionMap {  // partition.hpp:12-17
 public:
  static PartitionMap random(const Graph& g, std::uint32_t parts, std::uint64_t seed) {
    cb_partition* p = nullptr;
    check(cb_partition_random(g.get(), parts, seed, &p));
    return PartitionMap(p, parts);
  }
  static PartitionMap from_owner(const Graph& g, const std::vector<std::uint32_t>& owner,
                                 std::uint32_t parts) {
    if (owner.size() != g.num_vertices())
      throw InputError("partition: owner array does not cover all vertices");
    cb_partition* p = nullptr;
    check(cb_partition_create(g.get(), owner.data(), parts, &p));
    return PartitionMap(p, parts);
  }
  std::uint32_t num_parts() const { return parts_; }
  cb_partition* get() const { return h_.get(); }

 private:
  PartitionMap(cb_partition* p, std::uint32_t parts) : h_(p, cb_partition_destroy), parts_(parts) {}
  std::shared_ptr<cb_partition> h_;
  std::uint32_t parts_;
};

namespace detail {

inline BipartiteBlock download_block(cb_plan* pl, std::uint32_t p, int l) {
  std::uint64_t sz[6];
  check(cb_layer_sizes(pl, p, l, sz));
  BipartiteBlock b;
  b.layer = l;
  b.dst_vertices.resize(sz[0]);
  b.src_vertices.resize(sz[1]);
  std::vector<std::uint32_t> e(2 * sz[2]);
  b.dst_pos_in_src.resize(sz[0]);
  check(cb_download_block(pl, p, l, b.dst_vertices.data(), b.src_vertices.data(), e.data(),
                          b.dst_pos_in_src.data()));
  b.edges.resize(sz[2]);
  for (std::uint64_t i = 0; i < sz[2]; ++i) b.edges[i] = {e[2 * i], e[2 * i + 1]};
  return b;
}

struct PlanDeleter {
  void operator()(cb_plan* p) const { cb_plan_destroy(p); }
};
using PlanPtr = std::unique_ptr<cb_plan, PlanDeleter>;

inline PlanPtr make_plan(const Graph& g, const PartitionMap* pm, int L, const SamplerConfig& cfg,
                         std::uint64_t max_seeds) {
  if (L < 1) throw InputError("expand: num_layers must be >= 1");
  const auto fo = cfg.per_layer(L);
  cb_plan* pl = nullptr;
  check(cb_plan_create(g.get(), pm ? pm->get() : nullptr, L, static_cast<int>(cfg.kind),
                       fo.data(), max_seeds ? max_seeds : 1, &pl));
  PlanPtr plan(pl);
  if (cfg.kind == SamplerKind::kRw)
    check(cb_plan_set_rw(pl, cfg.rw_length, cfg.rw_restart, cfg.rw_walks));
  return plan;
}

}  // namespace detail

// samplers.cpp:340-354
inline LayerStack expand(const Graph& g, const std::vector<VertexId>& seeds, int num_layers,
                         const SamplerConfig& cfg, const SeedSchedule& schedule) {
  auto pl = detail::make_plan(g, nullptr, num_layers, cfg, seeds.size());
  const std::uint64_t off[2] = {0, seeds.size()};
  const cb_sched s = schedule.c();
  check(cb_sample_sync(pl.get(), CB_MODE_INDEP, seeds.data(), off, &s));
  LayerStack st;
  for (int l = 0; l < num_layers; ++l) st.blocks.push_back(detail::download_block(pl.get(), 0, l));
  return st;
}

// samplers.cpp:323-338: one block of any sampler at layer `layer` (the layer
// namespaces the variates), on a 1-layer plan whose block hashes as `layer`
inline BipartiteBlock sample_block(const Graph& g, const std::vector<VertexId>& seeds,
                                   const SamplerConfig& cfg, const SeedSchedule& schedule,
                                   int layer) {
  if (layer < 0) throw InputError("sample_block: layer must be >= 0");
  auto pl = detail::make_plan(g, nullptr, 1, cfg, seeds.size());
  check(cb_plan_set_layer_base(pl.get(), layer));
  const std::uint64_t off[2] = {0, seeds.size()};
  const cb_sched s = schedule.c();
  check(cb_sample_sync(pl.get(), CB_MODE_INDEP, seeds.data(), off, &s));
  BipartiteBlock b = detail::download_block(pl.get(), 0, 0);
  b.layer = layer;
  return b;
}

// samplers.cpp:89-104, 305-312: LABOR-0 with the caller's variate r(t), keep
// t -> s iff r(t) <= k / d_s. r is evaluated once per vertex on the host and
// the block is sampled on the GPU from that table.
inline BipartiteBlock sample_labor0(const Graph& g, const std::vector<VertexId>& seeds,
                                    std::uint32_t k,
                                    const std::function<double(VertexId)>& variate,
                                    int layer = 0) {
  if (k == 0) throw InputError("sample_labor0: fanout must be >= 1");
  std::vector<double> table(g.num_vertices());
  for (std::uint64_t t = 0; t < table.size(); ++t) table[t] = variate(static_cast<VertexId>(t));
  SamplerConfig cfg;
  cfg.kind = SamplerKind::kLabor0;
  cfg.fanout = k;
  auto pl = detail::make_plan(g, nullptr, 1, cfg, seeds.size());
  check(cb_plan_set_variate_table(pl.get(), table.data(), 0));
  const std::uint64_t off[2] = {0, seeds.size()};
  const cb_sched s{1, 0, 0, 0};
  check(cb_sample_sync(pl.get(), CB_MODE_INDEP, seeds.data(), off, &s));
  BipartiteBlock b = detail::download_block(pl.get(), 0, 0);
  b.layer = layer;
  return b;
}

// coop.cpp:108-119
inline std::vector<LayerStack> indep_sample(const Graph& g,
                                            const std::vector<std::vector<VertexId>>& per_pe,
                                            int num_layers, const SamplerConfig& cfg,
                                            const SeedSchedule& schedule) {
  std::vector<LayerStack> out;
  for (const auto& s : per_pe) out.push_back(expand(g, s, num_layers, cfg, schedule));
  return out;
}

// coop.cpp:68-106
inline CoopSampleResult coop_sample(const Graph& g, const PartitionMap& pm,
                                    const std::vector<std::vector<VertexId>>& per_pe,
                                    int num_layers, const SamplerConfig& cfg,
                                    const SeedSchedule& schedule) {
  const std::uint32_t P = pm.num_parts();
  if (per_pe.size() != P)
    throw InputError("coop_sample: seed lists must match the partition count");
  std::uint64_t maxb = 1;
  std::vector<VertexId> flat;
  std::vector<std::uint64_t> off{0};
  for (const auto& s : per_pe) {
    flat.insert(flat.end(), s.begin(), s.end());
    off.push_back(flat.size());
    maxb = std::max<std::uint64_t>(maxb, s.size());
  }
  auto pl = detail::make_plan(g, &pm, num_layers, cfg, maxb);
  const cb_sched s = schedule.c();
  check(cb_sample_sync(pl.get(), CB_MODE_COOP, flat.data(), off.data(), &s));
  CoopSampleResult r;
  r.stacks.resize(P);
  for (std::uint32_t p = 0; p < P; ++p)
    for (int l = 0; l < num_layers; ++l)
      r.stacks[p].blocks.push_back(detail::download_block(pl.get(), p, l));
  for (int l = 0; l < num_layers; ++l) {
    ExchangeRecord e;
    e.layer = l;
    std::vector<std::uint64_t> sc(P * P), orc(P);
    std::uint64_t tot = 0;
    for (std::uint32_t p = 0; p < P; ++p) tot += r.stacks[p].blocks[l].src_vertices.size();
    std::vector<std::uint32_t> lp(tot);
    std::vector<std::uint64_t> lr(tot);
    check(cb_download_exchange(pl.get(), l, sc.data(), orc.data(), lp.data(), lr.data()));
    e.send_counts.assign(P, std::vector<std::uint64_t>(P));
    for (std::uint32_t p = 0; p < P; ++p)
      for (std::uint32_t q = 0; q < P; ++q) e.send_counts[p][q] = sc[p * P + q];
    e.owner_row_counts = orc;
    std::uint64_t o = 0;
    e.src_location.resize(P);
    for (std::uint32_t p = 0; p < P; ++p)
      for (std::size_t j = 0; j < r.stacks[p].blocks[l].src_vertices.size(); ++j, ++o)
        e.src_location[p].push_back({lp[o], lr[o]});
    r.exchanges.push_back(std::move(e));
  }
  r.owner_sets.resize(P);
  for (std::uint32_t p = 0; p < P; ++p) {
    std::uint64_t n = 0;
    check(cb_owner_set_size(pl.get(), p, &n));
    r.owner_sets[p].resize(n);
    if (n) check(cb_download_owner_set(pl.get(), p, r.owner_sets[p].data()));
  }
  return r;
}

// ---- features, cache, training step ----------------------------------------
enum class Dtype { kF64 = CB_F64, kF32 = CB_F32, kF16 = CB_F16 };

class FeatureStore {  // coop.hpp:140-155, synthetic rows in HBM (sharded by pm)
 public:
  static FeatureStore synth(const Graph& g, std::uint32_t dim, std::uint64_t seed,
                            Dtype dtype = Dtype::kF64, const PartitionMap* pm = nullptr) {
    cb_features* f = nullptr;
    check(cb_features_synth(g.get(), pm ? pm->get() : nullptr, dim, static_cast<int>(dtype), seed,
                            &f));
    return FeatureStore(f);
  }
  cb_features* get() const { return h_.get(); }

 private:
  explicit FeatureStore(cb_features* f) : h_(f, cb_features_destroy) {}
  std::shared_ptr<cb_features> h_;
};

enum class CacheOutcome { kHit, kMiss };

class LruCache {  // cache.hpp:17-42 (exact LRU, evaluated on the device)
 public:
  LruCache(std::uint64_t capacity, std::uint64_t n_keys, int device = 0) {
    if (capacity == 0) throw InputError("LruCache: capacity must be >= 1");
    cb_cache* c = nullptr;
    check(cb_cache_create(device, n_keys, capacity, 0, &c));
    h_.reset(c, cb_cache_destroy);
  }
  CacheOutcome access(VertexId key) {
    std::uint8_t miss = 0;
    check(cb_cache_access_trace(h_.get(), &key, 1, &miss));
    return miss ? CacheOutcome::kMiss : CacheOutcome::kHit;
  }
  // LruCache::access over a whole trace, in order (one device batch per run
  // of distinct keys)
  std::vector<CacheOutcome> access_all(const std::vector<VertexId>& keys) {
    std::vector<std::uint8_t> miss(keys.size());
    check(cb_cache_access_trace(h_.get(), keys.data(), keys.size(), miss.data()));
    std::vector<CacheOutcome> out(keys.size());
    for (std::size_t i = 0; i < keys.size(); ++i)
      out[i] = miss[i] ? CacheOutcome::kMiss : CacheOutcome::kHit;
    return out;
  }
  std::uint64_t hits() const { return stat(0); }
  std::uint64_t misses() const { return stat(1); }
  std::uint64_t size() const { return stat(2); }
  std::vector<VertexId> resident() const {
    std::uint64_t n = 0;
    check(cb_cache_resident(h_.get(), nullptr, 0, &n));
    std::vector<VertexId> out(n);
    check(cb_cache_resident(h_.get(), out.data(), n, &n));
    return out;
  }

 private:
  std::uint64_t stat(int i) const {
    std::uint64_t v[3];
    check(cb_cache_stats(h_.get(), &v[0], &v[1], &v[2]));
    return v[i];
  }
  std::shared_ptr<cb_cache> h_;
};

class GcnModel {  // coop.hpp:126-135
 public:
  static GcnModel init(std::uint32_t in_dim, std::uint32_t hidden, std::uint32_t num_classes,
                       int num_layers, std::uint64_t seed, int device = 0) {
    cb_model* m = nullptr;
    check(cb_gcn_model_init(device, in_dim, hidden, num_classes, num_layers, seed, &m));
    return GcnModel(m, num_layers, num_classes);
  }
  int num_layers() const { return L_; }
  std::uint32_t num_classes() const { return C_; }
  cb_model* get() const { return h_.get(); }

 private:
  GcnModel(cb_model* m, int L, std::uint32_t C) : h_(m, cb_gcn_model_destroy), L_(L), C_(C) {}
  std::shared_ptr<cb_model> h_;
  int L_;
  std::uint32_t C_;
};

struct DenseMatrix {  // coop.hpp:95-103 (row-major)
  std::uint64_t rows = 0, cols = 0;
  std::vector<double> data;
};

struct TrainStepResult {  // coop.hpp:175-179 (metrics: see the Python mirror)
  double loss = 0.0;
  std::vector<DenseMatrix> grad_w;
};

namespace detail {
inline TrainStepResult train(cb_plan* pl, const FeatureStore& store, const GcnModel& model) {
  TrainStepResult r;
  std::uint64_t total = 0;
  for (int l = 0; l < model.num_layers(); ++l) {
    DenseMatrix d;
    check(cb_gcn_model_weights(model.get(), l, nullptr, 0, &d.rows, &d.cols));
    total += d.rows * d.cols;
    r.grad_w.push_back(d);
  }
  std::vector<double> gw(total);
  check(cb_train_step(pl, store.get(), model.num_classes(), model.get(), &r.loss, gw.data()));
  std::uint64_t o = 0;
  for (auto& d : r.grad_w) {
    d.data.assign(gw.begin() + o, gw.begin() + o + d.rows * d.cols);
    o += d.rows * d.cols;
  }
  return r;
}
}  // namespace detail

// coop.cpp:438-556 (store: f64, sharded by pm)
inline TrainStepResult coop_train_step(const Graph& g, const PartitionMap& pm,
                                       const std::vector<std::vector<VertexId>>& per_pe,
                                       int num_layers, const SamplerConfig& cfg,
                                       const SeedSchedule& schedule, const GcnModel& model,
                                       const FeatureStore& store) {
  if (per_pe.size() != pm.num_parts())
    throw InputError("coop_sample: seed lists must match the partition count");
  std::uint64_t maxb = 1;
  std::vector<VertexId> flat;
  std::vector<std::uint64_t> off{0};
  for (const auto& s : per_pe) {
    flat.insert(flat.end(), s.begin(), s.end());
    off.push_back(flat.size());
    maxb = std::max<std::uint64_t>(maxb, s.size());
  }
  auto pl = detail::make_plan(g, &pm, num_layers, cfg, maxb);
  const cb_sched s = schedule.c();
  check(cb_sample_sync(pl.get(), CB_MODE_COOP, flat.data(), off.data(), &s));
  return detail::train(pl.get(), store, model);
}

// coop.cpp:560-610, one part (P = 1) per call of the reference's parts loop
inline TrainStepResult indep_train_step(const Graph& g, const std::vector<VertexId>& seeds,
                                        int num_layers, const SamplerConfig& cfg,
                                        const SeedSchedule& schedule, const GcnModel& model,
                                        const FeatureStore& store) {
  auto pl = detail::make_plan(g, nullptr, num_layers, cfg, seeds.size());
  const std::uint64_t off[2] = {0, seeds.size()};
  const cb_sched s = schedule.c();
  check(cb_sample_sync(pl.get(), CB_MODE_INDEP, seeds.data(), off, &s));
  return detail::train(pl.get(), store, model);
}

}  // namespace coopbatch_b200
