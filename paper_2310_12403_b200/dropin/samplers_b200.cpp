// Drop-in replacement of the reference's src/samplers.cpp: the functions
// declared in include/coopbatch/samplers.hpp (unchanged), run by the sm_100a
// kernels of libcoopbatch_b200.so through its C-ABI.
//
//   sample_full    samplers.cpp:289-296   -> FULL plan, 1 layer
//   sample_ns      samplers.cpp:298-303   -> NS plan under VariateSource::plain
//   sample_labor0  samplers.cpp:305-312   -> LABOR plan with a caller variate table
//   sample_rw      samplers.cpp:314-321   -> RW plan under VariateSource::plain
//   sample_block   samplers.cpp:323-338   -> 1-layer plan, block hashed as `layer`,
//                                            variates from the given source
//   expand         samplers.cpp:340-354   -> L-layer plan, one batch
//   edge_pred_seeds samplers.cpp:356-393  -> host (seed generation, like the
//                                            reference's seed draws)
// Seeds are checked on the host first with Graph::check_vertex, so the
// exceptions (type and text) are the reference's own.
#include <unordered_set>

#include "ctx.hpp"

namespace coopbatch {

namespace {

using namespace b200;

void check_seeds(const Graph& g, std::span<const VertexId> seeds) {
  for (const VertexId s : seeds) g.check_vertex(s);
}

// One block of `cfg.kind` at layer `layer` with variates from `v` (nullptr:
// the plan's default plain stream; FULL draws nothing).
BipartiteBlock one_block(const Graph& g, std::span<const VertexId> seeds, const SamplerConfig& cfg,
                         const VariateSource* v, int layer) {
  if (layer < 0) throw InputError("sample_block: layer must be >= 0");
  cb_plan* pl = plan_for({&g, nullptr, 1, 1, &cfg, seeds.size()});
  check(cb_plan_set_layer_base(pl, layer));
  cb_sched sched{1, 0, 0, 0};
  if (v) {
    const cb_variates cv = to_variates(*v);
    check(cb_plan_set_variate_source(pl, &cv));
  }
  const std::uint64_t off[2] = {0, seeds.size()};
  check(cb_sample_sync(pl, CB_MODE_INDEP, seeds.data(), off, &sched));
  return download_block(pl, 0, 0, layer);
}

}  // namespace

BipartiteBlock sample_full(const Graph& g, std::span<const VertexId> seeds, int layer) {
  Lock lk(api_mutex());
  check_seeds(g, seeds);
  SamplerConfig cfg;
  cfg.kind = SamplerKind::kFull;
  return one_block(g, seeds, cfg, nullptr, layer);
}

BipartiteBlock sample_ns(const Graph& g, std::span<const VertexId> seeds, std::uint32_t k,
                         std::uint64_t epoch_seed, int layer) {
  Lock lk(api_mutex());
  check_seeds(g, seeds);
  if (k == 0) throw InputError("sample_ns: fanout must be >= 1");
  SamplerConfig cfg;
  cfg.kind = SamplerKind::kNs;
  cfg.fanout = k;
  const VariateSource v = VariateSource::plain(epoch_seed);
  return one_block(g, seeds, cfg, &v, layer);
}

BipartiteBlock sample_labor0(const Graph& g, std::span<const VertexId> seeds, std::uint32_t k,
                             const std::function<double(VertexId)>& variate, int layer) {
  Lock lk(api_mutex());
  check_seeds(g, seeds);
  if (k == 0) throw InputError("sample_labor0: fanout must be >= 1");
  // The caller's variate is host code: evaluate it once per distinct
  // neighbour of the seeds (the only vertices the rule reads) into a table
  // the kernels compare against k / d_s, samplers.cpp:89-104.
  std::vector<double> table(g.num_vertices, 0.0);
  std::vector<std::uint8_t> seen(g.num_vertices, 0);
  for (const VertexId s : seeds)
    for (const VertexId t : g.neighbors(s))
      if (!seen[t]) {
        seen[t] = 1;
        table[t] = variate(t);
      }
  SamplerConfig cfg;
  cfg.kind = SamplerKind::kLabor0;
  cfg.fanout = k;
  cb_plan* pl = plan_for({&g, nullptr, 1, 1, &cfg, seeds.size()});
  check(cb_plan_set_variate_table(pl, table.data(), 0));
  const cb_sched sched{1, 0, 0, 0};
  const std::uint64_t off[2] = {0, seeds.size()};
  check(cb_sample_sync(pl, CB_MODE_INDEP, seeds.data(), off, &sched));
  BipartiteBlock b = download_block(pl, 0, 0, layer);
  check(cb_plan_set_variate_table(pl, nullptr, 0));
  return b;
}

BipartiteBlock sample_rw(const Graph& g, std::span<const VertexId> seeds, const SamplerConfig& cfg,
                         std::uint64_t epoch_seed, int layer) {
  Lock lk(api_mutex());
  check_seeds(g, seeds);
  if (cfg.rw_length < 1 || cfg.rw_walks < 1)
    throw InputError("sample_rw: rw_length and rw_walks must be >= 1");
  SamplerConfig c = cfg;
  c.kind = SamplerKind::kRw;
  const VariateSource v = VariateSource::plain(epoch_seed);
  return one_block(g, seeds, c, &v, layer);
}

BipartiteBlock sample_block(const Graph& g, std::span<const VertexId> seeds,
                            const SamplerConfig& cfg, const VariateSource& source, int layer) {
  Lock lk(api_mutex());
  check_seeds(g, seeds);
  switch (cfg.kind) {
    case SamplerKind::kFull:
      return one_block(g, seeds, cfg, nullptr, layer);
    case SamplerKind::kNs:
    case SamplerKind::kLabor0:
    case SamplerKind::kRw:
      return one_block(g, seeds, cfg, &source, layer);
  }
  throw InputError("sample_block: unknown sampler kind");
}

LayerStack expand(const Graph& g, std::span<const VertexId> seeds, int num_layers,
                  const SamplerConfig& cfg, const SeedSchedule& schedule) {
  Lock lk(api_mutex());
  if (num_layers < 1) throw InputError("expand: num_layers must be >= 1");
  check_seeds(g, seeds);
  cb_plan* pl = plan_for({&g, nullptr, 1, num_layers, &cfg, seeds.size()});
  const cb_sched s = to_sched(schedule);
  const std::uint64_t off[2] = {0, seeds.size()};
  check(cb_sample_sync(pl, CB_MODE_INDEP, seeds.data(), off, &s));
  LayerStack stack;
  stack.blocks.reserve(num_layers);
  for (int l = 0; l < num_layers; ++l) stack.blocks.push_back(download_block(pl, 0, l, l));
  return stack;
}

// Positive edges plus one negative edge each; the union of endpoints in
// first-seen order (samplers.cpp:356-393). Host code: it draws seeds, like
// the reference's seed draws, and touches one neighbour list per edge.
std::vector<VertexId> edge_pred_seeds(const Graph& g,
                                      std::span<const std::pair<VertexId, VertexId>> edge_batch,
                                      std::uint64_t epoch_seed) {
  std::vector<VertexId> order;
  std::unordered_set<VertexId> in_order;
  const auto emit = [&](VertexId v) {
    if (in_order.insert(v).second) order.push_back(v);
  };
  for (const auto& [a, b] : edge_batch) {
    g.check_vertex(a);
    g.check_vertex(b);
    emit(a);
    emit(b);
    // endpoint kept by the negative edge, and the vertices it may not pair with
    const VertexId keep = hash_uniform(epoch_seed, {kStreamEdgeCoin, a, b}) < 0.5 ? a : b;
    const auto nbrs = g.neighbors(keep);
    const auto excluded = [&](VertexId w) {
      if (w == keep) return true;
      for (const VertexId t : nbrs)
        if (t == w) return true;
      return false;
    };
    bool placed = false;
    for (std::uint64_t attempt = 0; attempt < 100 && !placed; ++attempt) {
      const double u = hash_uniform(epoch_seed, {kStreamEdgeNeg, a, b, attempt});
      const auto w = static_cast<VertexId>(
          std::min<std::uint64_t>(static_cast<std::uint64_t>(u * static_cast<double>(g.num_vertices)),
                                  g.num_vertices - 1));
      if (excluded(w)) continue;
      emit(w);
      placed = true;
    }
    if (!placed)
      throw InputError("edge_pred_seeds: no negative endpoint found for vertex " +
                       std::to_string(keep) + " after 100 attempts");
  }
  return order;
}

}  // namespace coopbatch
