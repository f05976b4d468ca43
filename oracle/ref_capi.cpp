// TEST INFRASTRUCTURE ONLY — never the product path.
//
// extern "C" shim over the reference's OWN C++ sources (/root/reference/proj,
// compiled unmodified by oracle/Makefile into oracle/_ref/libcoopbatch_ref.so).
// It converts the reference's std::vector value types into the plain-C
// ob_types.h layouts so tests and bench.py's reference arm can call the real
// reference through ctypes. Used (1) to pin the plain-C restatement
// (coopbatch_oracle.c), (2) to generate tests/golden/, and (3) as the CPU
// baseline ("kind": "reference") in bench.py.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <span>
#include <string>
#include <vector>

#include "coopbatch/analysis.hpp"
#include "coopbatch/cache.hpp"
#include "coopbatch/coop.hpp"
#include "coopbatch/graph.hpp"
#include "coopbatch/parallel.hpp"
#include "coopbatch/partition.hpp"
#include "coopbatch/rng.hpp"
#include "coopbatch/samplers.hpp"
#include "ob_types.h"

using namespace coopbatch;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InputError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 1));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

void to_block(const BipartiteBlock& b, ob_block* o) {
  o->layer = b.layer;
  o->n_dst = b.dst_vertices.size();
  o->n_src = b.src_vertices.size();
  o->n_edges = b.edges.size();
  o->dst = dup(b.dst_vertices);
  o->src = dup(b.src_vertices);
  o->dst_pos = dup(b.dst_pos_in_src);
  o->edges = static_cast<uint32_t*>(std::malloc(2 * b.edges.size() * sizeof(uint32_t) + 1));
  for (std::size_t e = 0; e < b.edges.size(); ++e) {
    o->edges[2 * e] = b.edges[e].first;
    o->edges[2 * e + 1] = b.edges[e].second;
  }
}

void to_stack(const LayerStack& s, ob_stack* o) {
  o->num_layers = static_cast<int32_t>(s.blocks.size());
  o->blocks = static_cast<ob_block*>(std::calloc(s.blocks.size() + 1, sizeof(ob_block)));
  for (std::size_t l = 0; l < s.blocks.size(); ++l) to_block(s.blocks[l], &o->blocks[l]);
}

SeedSchedule to_sched(const ob_sched* s) {
  SeedSchedule r;
  r.kappa = s->kappa;
  r.z1 = s->z1;
  r.z2 = s->z2;
  r.iteration = s->iteration;
  return r;
}

SamplerConfig to_cfg(int kind, uint32_t fanout) {
  SamplerConfig c;
  c.kind = static_cast<SamplerKind>(kind);
  c.fanout = fanout;
  return c;
}

}  // namespace

extern "C" {

const char* rf_last_error(void) { return g_err.c_str(); }

uint64_t rf_mix64(uint64_t x) { return mix64(x); }
uint64_t rf_hash_bits(uint64_t seed, const uint64_t* ids, int n) {
  uint64_t h = hash_init(seed);
  for (int i = 0; i < n; ++i) h = hash_step(h, ids[i]);
  return h;
}
double rf_phi(double x) { return phi(x); }
double rf_inverse_phi(double p) { return inverse_phi(p); }
double rf_normal_from_bits(uint64_t b) { return normal_from_bits(b); }

void rf_sched_make(uint64_t kappa, uint64_t root, ob_sched* out) {
  const SeedSchedule s = SeedSchedule::make(kappa, root);
  out->kappa = s.kappa;
  out->z1 = s.z1;
  out->z2 = s.z2;
  out->iteration = s.iteration;
}
void rf_sched_advance(ob_sched* io) {
  const SeedSchedule s = schedule_advance(to_sched(io));
  io->kappa = s.kappa;
  io->z1 = s.z1;
  io->z2 = s.z2;
  io->iteration = s.iteration;
}

/* Variate exactly as labor_block_stream draws it (samplers.cpp:112-129). */
double rf_labor_variate(const ob_sched* sched, int layer, uint32_t t) {
  const VariateSource src = VariateSource::from_schedule(to_sched(sched));
  const VariatePrefix p =
      src.prefix({kStreamLabor, static_cast<std::uint64_t>(layer)});
  return src.uniform_tail1(p, t);
}

void* rf_graph_new(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                   uint64_t m) {
  auto* g = new Graph();
  g->num_vertices = n;
  g->indptr.assign(indptr, indptr + n + 1);
  g->indices.assign(indices, indices + m);
  return g;
}
void rf_graph_free(void* g) { delete static_cast<Graph*>(g); }
void rf_graph_set_weights(void* g, const float* w, uint64_t m) {
  static_cast<Graph*>(g)->weights.assign(w, w + m);
}

/* coop_train_step / indep_train_step (coop.cpp:438-610) with GcnModel::init
 * (in_dim = store dim); grad_w: layers concatenated, each rows x cols. */
int rf_train_step(void* g, void* fs, int mode, const uint32_t* owner, uint32_t parts,
                  const uint32_t* seeds_flat, const uint64_t* seeds_off, int L, int kind,
                  uint32_t fanout, const ob_sched* sched, uint32_t hidden, uint64_t model_seed,
                  double* loss, double* grad_w) {
  return guard([&] {
    const Graph& gr = *static_cast<Graph*>(g);
    const FeatureStore& store = *static_cast<FeatureStore*>(fs);
    std::vector<std::vector<VertexId>> seeds(parts);
    for (uint32_t p = 0; p < parts; ++p)
      seeds[p].assign(seeds_flat + seeds_off[p], seeds_flat + seeds_off[p + 1]);
    const GcnModel model = GcnModel::init(store.dim, hidden, store.num_classes, L, model_seed);
    TrainStepResult r;
    if (mode == 0) {
      PartitionMap pm;
      pm.num_parts = parts;
      pm.owner.assign(owner, owner + gr.num_vertices);
      r = coop_train_step(gr, pm, seeds, L, to_cfg(kind, fanout), to_sched(sched), model, store);
    } else {
      r = indep_train_step(gr, seeds, L, to_cfg(kind, fanout), to_sched(sched), model, store);
    }
    *loss = r.loss;
    std::size_t off = 0;
    for (const auto& w : r.grad_w) {
      std::memcpy(grad_w + off, w.data.data(), w.data.size() * sizeof(double));
      off += w.data.size();
    }
  });
}

/* partition.cpp:79-89 */
int rf_cross_edge_ratio(void* g, const uint32_t* owner, uint32_t parts, double* out) {
  return guard([&] {
    const Graph& gr = *static_cast<Graph*>(g);
    PartitionMap pm;
    pm.num_parts = parts;
    pm.owner.assign(owner, owner + gr.num_vertices);
    *out = cross_edge_ratio(gr, pm);
  });
}

/* samplers.cpp:356-393 edge_pred_seeds; out needs 3 * n_edges slots. */
int rf_edge_pred_seeds(void* g, const uint32_t* uv, uint64_t n_edges, uint64_t epoch_seed,
                       uint32_t* out, uint64_t* n_out) {
  return guard([&] {
    std::vector<std::pair<VertexId, VertexId>> batch(n_edges);
    for (uint64_t i = 0; i < n_edges; ++i) batch[i] = {uv[2 * i], uv[2 * i + 1]};
    const auto s = edge_pred_seeds(*static_cast<Graph*>(g), batch, epoch_seed);
    std::memcpy(out, s.data(), s.size() * 4);
    *n_out = s.size();
  });
}

/* analysis.cpp:78-124 work_curve; out[4 * i ..] = mean_sl, se_sl,
 * work_per_seed, se_work of batch size i. edge_mode selects SeedMode::kEdge. */
int rf_work_curve(void* g, int kind, uint32_t fanout, const uint64_t* sizes, uint64_t n_sizes,
                  uint32_t trials, int L, uint64_t seed, int edge_mode, double* out) {
  return guard([&] {
    const WorkCurve c = work_curve(*static_cast<Graph*>(g), to_cfg(kind, fanout),
                                   {sizes, n_sizes}, trials, L, seed,
                                   edge_mode ? SeedMode::kEdge : SeedMode::kNode);
    for (uint64_t i = 0; i < n_sizes; ++i) {
      out[4 * i] = c.points[i].mean_sl;
      out[4 * i + 1] = c.points[i].se_sl;
      out[4 * i + 2] = c.points[i].work_per_seed;
      out[4 * i + 3] = c.points[i].se_work;
    }
  });
}

/* analysis.cpp:126-151 concavity_check over (batch, mean, se) points;
 * entry i-1 of the outputs belongs to interior point i. */
int rf_concavity_check(const uint64_t* sizes, const double* mean, const double* se, uint64_t n,
                       double* second_diff, double* threshold, int* violation, int* pass) {
  return guard([&] {
    WorkCurve c;
    for (uint64_t i = 0; i < n; ++i) c.points.push_back({sizes[i], mean[i], se[i], 0.0, 0.0});
    const ConcavityReport r = concavity_check(c);
    for (size_t i = 0; i < r.entries.size(); ++i) {
      second_diff[i] = r.entries[i].second_diff;
      threshold[i] = r.entries[i].threshold;
      violation[i] = r.entries[i].violation ? 1 : 0;
    }
    *pass = r.pass ? 1 : 0;
  });
}

/* graph.cpp:216-252 — the reference's own CBCS writer / reader. */
int rf_save_csr(void* g, const char* path) {
  return guard([&] { save_csr(*static_cast<Graph*>(g), path); });
}
int rf_load_csr(const char* path, uint64_t* n, uint64_t* m, uint64_t** indptr,
                uint32_t** indices) {
  return guard([&] {
    const Graph g = load_csr(path);
    *n = g.num_vertices;
    *m = g.indices.size();
    *indptr = static_cast<uint64_t*>(std::malloc((g.num_vertices + 1) * 8));
    *indices = static_cast<uint32_t*>(std::malloc(g.indices.size() * 4 + 4));
    std::memcpy(*indptr, g.indptr.data(), (g.num_vertices + 1) * 8);
    std::memcpy(*indices, g.indices.data(), g.indices.size() * 4);
  });
}

int rf_validate_csr(void* g) {
  return guard([&] { validate_csr(*static_cast<Graph*>(g)); });
}

/* graph.cpp:111-151 — the reference's own generator, for fixtures. */
int rf_generate_powerlaw(uint64_t n, double deg, double skew, uint64_t seed,
                         uint64_t** indptr, uint32_t** indices, uint64_t* m) {
  return guard([&] {
    const Graph g = generate_powerlaw(n, deg, skew, seed);
    *indptr = dup(g.indptr);
    *indices = dup(g.indices);
    *m = g.indices.size();
  });
}

int rf_build_csr(const uint32_t* src, const uint32_t* dst, uint64_t m, uint64_t n,
                 uint64_t* indptr, uint32_t* indices) {
  return guard([&] {
    std::vector<Edge> edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i]};
    const Graph g = build_csr(edges, n);
    std::memcpy(indptr, g.indptr.data(), (n + 1) * sizeof(uint64_t));
    if (m) std::memcpy(indices, g.indices.data(), m * sizeof(uint32_t));
  });
}

int rf_partition_random(uint64_t n, uint32_t parts, uint64_t seed, uint32_t* owner) {
  return guard([&] {
    const PartitionMap pm = partition_random(n, parts, seed);
    std::memcpy(owner, pm.owner.data(), n * sizeof(uint32_t));
  });
}

int rf_sample_block(void* g, const uint32_t* seeds, uint64_t n_seeds, int kind,
                    uint32_t fanout, const ob_sched* sched, int layer, ob_block* out) {
  return guard([&] {
    const VariateSource src = VariateSource::from_schedule(to_sched(sched));
    to_block(sample_block(*static_cast<Graph*>(g), {seeds, n_seeds},
                          to_cfg(kind, fanout), src, layer),
             out);
  });
}

/* sample_labor0 (samplers.cpp:305-312) with the variate r(t) = table[t]. */
int rf_sample_labor0(void* g, const uint32_t* seeds, uint64_t n_seeds, uint32_t k,
                     const double* table, int layer, ob_block* out) {
  return guard([&] {
    const std::function<double(VertexId)> variate = [table](VertexId t) { return table[t]; };
    to_block(sample_labor0(*static_cast<Graph*>(g), {seeds, n_seeds}, k, variate, layer), out);
  });
}

/* expand (samplers.cpp:340-354). With non-uniform fanouts the reference has
 * no single call, so the same loop is run over its public sample_block. */
int rf_expand(void* g, const uint32_t* seeds, uint64_t n_seeds, int L, int kind,
              const uint32_t* fanouts, const ob_sched* sched, ob_stack* out) {
  return guard([&] {
    bool uniform = true;
    for (int l = 1; l < L; ++l) uniform = uniform && fanouts[l] == fanouts[0];
    const Graph& gr = *static_cast<Graph*>(g);
    if (uniform) {
      to_stack(expand(gr, {seeds, n_seeds}, L, to_cfg(kind, L > 0 ? fanouts[0] : 1),
                      to_sched(sched)),
               out);
      return;
    }
    const VariateSource src = VariateSource::from_schedule(to_sched(sched));
    LayerStack st;
    std::vector<VertexId> cur(seeds, seeds + n_seeds);
    for (int l = 0; l < L; ++l) {
      st.blocks.push_back(sample_block(gr, cur, to_cfg(kind, fanouts[l]), src, l));
      cur = st.blocks.back().src_vertices;
    }
    to_stack(st, out);
  });
}

/* coop_sample (coop.cpp:68-106); uniform fanout only (reference API). */
int rf_coop_sample(void* g, const uint32_t* owner, uint32_t parts,
                   const uint32_t* seeds_flat, const uint64_t* seeds_off, int L,
                   int kind, uint32_t fanout, const ob_sched* sched, ob_coop* out) {
  std::memset(out, 0, sizeof(*out));
  return guard([&] {
    const Graph& gr = *static_cast<Graph*>(g);
    PartitionMap pm;
    pm.num_parts = parts;
    pm.owner.assign(owner, owner + gr.num_vertices);
    std::vector<std::vector<VertexId>> seeds(parts);
    for (uint32_t p = 0; p < parts; ++p)
      seeds[p].assign(seeds_flat + seeds_off[p], seeds_flat + seeds_off[p + 1]);
    const CoopSampleResult r =
        coop_sample(gr, pm, seeds, L, to_cfg(kind, fanout), to_sched(sched));
    out->num_parts = parts;
    out->num_layers = L;
    out->stacks = static_cast<ob_stack*>(std::calloc(parts, sizeof(ob_stack)));
    for (uint32_t p = 0; p < parts; ++p) to_stack(r.stacks[p], &out->stacks[p]);
    out->exchanges = static_cast<ob_exchange*>(std::calloc(L, sizeof(ob_exchange)));
    for (int l = 0; l < L; ++l) {
      const ExchangeRecord& rec = r.exchanges[l];
      ob_exchange* e = &out->exchanges[l];
      e->layer = rec.layer;
      e->num_parts = parts;
      e->send_counts = static_cast<uint64_t*>(std::malloc(parts * parts * sizeof(uint64_t)));
      for (uint32_t p = 0; p < parts; ++p)
        for (uint32_t q = 0; q < parts; ++q)
          e->send_counts[p * parts + q] = rec.send_counts[p][q];
      e->owner_row_counts = dup(rec.owner_row_counts);
      e->loc_len = static_cast<uint64_t*>(std::malloc(parts * sizeof(uint64_t)));
      e->loc_part = static_cast<uint32_t**>(std::calloc(parts, sizeof(uint32_t*)));
      e->loc_row = static_cast<uint64_t**>(std::calloc(parts, sizeof(uint64_t*)));
      for (uint32_t p = 0; p < parts; ++p) {
        const auto& loc = rec.src_location[p];
        e->loc_len[p] = loc.size();
        e->loc_part[p] = static_cast<uint32_t*>(std::malloc(loc.size() * 4 + 1));
        e->loc_row[p] = static_cast<uint64_t*>(std::malloc(loc.size() * 8 + 1));
        for (std::size_t j = 0; j < loc.size(); ++j) {
          e->loc_part[p][j] = loc[j].part;
          e->loc_row[p][j] = loc[j].row;
        }
      }
    }
    out->owner_len = static_cast<uint64_t*>(std::malloc(parts * sizeof(uint64_t)));
    out->owner_sets = static_cast<uint32_t**>(std::calloc(parts, sizeof(uint32_t*)));
    for (uint32_t p = 0; p < parts; ++p) {
      out->owner_len[p] = r.owner_sets[p].size();
      out->owner_sets[p] = dup(r.owner_sets[p]);
    }
  });
}

void rf_block_free(ob_block* b) {
  std::free(b->dst); std::free(b->src); std::free(b->edges); std::free(b->dst_pos);
  std::memset(b, 0, sizeof(*b));
}
void rf_stack_free(ob_stack* s) {
  for (int l = 0; l < s->num_layers; ++l) rf_block_free(&s->blocks[l]);
  std::free(s->blocks);
  s->blocks = nullptr;
  s->num_layers = 0;
}
void rf_coop_free(ob_coop* c) {
  if (c->stacks)
    for (uint32_t p = 0; p < c->num_parts; ++p) rf_stack_free(&c->stacks[p]);
  if (c->exchanges)
    for (int l = 0; l < c->num_layers; ++l) {
      ob_exchange* e = &c->exchanges[l];
      for (uint32_t p = 0; p < e->num_parts; ++p) {
        std::free(e->loc_part[p]);
        std::free(e->loc_row[p]);
      }
      std::free(e->send_counts); std::free(e->owner_row_counts); std::free(e->loc_len);
      std::free(e->loc_part); std::free(e->loc_row);
    }
  if (c->owner_sets)
    for (uint32_t p = 0; p < c->num_parts; ++p) std::free(c->owner_sets[p]);
  std::free(c->stacks); std::free(c->exchanges); std::free(c->owner_sets);
  std::free(c->owner_len);
  std::memset(c, 0, sizeof(*c));
}
void rf_free(void* p) { std::free(p); }

/* FeatureStore (coop.cpp:359-388). Holding the f64 table is the reference's
 * own behaviour; the caller bounds n*dim. */
void* rf_features_new(uint64_t n, uint32_t dim, uint32_t classes, uint64_t seed) {
  return new FeatureStore(FeatureStore::synth(n, dim, classes, seed));
}
void rf_features_free(void* f) { delete static_cast<FeatureStore*>(f); }
void rf_load_rows(void* f, const uint32_t* ids, uint64_t n, double* out) {
  const FeatureMatrix m = static_cast<FeatureStore*>(f)->load_rows({ids, n});
  if (!m.values.empty()) std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
}

/* all_to_all_forward (coop.cpp:145-159) along the exchange of a coop result's
 * layer l: owner rows are given flat with per-part offsets (rows). */
int rf_all_to_all_forward(const ob_coop* c, int layer, const double* owner_flat,
                          const uint64_t* owner_row_off, uint32_t dim, double* out_flat) {
  return guard([&] {
    const ob_exchange* e = &c->exchanges[layer];
    ExchangeRecord rec;
    rec.layer = e->layer;
    const uint32_t P = e->num_parts;
    rec.send_counts.assign(P, std::vector<std::uint64_t>(P));
    rec.src_location.resize(P);
    rec.owner_row_counts.assign(e->owner_row_counts, e->owner_row_counts + P);
    for (uint32_t p = 0; p < P; ++p) {
      for (uint32_t q = 0; q < P; ++q) rec.send_counts[p][q] = e->send_counts[p * P + q];
      for (uint64_t j = 0; j < e->loc_len[p]; ++j)
        rec.src_location[p].push_back({e->loc_part[p][j], e->loc_row[p][j]});
    }
    std::vector<std::vector<double>> owner(P);
    for (uint32_t q = 0; q < P; ++q)
      owner[q].assign(owner_flat + owner_row_off[q] * dim,
                      owner_flat + owner_row_off[q + 1] * dim);
    const auto fwd = all_to_all_forward(rec, owner, dim);
    std::size_t o = 0;
    for (uint32_t p = 0; p < P; ++p) {
      if (!fwd[p].empty()) std::memcpy(out_flat + o, fwd[p].data(), fwd[p].size() * 8);
      o += fwd[p].size();
    }
  });
}

/* One minibatch of the reference's own stock path, timed inside C++:
 *   coop : coop_sample -> per-part load_rows(owner_sets) -> all_to_all_forward
 *          (coop_train_step's prefix, coop.cpp:445-467)
 *   indep: indep_sample -> per-part load_rows(input_vertices)
 *          (indep_train_step's prefix, coop.cpp:560 + FeatureStore use)
 * Returns seconds spent sampling and loading features and the rows
 * delivered (requester-aligned). */
int rf_step(void* g, void* fs, int mode, const uint32_t* owner, uint32_t parts,
            const uint32_t* seeds_flat, const uint64_t* seeds_off, int L, int kind,
            uint32_t fanout, const ob_sched* sched, double* t_sample, double* t_gather,
            uint64_t* rows_out) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    const Graph& gr = *static_cast<Graph*>(g);
    const FeatureStore& store = *static_cast<FeatureStore*>(fs);
    std::vector<std::vector<VertexId>> seeds(parts);
    for (uint32_t p = 0; p < parts; ++p)
      seeds[p].assign(seeds_flat + seeds_off[p], seeds_flat + seeds_off[p + 1]);
    const SamplerConfig cfg = to_cfg(kind, fanout);
    const SeedSchedule sc = to_sched(sched);
    uint64_t rows = 0;
    if (mode == 0) {
      PartitionMap pm;
      pm.num_parts = parts;
      pm.owner.assign(owner, owner + gr.num_vertices);
      const auto t0 = clk::now();
      const CoopSampleResult r = coop_sample(gr, pm, seeds, L, cfg, sc);
      const auto t1 = clk::now();
      std::vector<std::vector<double>> owner_rows(parts);
      for (uint32_t p = 0; p < parts; ++p)
        owner_rows[p] = store.load_rows(r.owner_sets[p]).values;
      const auto fwd = all_to_all_forward(r.exchanges[L - 1], owner_rows, store.dim);
      const auto t2 = clk::now();
      for (const auto& f : fwd) rows += f.size() / store.dim;
      *t_sample = std::chrono::duration<double>(t1 - t0).count();
      *t_gather = std::chrono::duration<double>(t2 - t1).count();
    } else {
      const auto t0 = clk::now();
      const auto stacks = indep_sample(gr, seeds, L, cfg, sc);
      const auto t1 = clk::now();
      for (uint32_t p = 0; p < parts; ++p)
        rows += store.load_rows(stacks[p].input_vertices()).rows();
      const auto t2 = clk::now();
      *t_sample = std::chrono::duration<double>(t1 - t0).count();
      *t_gather = std::chrono::duration<double>(t2 - t1).count();
    }
    *rows_out = rows;
  });
}

/* The same stock path for graphs whose f64 FeatureStore does not fit host
 * memory (c4: 111M x 128 x 8 B = 113 GB): sampling is the
 * reference's own coop_sample / indep_sample, and load_rows is replaced by
 * computing each requested row from FeatureStore::synth's formula
 * (coop.cpp:369-371: 2 * hash_uniform(seed, {kStreamFeature, v, j}) - 1) with
 * the reference's hash, parallel over parts (parallel.hpp). Coop mode then
 * runs the reference's all_to_all_forward on the owner rows. */
static std::vector<double> rows_on_the_fly(std::span<const VertexId> ids, uint32_t dim,
                                           uint64_t seed) {
  std::vector<double> out(ids.size() * dim);
  for (std::size_t r = 0; r < ids.size(); ++r)
    for (uint32_t j = 0; j < dim; ++j)
      out[r * dim + j] = 2.0 * hash_uniform(seed, {kStreamFeature, ids[r], j}) - 1.0;
  return out;
}

int rf_step_onfly(void* g, uint64_t feat_seed, uint32_t dim, int mode, const uint32_t* owner,
                  uint32_t parts, const uint32_t* seeds_flat, const uint64_t* seeds_off, int L,
                  int kind, uint32_t fanout, const ob_sched* sched, double* t_sample,
                  double* t_gather, uint64_t* rows_out) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    const Graph& gr = *static_cast<Graph*>(g);
    std::vector<std::vector<VertexId>> seeds(parts);
    for (uint32_t p = 0; p < parts; ++p)
      seeds[p].assign(seeds_flat + seeds_off[p], seeds_flat + seeds_off[p + 1]);
    const SamplerConfig cfg = to_cfg(kind, fanout);
    const SeedSchedule sc = to_sched(sched);
    uint64_t rows = 0;
    std::vector<std::vector<double>> part_rows(parts);
    if (mode == 0) {
      PartitionMap pm;
      pm.num_parts = parts;
      pm.owner.assign(owner, owner + gr.num_vertices);
      const auto t0 = clk::now();
      const CoopSampleResult r = coop_sample(gr, pm, seeds, L, cfg, sc);
      const auto t1 = clk::now();
      parallel_for(parts, [&](std::size_t p) {
        part_rows[p] = rows_on_the_fly(r.owner_sets[p], dim, feat_seed);
      });
      const auto fwd = all_to_all_forward(r.exchanges[L - 1], part_rows, dim);
      const auto t2 = clk::now();
      for (const auto& f : fwd) rows += f.size() / dim;
      *t_sample = std::chrono::duration<double>(t1 - t0).count();
      *t_gather = std::chrono::duration<double>(t2 - t1).count();
    } else {
      const auto t0 = clk::now();
      const auto stacks = indep_sample(gr, seeds, L, cfg, sc);
      const auto t1 = clk::now();
      parallel_for(parts, [&](std::size_t p) {
        part_rows[p] = rows_on_the_fly(stacks[p].input_vertices(), dim, feat_seed);
      });
      const auto t2 = clk::now();
      for (const auto& f : part_rows) rows += f.size() / dim;
      *t_sample = std::chrono::duration<double>(t1 - t0).count();
      *t_gather = std::chrono::duration<double>(t2 - t1).count();
    }
    *rows_out = rows;
  });
}

/* LruCache (cache.cpp:8-32) */
void* rf_lru_new(uint64_t cap) {
  try {
    return new LruCache(cap);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int rf_lru_access(void* c, uint32_t key) {
  return static_cast<LruCache*>(c)->access(key) == CacheOutcome::kMiss ? 1 : 0;
}
void rf_lru_free(void* c) { delete static_cast<LruCache*>(c); }

/* run_dependent_experiment (cache.cpp:137-208): per-step fingerprint, input
 * count and miss bytes, plus the steady miss rate. */
int rf_dependent_experiment(void* g, int mode, uint64_t kappa, uint64_t batch,
                            uint64_t steps, uint64_t capacity, int kind, uint32_t fanout,
                            int L, uint32_t dim, uint32_t bps, uint64_t seed,
                            uint64_t* fingerprints, uint64_t* s_l, uint64_t* bytes,
                            double* steady) {
  return guard([&] {
    MinibatchSchedule ms;
    ms.mode = static_cast<BatchMode>(mode);
    ms.kappa = kappa;
    ms.batch_size = batch;
    const auto r = run_dependent_experiment(*static_cast<Graph*>(g), ms, steps, capacity,
                                            to_cfg(kind, fanout), L, dim, bps, seed);
    for (std::size_t i = 0; i < r.rows.size(); ++i) {
      fingerprints[i] = r.rows[i].fingerprint;
      s_l[i] = r.rows[i].s_l;
      bytes[i] = r.rows[i].bytes;
    }
    *steady = r.steady_miss_rate;
  });
}

}  // extern "C"
