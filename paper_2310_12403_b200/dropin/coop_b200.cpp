// Drop-in replacement of the reference's src/coop.cpp: the functions declared
// in include/coopbatch/coop.hpp (unchanged), run by libcoopbatch_b200.so.
//
//   coop_sample             coop.cpp:68-106 (+ build_exchange 25-64)
//                           -> one cooperative batch of P parts on the device
//   indep_sample            coop.cpp:108-119 -> the P parts as one batch
//   all_to_all_forward      coop.cpp:145-159 -> cb_op_forward_rows
//   all_to_all_reverse(_sum) coop.cpp:161-194 -> cb_op_reverse_rows
//   gcn_forward/backward    coop.cpp:196-331 -> cb_op_gcn_block (FP64)
//   GcnModel::init          coop.cpp:333-357 -> cb_gcn_model_init
//   FeatureStore::synth     coop.cpp:359-376 -> cb_synth_host
//   FeatureStore::load_rows coop.cpp:378-388 -> rows gathered on the device
//                           from the store's host table, read in place
//   coop_/indep_train_step  coop.cpp:438-610 -> cb_train_step
// Argument checks run on the host first, in the reference's order and with
// its messages, so the same calls throw the same InputErrors.
#include <numeric>

#include "ctx.hpp"

namespace coopbatch {

namespace {

using namespace b200;

struct Flat {
  std::vector<VertexId> ids;
  std::vector<std::uint64_t> off{0};
  std::uint64_t max_part = 0;
};

Flat flatten(const std::vector<std::vector<VertexId>>& per_pe) {
  Flat f;
  for (const auto& s : per_pe) {
    f.ids.insert(f.ids.end(), s.begin(), s.end());
    f.off.push_back(f.ids.size());
    f.max_part = std::max<std::uint64_t>(f.max_part, s.size());
  }
  return f;
}

// coop_sample's checks (coop.cpp:72-83)
void check_coop_inputs(const Graph& g, const PartitionMap& pm,
                       const std::vector<std::vector<VertexId>>& per_pe, int num_layers) {
  const std::uint32_t parts = pm.num_parts;
  if (per_pe.size() != parts)
    throw InputError("coop_sample: seed lists must match the partition count");
  validate_partition(pm, g.num_vertices);
  for (std::uint32_t p = 0; p < parts; ++p)
    for (const VertexId s : per_pe[p]) {
      g.check_vertex(s);
      if (pm.owner[s] != p)
        throw InputError("coop_sample: seed " + std::to_string(s) + " is not owned by part " +
                         std::to_string(p));
    }
  if (num_layers < 1) throw InputError("coop_sample: num_layers must be >= 1");
}

// one cooperative batch on the device; the plan holds its result
cb_plan* coop_batch(const Graph& g, const PartitionMap& pm,
                    const std::vector<std::vector<VertexId>>& per_pe, int num_layers,
                    const SamplerConfig& cfg, const SeedSchedule& schedule) {
  check_coop_inputs(g, pm, per_pe, num_layers);
  const Flat f = flatten(per_pe);
  cb_plan* pl = plan_for({&g, &pm, pm.num_parts, num_layers, &cfg, std::max<std::uint64_t>(f.max_part, 1)});
  const cb_sched s = to_sched(schedule);
  check(cb_sample_sync(pl, CB_MODE_COOP, f.ids.data(), f.off.data(), &s));
  return pl;
}

ExchangeRecord download_exchange(cb_plan* pl, std::uint32_t P, int l,
                                 const std::vector<std::uint64_t>& n_src) {
  ExchangeRecord e;
  e.layer = l;
  std::vector<std::uint64_t> sc(static_cast<std::size_t>(P) * P), orc(P);
  const std::uint64_t tot = std::accumulate(n_src.begin(), n_src.end(), std::uint64_t{0});
  std::vector<std::uint32_t> lp(tot);
  std::vector<std::uint64_t> lr(tot);
  check(cb_download_exchange(pl, l, sc.data(), orc.data(), lp.data(), lr.data()));
  e.send_counts.assign(P, std::vector<std::uint64_t>(P));
  for (std::uint32_t p = 0; p < P; ++p)
    for (std::uint32_t q = 0; q < P; ++q) e.send_counts[p][q] = sc[p * P + q];
  e.owner_row_counts = std::move(orc);
  e.src_location.resize(P);
  std::uint64_t o = 0;
  for (std::uint32_t p = 0; p < P; ++p) {
    e.src_location[p].resize(n_src[p]);
    for (std::uint64_t j = 0; j < n_src[p]; ++j, ++o) e.src_location[p][j] = {lp[o], lr[o]};
  }
  return e;
}

std::vector<std::uint64_t> src_counts(cb_plan* pl, std::uint32_t P, int l) {
  std::vector<std::uint64_t> n(P);
  for (std::uint32_t p = 0; p < P; ++p) {
    std::uint64_t sz[6];
    layer_sizes(pl, p, l, sz);
    n[p] = sz[1];
  }
  return n;
}

// indep_sample's batches: the parts run as one device batch (at most 64 parts
// per plan, so larger part counts run in groups)
template <typename Fn>
void indep_batches(const Graph& g, const std::vector<std::vector<VertexId>>& per_pe,
                   int num_layers, const SamplerConfig& cfg, const SeedSchedule& schedule,
                   Fn&& consume) {
  constexpr std::size_t kGroup = 64;
  const cb_sched s = to_sched(schedule);
  for (std::size_t p0 = 0; p0 < per_pe.size(); p0 += kGroup) {
    const std::size_t p1 = std::min(per_pe.size(), p0 + kGroup);
    const std::vector<std::vector<VertexId>> group(per_pe.begin() + p0, per_pe.begin() + p1);
    const Flat f = flatten(group);
    const auto parts = static_cast<std::uint32_t>(group.size());
    cb_plan* pl =
        plan_for({&g, nullptr, parts, num_layers, &cfg, std::max<std::uint64_t>(f.max_part, 1)});
    check(cb_sample_sync(pl, CB_MODE_INDEP, f.ids.data(), f.off.data(), &s));
    consume(pl, p0, parts);
  }
}

void check_owner_rows(const ExchangeRecord& rec, const std::vector<std::vector<double>>& rows,
                      std::uint32_t dim, const char* what) {
  if (rows.size() != rec.num_parts()) throw InputError(std::string(what) + ": part count mismatch");
  for (std::uint32_t q = 0; q < rec.num_parts(); ++q)
    if (rows[q].size() != rec.owner_row_counts[q] * dim)
      throw InputError(std::string(what) + ": owner payload shape mismatch");
}

void check_requester_rows(const ExchangeRecord& rec, const std::vector<std::vector<double>>& rows,
                          std::uint32_t dim, const char* what) {
  if (rows.size() != rec.num_parts()) throw InputError(std::string(what) + ": part count mismatch");
  for (std::uint32_t p = 0; p < rec.num_parts(); ++p)
    if (rows[p].size() != rec.src_location[p].size() * dim)
      throw InputError(std::string(what) + ": requester payload shape mismatch");
}

// an ExchangeRecord as the C-ABI's flat arrays
struct FlatRecord {
  std::vector<std::uint64_t> off{0}, row;
  std::vector<std::uint32_t> part;
};

FlatRecord flat_record(const ExchangeRecord& rec) {
  FlatRecord f;
  for (const auto& loc : rec.src_location) {
    for (const RemoteRef& r : loc) {
      f.part.push_back(r.part);
      f.row.push_back(r.row);
    }
    f.off.push_back(f.part.size());
  }
  return f;
}

std::vector<std::vector<double>> split_rows(const std::vector<double>& flat,
                                            const std::vector<std::uint64_t>& counts,
                                            std::uint32_t dim) {
  std::vector<std::vector<double>> out(counts.size());
  std::uint64_t o = 0;
  for (std::size_t i = 0; i < counts.size(); ++i) {
    out[i].assign(flat.begin() + o * dim, flat.begin() + (o + counts[i]) * dim);
    o += counts[i];
  }
  return out;
}

std::vector<std::vector<double>> reverse_rows(const ExchangeRecord& rec,
                                              const std::vector<std::vector<double>>& req,
                                              std::uint32_t dim, bool sum) {
  const FlatRecord f = flat_record(rec);
  std::vector<double> in;
  for (const auto& r : req) in.insert(in.end(), r.begin(), r.end());
  const std::uint64_t n_owner =
      std::accumulate(rec.owner_row_counts.begin(), rec.owner_row_counts.end(), std::uint64_t{0});
  std::vector<double> out(n_owner * dim, 0.0);
  check(cb_op_reverse_rows(device(), rec.num_parts(), f.off.data(), f.part.data(), f.row.data(),
                           rec.owner_row_counts.data(), dim, in.data(), sum ? 1 : 0, out.data()));
  return split_rows(out, rec.owner_row_counts, dim);
}

void check_forward_shapes(const BipartiteBlock& block, const FeatureMatrix& h_in,
                          const DenseMatrix& w) {
  if (h_in.rows() != block.src_vertices.size())
    throw InputError("gcn: input rows do not align with block sources");
  if (w.rows != h_in.dim) throw InputError("gcn: weight rows do not match input dim");
}

void check_model(const GcnModel& model, int num_layers, const FeatureStore& store) {
  if (static_cast<int>(model.weights.size()) != num_layers)
    throw InputError("train step: model depth does not match layer count");
  if (model.weights.back().rows != store.dim)
    throw InputError("train step: model input dim does not match store");
}

// The model on the device (weights uploaded, shapes as the host model's).
struct DeviceModel {
  cb_model* m = nullptr;
  explicit DeviceModel(const GcnModel& model) {
    const int L = static_cast<int>(model.weights.size());
    std::vector<std::uint32_t> rows, cols;
    std::vector<double> w;
    for (const auto& d : model.weights) {
      rows.push_back(static_cast<std::uint32_t>(d.rows));
      cols.push_back(static_cast<std::uint32_t>(d.cols));
      w.insert(w.end(), d.data.begin(), d.data.end());
    }
    check(cb_gcn_model_create(device(), L, rows.data(), cols.data(),
                              model.hidden_activation == Activation::kTanh ? 1 : 0, w.data(), &m));
  }
  ~DeviceModel() { cb_gcn_model_destroy(m); }
};

// The store's rows and labels as a device table (read in place for large
// tables, see MappedHostTable).
struct DeviceStore {
  MappedHostTable table;
  explicit DeviceStore(const FeatureStore& s)
      : table(s.values.data(), s.dim ? s.values.size() / s.dim : 0, s.dim) {
    if (!s.labels.empty()) check(cb_features_set_labels(table.get(), s.labels.data()));
  }
};

TrainStepResult run_train(cb_plan* pl, const GcnModel& model, const FeatureStore& store) {
  if (store.labels.size() * store.dim != store.values.size())
    throw InputError("train step: store labels do not cover its rows");
  DeviceModel dm(model);
  DeviceStore ds(store);
  TrainStepResult r;
  std::uint64_t total = 0;
  for (const auto& w : model.weights) total += w.rows * w.cols;
  std::vector<double> gw(total);
  check(cb_train_step(pl, ds.table.get(), model.num_classes(), dm.m, &r.loss, gw.data()));
  std::uint64_t o = 0;
  for (const auto& w : model.weights) {
    DenseMatrix d = DenseMatrix::zeros(w.rows, w.cols);
    std::copy(gw.begin() + o, gw.begin() + o + w.rows * w.cols, d.data.begin());
    o += w.rows * w.cols;
    r.grad_w.push_back(std::move(d));
  }
  r.metrics.loss = r.loss;
  return r;
}

std::vector<LayerMetrics> part_metrics(cb_plan* pl, std::uint32_t p, int L) {
  std::vector<LayerMetrics> out;
  for (int l = 0; l < L; ++l) {
    std::uint64_t sz[6];
    layer_sizes(pl, p, l, sz);
    out.push_back({sz[0], sz[1], sz[2], 0});
  }
  return out;
}

}  // namespace

std::uint64_t ExchangeRecord::communicated(std::uint32_t p) const {
  std::uint64_t n = 0;
  for (std::uint32_t q = 0; q < num_parts(); ++q) n += q == p ? 0 : send_counts[p][q];
  return n;
}

std::uint64_t ExchangeRecord::total_communicated() const {
  std::uint64_t n = 0;
  for (std::uint32_t p = 0; p < num_parts(); ++p) n += communicated(p);
  return n;
}

CoopSampleResult coop_sample(const Graph& g, const PartitionMap& pm,
                             const std::vector<std::vector<VertexId>>& per_pe_seeds,
                             int num_layers, const SamplerConfig& cfg,
                             const SeedSchedule& schedule) {
  Lock lk(api_mutex());
  cb_plan* pl = coop_batch(g, pm, per_pe_seeds, num_layers, cfg, schedule);
  const std::uint32_t P = pm.num_parts;
  CoopSampleResult r;
  r.stacks.resize(P);
  for (std::uint32_t p = 0; p < P; ++p)
    for (int l = 0; l < num_layers; ++l) r.stacks[p].blocks.push_back(download_block(pl, p, l, l));
  for (int l = 0; l < num_layers; ++l) {
    std::vector<std::uint64_t> ns(P);
    for (std::uint32_t p = 0; p < P; ++p) ns[p] = r.stacks[p].blocks[l].src_vertices.size();
    r.exchanges.push_back(download_exchange(pl, P, l, ns));
  }
  r.owner_sets.resize(P);
  for (std::uint32_t p = 0; p < P; ++p) {
    std::uint64_t n = 0;
    check(cb_owner_set_size(pl, p, &n));
    r.owner_sets[p].resize(n);
    if (n) check(cb_download_owner_set(pl, p, r.owner_sets[p].data()));
  }
  return r;
}

std::vector<LayerStack> indep_sample(const Graph& g,
                                     const std::vector<std::vector<VertexId>>& per_pe_seeds,
                                     int num_layers, const SamplerConfig& cfg,
                                     const SeedSchedule& schedule) {
  Lock lk(api_mutex());
  for (const auto& seeds : per_pe_seeds)
    for (const VertexId s : seeds) g.check_vertex(s);
  if (num_layers < 1) throw InputError("expand: num_layers must be >= 1");
  std::vector<LayerStack> stacks(per_pe_seeds.size());
  indep_batches(g, per_pe_seeds, num_layers, cfg, schedule,
                [&](cb_plan* pl, std::size_t p0, std::uint32_t parts) {
                  for (std::uint32_t p = 0; p < parts; ++p)
                    for (int l = 0; l < num_layers; ++l)
                      stacks[p0 + p].blocks.push_back(download_block(pl, p, l, l));
                });
  return stacks;
}

std::vector<std::vector<double>> all_to_all_forward(
    const ExchangeRecord& rec, const std::vector<std::vector<double>>& owner_rows,
    std::uint32_t dim) {
  Lock lk(api_mutex());
  check_owner_rows(rec, owner_rows, dim, "all_to_all_forward");
  const FlatRecord f = flat_record(rec);
  std::vector<double> in;
  for (const auto& r : owner_rows) in.insert(in.end(), r.begin(), r.end());
  std::vector<double> out(f.part.size() * dim);
  check(cb_op_forward_rows(device(), rec.num_parts(), f.off.data(), f.part.data(), f.row.data(),
                           rec.owner_row_counts.data(), dim, in.data(), out.data()));
  std::vector<std::uint64_t> counts;
  for (const auto& loc : rec.src_location) counts.push_back(loc.size());
  return split_rows(out, counts, dim);
}

std::vector<std::vector<double>> all_to_all_reverse(
    const ExchangeRecord& rec, const std::vector<std::vector<double>>& requester_rows,
    std::uint32_t dim) {
  Lock lk(api_mutex());
  check_requester_rows(rec, requester_rows, dim, "all_to_all_reverse");
  return reverse_rows(rec, requester_rows, dim, false);
}

std::vector<std::vector<double>> all_to_all_reverse_sum(
    const ExchangeRecord& rec, const std::vector<std::vector<double>>& requester_rows,
    std::uint32_t dim) {
  Lock lk(api_mutex());
  check_requester_rows(rec, requester_rows, dim, "all_to_all_reverse_sum");
  return reverse_rows(rec, requester_rows, dim, true);
}

FeatureMatrix gcn_forward(const BipartiteBlock& block, const FeatureMatrix& h_in,
                          const DenseMatrix& w, Activation act) {
  Lock lk(api_mutex());
  check_forward_shapes(block, h_in, w);
  FeatureMatrix out;
  out.row_ids = block.dst_vertices;
  out.dim = static_cast<std::uint32_t>(w.cols);
  out.values.assign(block.dst_vertices.size() * w.cols, 0.0);
  check(cb_op_gcn_block(device(), block.src_vertices.size(), block.dst_vertices.size(),
                        block.edges.size(), reinterpret_cast<const std::uint32_t*>(block.edges.data()),
                        block.dst_pos_in_src.data(), h_in.values.data(), h_in.dim, w.data.data(),
                        out.dim, act == Activation::kTanh ? 1 : 0, nullptr, out.values.data(),
                        nullptr, nullptr));
  return out;
}

GcnBackwardResult gcn_backward(const BipartiteBlock& block, const FeatureMatrix& h_in,
                               const DenseMatrix& w, const FeatureMatrix& grad_out,
                               Activation act) {
  Lock lk(api_mutex());
  check_forward_shapes(block, h_in, w);
  if (grad_out.rows() != block.dst_vertices.size() || grad_out.dim != w.cols)
    throw InputError("gcn_backward: grad_out shape mismatch");
  GcnBackwardResult r;
  r.grad_w = DenseMatrix::zeros(w.rows, w.cols);
  r.grad_h_in.row_ids = block.src_vertices;
  r.grad_h_in.dim = h_in.dim;
  r.grad_h_in.values.assign(h_in.values.size(), 0.0);
  check(cb_op_gcn_block(device(), block.src_vertices.size(), block.dst_vertices.size(),
                        block.edges.size(), reinterpret_cast<const std::uint32_t*>(block.edges.data()),
                        block.dst_pos_in_src.data(), h_in.values.data(), h_in.dim, w.data.data(),
                        static_cast<std::uint32_t>(w.cols), act == Activation::kTanh ? 1 : 0,
                        grad_out.values.data(), nullptr, r.grad_h_in.values.data(),
                        r.grad_w.data.data()));
  return r;
}

GcnModel GcnModel::init(std::uint32_t in_dim, std::uint32_t hidden, std::uint32_t num_classes,
                        int num_layers, std::uint64_t seed) {
  Lock lk(api_mutex());
  if (num_layers < 1) throw InputError("GcnModel: num_layers must be >= 1");
  cb_model* m = nullptr;
  check(cb_gcn_model_init(device(), in_dim, hidden, num_classes, num_layers, seed, &m));
  GcnModel model;
  try {
    for (int l = 0; l < num_layers; ++l) {
      std::uint64_t rows = 0, cols = 0;
      check(cb_gcn_model_weights(m, l, nullptr, 0, &rows, &cols));
      DenseMatrix w = DenseMatrix::zeros(rows, cols);
      check(cb_gcn_model_weights(m, l, w.data.data(), 0, &rows, &cols));
      model.weights.push_back(std::move(w));
    }
  } catch (...) {
    cb_gcn_model_destroy(m);
    throw;
  }
  cb_gcn_model_destroy(m);
  return model;
}

FeatureStore FeatureStore::synth(std::uint64_t num_vertices, std::uint32_t dim,
                                 std::uint32_t num_classes, std::uint64_t seed,
                                 std::uint32_t bytes_per_scalar) {
  Lock lk(api_mutex());
  FeatureStore fs;
  fs.dim = dim;
  fs.num_classes = num_classes;
  fs.bytes_per_scalar = bytes_per_scalar;
  fs.values.resize(num_vertices * dim);
  fs.labels.resize(num_vertices);
  check(cb_synth_host(device(), num_vertices, dim, num_classes, seed,
                      fs.values.empty() ? nullptr : fs.values.data(),
                      fs.labels.empty() ? nullptr : fs.labels.data()));
  return fs;
}

FeatureMatrix FeatureStore::load_rows(std::span<const VertexId> ids) const {
  Lock lk(api_mutex());
  FeatureMatrix m;
  m.row_ids.assign(ids.begin(), ids.end());
  m.dim = dim;
  m.values.resize(ids.size() * dim);
  if (ids.empty() || dim == 0) return m;
  const std::uint64_t n_rows = values.size() / dim;
  if (n_rows * dim * 8 <= (16ULL << 20)) {  // small: copied to HBM per call
    MappedHostTable t(values.data(), n_rows, dim);
    check(cb_op_load_rows(t.get(), ids.data(), ids.size(), m.values.data()));
  } else {  // large: registered once, read in place
    cb_features* t = cached_host_table(values.data(), n_rows, dim);
    check(cb_op_load_rows(t, ids.data(), ids.size(), m.values.data()));
  }
  return m;
}

TrainStepResult coop_train_step(const Graph& g, const PartitionMap& pm,
                                const std::vector<std::vector<VertexId>>& per_pe_seeds,
                                int num_layers, const SamplerConfig& cfg,
                                const SeedSchedule& schedule, const GcnModel& model,
                                const FeatureStore& store) {
  Lock lk(api_mutex());
  check_model(model, num_layers, store);
  cb_plan* pl = coop_batch(g, pm, per_pe_seeds, num_layers, cfg, schedule);
  TrainStepResult r = run_train(pl, model, store);
  const std::uint32_t P = pm.num_parts;
  r.metrics.per_pe.resize(P);
  std::vector<ExchangeRecord> ex;
  for (int l = 0; l < num_layers; ++l) ex.push_back(download_exchange(pl, P, l, src_counts(pl, P, l)));
  for (std::uint32_t p = 0; p < P; ++p) {
    PeMetrics& m = r.metrics.per_pe[p];
    std::uint64_t owned = 0;
    check(cb_owner_set_size(pl, p, &owned));
    m.feat_bytes = store.bytes_for(owned);
    m.input_rows = owned;
    m.layers = part_metrics(pl, p, num_layers);
    for (int l = 0; l < num_layers; ++l) m.layers[l].comm_vertices = ex[l].communicated(p);
  }
  return r;
}

TrainStepResult indep_train_step(const Graph& g,
                                 const std::vector<std::vector<VertexId>>& per_pe_seeds,
                                 int num_layers, const SamplerConfig& cfg,
                                 const SeedSchedule& schedule, const GcnModel& model,
                                 const FeatureStore& store) {
  Lock lk(api_mutex());
  check_model(model, num_layers, store);
  if (per_pe_seeds.empty()) throw InputError("indep_train_step: no parts");
  if (per_pe_seeds.size() > 64)
    throw InputError("indep_train_step: at most 64 parts per step on the device");
  for (const auto& seeds : per_pe_seeds)
    for (const VertexId s : seeds) g.check_vertex(s);
  TrainStepResult r;
  indep_batches(g, per_pe_seeds, num_layers, cfg, schedule,
                [&](cb_plan* pl, std::size_t, std::uint32_t parts) {
                  r = run_train(pl, model, store);
                  r.metrics.per_pe.resize(parts);
                  for (std::uint32_t p = 0; p < parts; ++p) {
                    PeMetrics& m = r.metrics.per_pe[p];
                    m.layers = part_metrics(pl, p, num_layers);
                    m.input_rows = m.layers.back().s_tilde_l;
                    m.feat_bytes = store.bytes_for(m.input_rows);
                  }
                });
  return r;
}

}  // namespace coopbatch
