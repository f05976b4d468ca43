// GPU: the C++ drop-in (include/coopbatch_b200.hpp) exercised like the
// reference's own doctest suites (test_samplers.cpp / test_coop.cpp), with
// the compiled reference (oracle/_ref, through its rf_* shim) as the checker.
// Built and run by tests/test_gpu_cpp.py. Exit code 0 = pass.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "coopbatch_b200.hpp"
#include "ob_types.h"

extern "C" {
void* rf_graph_new(const uint64_t*, const uint32_t*, uint64_t, uint64_t);
void rf_graph_free(void*);
int rf_generate_powerlaw(uint64_t, double, double, uint64_t, uint64_t**, uint32_t**, uint64_t*);
int rf_expand(void*, const uint32_t*, uint64_t, int, int, const uint32_t*, const ob_sched*,
              ob_stack*);
int rf_coop_sample(void*, const uint32_t*, uint32_t, const uint32_t*, const uint64_t*, int, int,
                   uint32_t, const ob_sched*, ob_coop*);
int rf_partition_random(uint64_t, uint32_t, uint64_t, uint32_t*);
void rf_stack_free(ob_stack*);
void rf_coop_free(ob_coop*);
void rf_sched_make(uint64_t, uint64_t, ob_sched*);
void rf_free(void*);
void* rf_lru_new(uint64_t);
int rf_lru_access(void*, uint32_t);
void rf_lru_free(void*);
void* rf_features_new(uint64_t, uint32_t, uint32_t, uint64_t);
void rf_features_free(void*);
int rf_train_step(void*, void*, int, const uint32_t*, uint32_t, const uint32_t*, const uint64_t*,
                  int, int, uint32_t, const ob_sched*, uint32_t, uint64_t, double*, double*);
int rf_save_csr(void*, const char*);
int rf_sample_block(void*, const uint32_t*, uint64_t, int, uint32_t, const ob_sched*, int,
                    ob_block*);
int rf_sample_labor0(void*, const uint32_t*, uint64_t, uint32_t, const double*, int, ob_block*);
void rf_block_free(ob_block*);
}

#include <cmath>
#include <string>

namespace cb = coopbatch_b200;

static int g_fail = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

static bool same_block(const cb::BipartiteBlock& a, const ob_block& b) {
  if (a.dst_vertices.size() != b.n_dst || a.src_vertices.size() != b.n_src ||
      a.edges.size() != b.n_edges)
    return false;
  for (uint64_t i = 0; i < b.n_dst; ++i)
    if (a.dst_vertices[i] != b.dst[i] || a.dst_pos_in_src[i] != b.dst_pos[i]) return false;
  for (uint64_t i = 0; i < b.n_src; ++i)
    if (a.src_vertices[i] != b.src[i]) return false;
  for (uint64_t e = 0; e < b.n_edges; ++e)
    if (a.edges[e].first != b.edges[2 * e] || a.edges[e].second != b.edges[2 * e + 1])
      return false;
  return true;
}

int main() {
  uint64_t* ip = nullptr;
  uint32_t* ix = nullptr;
  uint64_t m = 0;
  const uint64_t n = 2000;
  if (rf_generate_powerlaw(n, 8, 0.6, 7, &ip, &ix, &m) != 0) return 2;
  std::vector<uint64_t> indptr(ip, ip + n + 1);
  std::vector<uint32_t> indices(ix, ix + m);
  void* rg = rf_graph_new(ip, ix, n, m);
  auto g = cb::Graph::from_csr(indptr, indices);

  // expand == reference expand, every kind, kappa 1 and 4 (smoothed)
  const std::vector<uint32_t> seeds{5, 9, 100, 317, 1999, 0, 1024};
  for (int kind : {CB_FULL, CB_NS, CB_LABOR0})
    for (uint64_t kappa : {1ULL, 4ULL}) {
      ob_sched s;
      rf_sched_make(kappa, 31, &s);
      cb::SamplerConfig cfg;
      cfg.kind = static_cast<cb::SamplerKind>(kind);
      cfg.fanout = 4;
      const auto got = cb::expand(g, seeds, 3, cfg, {s.kappa, s.z1, s.z2, s.iteration});
      const uint32_t fo[3] = {4, 4, 4};
      ob_stack want{};
      CHECK(rf_expand(rg, seeds.data(), seeds.size(), 3, kind, fo, &s, &want) == 0);
      for (int l = 0; l < 3; ++l) CHECK(same_block(got.blocks[l], want.blocks[l]));
      rf_stack_free(&want);
    }

  // coop_sample == reference coop_sample (P = 4)
  std::vector<uint32_t> owner(n);
  rf_partition_random(n, 4, 3, owner.data());
  auto pm = cb::PartitionMap::from_owner(g, owner, 4);
  std::vector<std::vector<uint32_t>> per_pe(4);
  for (uint32_t v = 0; v < n; v += 13) per_pe[owner[v]].push_back(v);
  std::vector<uint32_t> flat;
  std::vector<uint64_t> off{0};
  for (auto& s : per_pe) {
    flat.insert(flat.end(), s.begin(), s.end());
    off.push_back(flat.size());
  }
  ob_sched s{1, 77, 77, 0};
  cb::SamplerConfig cfg;
  cfg.kind = cb::SamplerKind::kLabor0;
  cfg.fanout = 5;
  const auto got = cb::coop_sample(g, pm, per_pe, 3, cfg, {1, 77, 77, 0});
  ob_coop want{};
  CHECK(rf_coop_sample(rg, owner.data(), 4, flat.data(), off.data(), 3, CB_LABOR0, 5, &s,
                       &want) == 0);
  for (uint32_t p = 0; p < 4; ++p) {
    for (int l = 0; l < 3; ++l) CHECK(same_block(got.stacks[p].blocks[l], want.stacks[p].blocks[l]));
    CHECK(got.owner_sets[p].size() == want.owner_len[p]);
    for (uint64_t i = 0; i < want.owner_len[p]; ++i)
      CHECK(got.owner_sets[p][i] == want.owner_sets[p][i]);
  }
  for (int l = 0; l < 3; ++l)
    for (uint32_t p = 0; p < 4; ++p) {
      for (uint32_t q = 0; q < 4; ++q)
        CHECK(got.exchanges[l].send_counts[p][q] == want.exchanges[l].send_counts[p * 4 + q]);
      for (uint64_t j = 0; j < want.exchanges[l].loc_len[p]; ++j) {
        CHECK(got.exchanges[l].src_location[p][j].part == want.exchanges[l].loc_part[p][j]);
        CHECK(got.exchanges[l].src_location[p][j].row == want.exchanges[l].loc_row[p][j]);
      }
    }
  rf_coop_free(&want);

  // contract violations throw InputError (graph.hpp:48-52, coop.cpp:75-81)
  bool threw = false;
  try {
    cb::expand(g, {static_cast<uint32_t>(n)}, 1, cfg, {});
  } catch (const cb::InputError&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    std::vector<std::vector<uint32_t>> bad(4);
    for (uint32_t v = 0; v < n; ++v)
      if (owner[v] == 1) {
        bad[0].push_back(v);
        break;
      }
    cb::coop_sample(g, pm, bad, 1, cfg, {});
  } catch (const cb::InputError&) {
    threw = true;
  }
  CHECK(threw);

  // LruCache == reference LruCache, access by access (cache.cpp:12-27)
  {
    cb::LruCache c(7, n);
    void* r = rf_lru_new(7);
    std::vector<uint32_t> keys;
    uint64_t x = 1;
    for (int i = 0; i < 3000; ++i) {
      x = x * 6364136223846793005ULL + 1442695040888963407ULL;
      keys.push_back(static_cast<uint32_t>((x >> 33) % 23));
    }
    const auto got_m = c.access_all(keys);
    uint64_t misses = 0;
    for (std::size_t i = 0; i < keys.size(); ++i) {
      const int miss = rf_lru_access(r, keys[i]);
      misses += miss;
      CHECK((got_m[i] == cb::CacheOutcome::kMiss) == (miss != 0));
    }
    CHECK(c.misses() == misses && c.hits() == keys.size() - misses && c.size() == 7);
    rf_lru_free(r);
  }

  // coop_train_step == reference coop_train_step (coop.cpp:438-556)
  {
    const uint32_t dim = 6, classes = 4, hidden = 5;
    auto store = cb::FeatureStore::synth(g, dim, 1, cb::Dtype::kF64, &pm);
    auto model = cb::GcnModel::init(dim, hidden, classes, 2, 2);
    cb::SamplerConfig tc;
    tc.kind = cb::SamplerKind::kLabor0;
    tc.fanout = 4;
    const auto tr = cb::coop_train_step(g, pm, per_pe, 2, tc, {1, 31, 31, 0}, model, store);
    void* rfs = rf_features_new(n, dim, classes, 1);
    double loss = 0;
    std::vector<double> gw(hidden * classes + dim * hidden);
    ob_sched ts{1, 31, 31, 0};
    CHECK(rf_train_step(rg, rfs, 0, owner.data(), 4, flat.data(), off.data(), 2, CB_LABOR0, 4,
                        &ts, hidden, 2, &loss, gw.data()) == 0);
    CHECK(std::fabs(tr.loss - loss) <= 1e-12 * std::fabs(loss));
    std::size_t o = 0;
    double err = 0, mag = 0;
    for (const auto& d : tr.grad_w)
      for (double v : d.data) {
        err = std::fmax(err, std::fabs(v - gw[o]));
        mag = std::fmax(mag, std::fabs(gw[o]));
        ++o;
      }
    CHECK(o == gw.size() && err <= 1e-12 * mag);
    rf_features_free(rfs);
  }

  // CBCS written by the reference loads into HBM (graph.cpp:216-252)
  {
    const std::string path = "/tmp/cb_test_shim.cbcs";
    CHECK(rf_save_csr(rg, path.c_str()) == 0);
    auto h = cb::Graph::load_csr(path);
    CHECK(h.num_vertices() == n);
    const auto a = cb::expand(h, seeds, 2, cfg, {1, 5, 5, 0});
    const auto b = cb::expand(g, seeds, 2, cfg, {1, 5, 5, 0});
    for (int l = 0; l < 2; ++l) CHECK(a.blocks[l].edges == b.blocks[l].edges);
    std::remove(path.c_str());
  }

  // sample_block at layers > 0 (samplers.cpp:323-338) and sample_labor0 with a
  // caller variate (samplers.cpp:305-312) == the reference's
  for (int kind : {CB_NS, CB_LABOR0})
    for (int layer : {1, 2}) {
      ob_sched s;
      rf_sched_make(1, 77, &s);
      cb::SamplerConfig cfg;
      cfg.kind = static_cast<cb::SamplerKind>(kind);
      cfg.fanout = 3;
      const auto got = cb::sample_block(g, seeds, cfg, {s.kappa, s.z1, s.z2, s.iteration}, layer);
      ob_block want{};
      CHECK(rf_sample_block(rg, seeds.data(), seeds.size(), kind, 3, &s, layer, &want) == 0);
      CHECK(same_block(got, want) && got.layer == layer);
      rf_block_free(&want);
    }
  {
    std::vector<double> table(n);
    for (uint64_t t = 0; t < n; ++t) table[t] = std::fmod(0.6180339887 * double(t * t + 3), 1.0);
    const auto got = cb::sample_labor0(g, seeds, 3, [&](uint32_t t) { return table[t]; }, 1);
    ob_block want{};
    CHECK(rf_sample_labor0(rg, seeds.data(), seeds.size(), 3, table.data(), 1, &want) == 0);
    CHECK(same_block(got, want) && got.layer == 1);
    rf_block_free(&want);
  }

  rf_graph_free(rg);
  rf_free(ip);
  rf_free(ix);
  std::printf("test_shim: %s (%d failures)\n", g_fail ? "FAIL" : "PASS", g_fail);
  return g_fail ? 1 : 0;
}
