// Device context of the C++ drop-in: see ctx.hpp.
#include "ctx.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <stdexcept>
#include <thread>
#include <tuple>

namespace coopbatch::b200 {

[[noreturn]] void raise(int rc) {
  const std::string msg = cb_last_error();
  switch (rc) {
    case CB_INPUT:
      throw InputError(msg);
    case CB_FORMAT:
      throw FormatError(msg);
    case CB_IO:
      throw IoError(msg);
    default:
      throw std::runtime_error("coopbatch (B200): " + msg);
  }
}

std::recursive_mutex& api_mutex() {
  static std::recursive_mutex m;
  return m;
}

int device() {
  static const int d = [] {
    const char* e = std::getenv("COOPBATCH_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return d;
}

namespace {

// 64-bit content hash over a byte range, 4 independent lanes (~10 GB/s per
// thread); ranges above 8 MiB are split over host threads.
std::uint64_t hash_range(const unsigned char* p, std::size_t n, std::uint64_t seed) {
  constexpr std::uint64_t kM = 0x9E3779B97F4A7C15ULL;
  std::uint64_t a = seed ^ 0x243F6A8885A308D3ULL, b = seed ^ 0x13198A2E03707344ULL,
                c = seed ^ 0xA4093822299F31D0ULL, d = seed ^ 0x082EFA98EC4E6C89ULL;
  std::size_t i = 0;
  for (; i + 32 <= n; i += 32) {
    std::uint64_t w[4];
    std::memcpy(w, p + i, 32);
    a = (a ^ w[0]) * kM;
    b = (b ^ w[1]) * kM;
    c = (c ^ w[2]) * kM;
    d = (d ^ w[3]) * kM;
    a ^= a >> 29;
    b ^= b >> 29;
    c ^= c >> 29;
    d ^= d >> 29;
  }
  std::uint64_t t = 0;
  for (std::size_t k = 0; i + k < n; ++k) t |= static_cast<std::uint64_t>(p[i + k]) << (8 * (k & 7));
  std::uint64_t h = mix64(a) ^ mix64(b + 1) ^ mix64(c + 2) ^ mix64(d + 3) ^ mix64(t ^ n);
  return h;
}

std::uint64_t content_hash(const void* data, std::size_t bytes) {
  const auto* p = static_cast<const unsigned char*>(data);
  constexpr std::size_t kChunk = 8ULL << 20;  // spread over every host thread
  if (bytes <= kChunk) return hash_range(p, bytes, 0);
  const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
  std::vector<std::uint64_t> hs(chunks);
  const std::size_t workers =
      std::max<std::size_t>(1, std::min<std::size_t>(chunks, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (std::size_t w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (std::size_t c = w; c < chunks; c += workers) {
        const std::size_t off = c * kChunk;
        hs[c] = hash_range(p + off, std::min(kChunk, bytes - off), c);
      }
    });
  for (auto& t : pool) t.join();
  return hash_range(reinterpret_cast<const unsigned char*>(hs.data()), hs.size() * 8, bytes);
}

struct GraphEntry {
  std::uint64_t id;
  const void* indptr;
  const void* indices;
  const void* weights;
  std::uint64_t n, m, nw;
  std::uint64_t hash;
  cb_graph* h;
};

struct PartEntry {
  std::uint64_t id;
  std::uint64_t graph_id;
  const void* owner;
  std::uint64_t n;
  std::uint32_t parts;
  std::uint64_t hash;
  cb_partition* h;
};

struct PlanEntry {
  std::uint64_t graph_id, part_id;
  std::uint32_t parts;
  int layers, kind;
  std::uint32_t fanout, rw_length, rw_walks;
  double rw_restart;
  std::uint64_t cap;
  cb_plan* h;
};

constexpr std::size_t kMaxGraphs = 4;
constexpr std::size_t kMaxParts = 8;
constexpr std::size_t kMaxPlans = 16;

struct Registry {
  std::list<GraphEntry> graphs;  // front = most recently used
  std::list<PartEntry> parts;
  std::list<PlanEntry> plans;
  std::uint64_t next_id = 1;

  void drop_plans_if(const std::function<bool(const PlanEntry&)>& pred) {
    for (auto it = plans.begin(); it != plans.end();) {
      if (pred(*it)) {
        cb_plan_destroy(it->h);
        it = plans.erase(it);
      } else {
        ++it;
      }
    }
  }
  void drop_parts_of(std::uint64_t gid) {
    for (auto it = parts.begin(); it != parts.end();) {
      if (it->graph_id == gid) {
        const std::uint64_t pid = it->id;
        drop_plans_if([pid](const PlanEntry& e) { return e.part_id == pid; });
        cb_partition_destroy(it->h);
        it = parts.erase(it);
      } else {
        ++it;
      }
    }
  }
  void drop_graph(std::list<GraphEntry>::iterator it) {
    const std::uint64_t gid = it->id;
    drop_plans_if([gid](const PlanEntry& e) { return e.graph_id == gid; });
    drop_parts_of(gid);
    cb_graph_destroy(it->h);
    graphs.erase(it);
  }
};

Registry& reg() {
  static Registry r;
  return r;
}

std::uint64_t graph_hash(const Graph& g) {
  std::uint64_t h = content_hash(g.indptr.data(), g.indptr.size() * 8);
  h ^= mix64(content_hash(g.indices.data(), g.indices.size() * 4) + 1);
  if (!g.weights.empty()) h ^= mix64(content_hash(g.weights.data(), g.weights.size() * 4) + 2);
  return h ^ mix64(g.num_vertices + 3);
}

GraphEntry& graph_entry(const Graph& g) {
  Registry& r = reg();
  const std::uint64_t h = graph_hash(g);
  for (auto it = r.graphs.begin(); it != r.graphs.end(); ++it) {
    if (it->indptr == g.indptr.data() && it->indices == g.indices.data() &&
        it->weights == g.weights.data() && it->n == g.num_vertices && it->m == g.indices.size() &&
        it->nw == g.weights.size()) {
      if (it->hash == h) {
        r.graphs.splice(r.graphs.begin(), r.graphs, it);
        return r.graphs.front();
      }
      r.drop_graph(it);  // same storage, new contents
      break;
    }
  }
  if (g.indptr.size() != g.num_vertices + 1)
    throw InputError("graph: indptr must hold num_vertices + 1 entries");
  cb_graph* gh = nullptr;
  check(cb_graph_create_from_csr(g.indptr.data(), g.indices.data(), g.num_vertices,
                                 g.indices.size(), device(), &gh));
  if (!g.weights.empty()) {
    const int rc = cb_graph_set_weights(gh, g.weights.data());
    if (rc != CB_OK) {
      cb_graph_destroy(gh);
      raise(rc);
    }
  }
  while (r.graphs.size() >= kMaxGraphs) r.drop_graph(std::prev(r.graphs.end()));
  r.graphs.push_front({r.next_id++, g.indptr.data(), g.indices.data(), g.weights.data(),
                       g.num_vertices, g.indices.size(), g.weights.size(), h, gh});
  return r.graphs.front();
}

PartEntry& part_entry(const GraphEntry& ge, const Graph& g, const PartitionMap& pm) {
  Registry& r = reg();
  const std::uint64_t h = content_hash(pm.owner.data(), pm.owner.size() * 4) ^ pm.num_parts;
  for (auto it = r.parts.begin(); it != r.parts.end(); ++it) {
    if (it->graph_id == ge.id && it->owner == pm.owner.data() && it->n == pm.owner.size() &&
        it->parts == pm.num_parts) {
      if (it->hash == h) {
        r.parts.splice(r.parts.begin(), r.parts, it);
        return r.parts.front();
      }
      const std::uint64_t pid = it->id;
      r.drop_plans_if([pid](const PlanEntry& e) { return e.part_id == pid; });
      cb_partition_destroy(it->h);
      r.parts.erase(it);
      break;
    }
  }
  validate_partition(pm, g.num_vertices);
  cb_partition* ph = nullptr;
  check(cb_partition_create(ge.h, pm.owner.data(), pm.num_parts, &ph));
  while (r.parts.size() >= kMaxParts) {
    auto last = std::prev(r.parts.end());
    const std::uint64_t pid = last->id;
    r.drop_plans_if([pid](const PlanEntry& e) { return e.part_id == pid; });
    cb_partition_destroy(last->h);
    r.parts.erase(last);
  }
  r.parts.push_front({r.next_id++, ge.id, pm.owner.data(), pm.owner.size(), pm.num_parts, h, ph});
  return r.parts.front();
}

}  // namespace

cb_graph* graph_handle(const Graph& g) { return graph_entry(g).h; }

cb_partition* partition_handle(const Graph& g, const PartitionMap& pm) {
  return part_entry(graph_entry(g), g, pm).h;
}

cb_plan* plan_for(const PlanSpec& s) {
  Registry& r = reg();
  const SamplerConfig& cfg = *s.cfg;
  GraphEntry& ge = graph_entry(*s.g);
  // (a changed owner array drops the plans of the old one here)
  PartEntry* pe = s.pm ? &part_entry(ge, *s.g, *s.pm) : nullptr;
  const std::uint64_t pid = pe ? pe->id : 0;
  std::uint64_t cap = 64;
  while (cap < s.max_seeds) cap <<= 1;
  const int kind = static_cast<int>(cfg.kind);
  const bool rw = cfg.kind == SamplerKind::kRw;
  const std::uint32_t parts = s.pm ? s.pm->num_parts : s.parts;
  for (auto it = r.plans.begin(); it != r.plans.end(); ++it) {
    if (it->graph_id == ge.id && it->part_id == pid && it->parts == parts &&
        it->layers == s.layers && it->kind == kind && it->fanout == cfg.fanout &&
        it->cap >= cap && it->cap <= 4 * cap &&
        (!rw || (it->rw_length == cfg.rw_length && it->rw_walks == cfg.rw_walks &&
                 it->rw_restart == cfg.rw_restart))) {
      r.plans.splice(r.plans.begin(), r.plans, it);
      cb_plan* pl = r.plans.front().h;
      check(cb_plan_set_layer_base(pl, 0));
      check(cb_plan_set_variate_source(pl, nullptr));
      if (cfg.kind == SamplerKind::kLabor0) check(cb_plan_set_variate_table(pl, nullptr, 0));
      return pl;
    }
  }
  std::vector<std::uint32_t> fo(s.layers, cfg.fanout);
  cb_plan* pl = nullptr;
  if (s.pm) {
    check(cb_plan_create(ge.h, pe->h, s.layers, kind, fo.data(), cap, &pl));
  } else if (parts > 1) {
    check(cb_plan_create_parts(ge.h, parts, s.layers, kind, fo.data(), cap, &pl));
  } else {
    check(cb_plan_create(ge.h, nullptr, s.layers, kind, fo.data(), cap, &pl));
  }
  if (rw) {
    const int rc = cb_plan_set_rw(pl, cfg.rw_length, cfg.rw_restart, cfg.rw_walks);
    if (rc != CB_OK) {
      cb_plan_destroy(pl);
      raise(rc);
    }
  }
  while (r.plans.size() >= kMaxPlans) {
    cb_plan_destroy(r.plans.back().h);
    r.plans.pop_back();
  }
  r.plans.push_front({ge.id, pid, parts, s.layers, kind, cfg.fanout, cfg.rw_length, cfg.rw_walks,
                      cfg.rw_restart, cap, pl});
  return pl;
}

cb_sched to_sched(const SeedSchedule& s) { return {s.kappa, s.z1, s.z2, s.iteration}; }

cb_variates to_variates(const VariateSource& v) {
  return {v.z1, v.z2, v.cos_c, v.sin_c, v.smoothed ? 1 : 0};
}

void layer_sizes(cb_plan* pl, std::uint32_t part, int l, std::uint64_t sz[6]) {
  check(cb_layer_sizes(pl, part, l, sz));
}

BipartiteBlock download_block(cb_plan* pl, std::uint32_t part, int l, int layer_label) {
  std::uint64_t sz[6];
  layer_sizes(pl, part, l, sz);
  BipartiteBlock b;
  b.layer = layer_label;
  b.dst_vertices.resize(sz[0]);
  b.src_vertices.resize(sz[1]);
  b.edges.resize(sz[2]);
  b.dst_pos_in_src.resize(sz[0]);
  static_assert(sizeof(std::pair<std::uint32_t, std::uint32_t>) == 8,
                "edge pairs are downloaded as packed (src_idx, dst_idx) u32 pairs");
  check(cb_download_block(pl, part, l, b.dst_vertices.data(), b.src_vertices.data(),
                          reinterpret_cast<std::uint32_t*>(b.edges.data()),
                          b.dst_pos_in_src.data()));
  return b;
}

namespace {

struct HostTableEntry {
  const double* rows;
  std::uint64_t n_rows;
  std::uint32_t dim;
  std::uint64_t fp;
  cb_features* f;
};

// 64 words spread over the table, plus its shape
std::uint64_t sampled_fingerprint(const double* rows, std::uint64_t n) {
  std::uint64_t h = mix64(n);
  if (n == 0) return h;
  for (std::uint64_t i = 0; i < 64; ++i) {
    std::uint64_t w;
    std::memcpy(&w, rows + (i * (n - 1)) / 63, 8);
    h = mix64(h ^ w ^ (i << 56));
  }
  return h;
}

std::list<HostTableEntry>& host_tables() {
  static std::list<HostTableEntry> t;
  return t;
}

}  // namespace

cb_features* cached_host_table(const double* rows, std::uint64_t n_rows, std::uint32_t dim) {
  auto& ts = host_tables();
  const std::uint64_t fp = sampled_fingerprint(rows, n_rows * dim);
  for (auto it = ts.begin(); it != ts.end(); ++it) {
    if (it->rows == rows && it->n_rows == n_rows && it->dim == dim) {
      if (it->fp == fp) {
        ts.splice(ts.begin(), ts, it);
        return ts.front().f;
      }
      cb_features_destroy(it->f);  // other contents at the same address
      ts.erase(it);
      break;
    }
  }
  while (ts.size() >= 4) {
    cb_features_destroy(ts.back().f);
    ts.pop_back();
  }
  cb_features* f = nullptr;
  check(cb_features_wrap_host(device(), n_rows, dim, CB_F64, rows, &f));
  ts.push_front({rows, n_rows, dim, fp, f});
  return f;
}

MappedHostTable::MappedHostTable(const double* rows, std::uint64_t n_rows, std::uint32_t dim) {
  // small tables are copied to HBM (cheaper than pinning their pages)
  if (n_rows * dim * 8 <= (16ULL << 20))
    check(cb_features_from_host(device(), n_rows, dim, CB_F64, rows, &f_));
  else
    check(cb_features_wrap_host(device(), n_rows, dim, CB_F64, rows, &f_));
}

MappedHostTable::~MappedHostTable() { cb_features_destroy(f_); }

}  // namespace coopbatch::b200
