// End to end through the C++ drop-in (libcoopbatch_core_b200.so): the
// reference's own API and value types, host in, host out -- a sampler caller
// that never sees the C-ABI. Per step: coopbatch::expand (3-layer LABOR-0,
// fanout 10) over a host coopbatch::Graph, then FeatureStore::load_rows of the
// last layer's input vertices (the reference's f64 rows, read in place from
// the host table by the device), both returned as the reference's host
// objects (LayerStack, FeatureMatrix). Prints one JSON line.
//   _build/dropin_bench [n m dim steps]   (tests/cpp/Makefile builds it)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "coopbatch/coop.hpp"
#include "coopbatch/rng.hpp"
#include "coopbatch/samplers.hpp"
#include "coopbatch_cuda.h"

using namespace coopbatch;

int main(int argc, char** argv) {
  const std::uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 2449029ULL;
  const std::uint64_t m = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 61859140ULL;
  const std::uint32_t dim = argc > 3 ? std::atoi(argv[3]) : 100;
  const int steps = argc > 4 ? std::atoi(argv[4]) : 40;
  const int warmup = 3, L = 3;
  const std::uint32_t b = 1024;
  // the graph: the bench's R-MAT, generated on the device and downloaded into
  // the reference's host Graph (the drop-in uploads it once and caches it)
  cb_graph* dg = nullptr;
  if (cb_graph_generate_rmat(n, m, 42, 0, &dg) != CB_OK) {
    std::printf("{\"error\": \"%s\"}\n", cb_last_error());
    return 1;
  }
  Graph g;
  g.num_vertices = n;
  g.indptr.resize(n + 1);
  g.indices.resize(m);
  cb_graph_download(dg, g.indptr.data(), g.indices.data());
  cb_graph_destroy(dg);
  const FeatureStore fs = FeatureStore::synth(n, dim, 2, 7);
  SamplerConfig cfg;
  cfg.kind = SamplerKind::kLabor0;
  cfg.fanout = 10;
  SeedSchedule sched = SeedSchedule::make(1, 1234);
  std::vector<VertexId> seeds(b);
  double rows = 0, edges = 0, t_expand = 0, t_rows = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < warmup + steps; ++s) {
    if (s == warmup) t0 = std::chrono::steady_clock::now();
    for (std::uint32_t i = 0; i < b; ++i)
      seeds[i] = static_cast<VertexId>(hash_bits(1234, {static_cast<std::uint64_t>(s), i}) % n);
    const auto ta = std::chrono::steady_clock::now();
    const LayerStack st = expand(g, seeds, L, cfg, sched);
    const auto tb = std::chrono::steady_clock::now();
    const FeatureMatrix fm = fs.load_rows(st.input_vertices());
    const auto tc = std::chrono::steady_clock::now();
    if (s >= warmup) {
      t_expand += std::chrono::duration<double>(tb - ta).count();
      t_rows += std::chrono::duration<double>(tc - tb).count();
      rows += static_cast<double>(fm.rows());
      for (const auto& blk : st.blocks) edges += static_cast<double>(blk.edges.size());
    }
    sched = schedule_advance(sched);
  }
  const double dt =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf(
      "{\"seeds_per_s\": %.1f, \"ms_per_step\": %.4f, \"steps\": %d, \"rows_per_step\": %.1f, "
      "\"edges_per_step\": %.1f, \"row_bytes\": %u, \"graph\": [%llu, %llu], "
      "\"ms_expand\": %.3f, \"ms_load_rows\": %.3f}\n",
      steps * static_cast<double>(b) / dt, 1e3 * dt / steps, steps, rows / steps, edges / steps,
      dim * 8, static_cast<unsigned long long>(n), static_cast<unsigned long long>(m),
      1e3 * t_expand / steps, 1e3 * t_rows / steps);
  return 0;
}
