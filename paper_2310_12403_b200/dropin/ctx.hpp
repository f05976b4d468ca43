// Device context of the C++ drop-in (libcoopbatch_dropin_b200.so).
//
// The drop-in defines the reference's hot-path functions (samplers.hpp,
// coop.hpp, cache.hpp of /root/reference/proj/include/coopbatch, unchanged)
// over the C-ABI of libcoopbatch_b200.so. The reference passes host objects
// (const Graph&, const PartitionMap&, FeatureStore with host rows); this
// context keeps their device images so repeated calls reuse them:
//   * one cb_graph per distinct CSR (keyed by data pointers + sizes, verified
//     against a content hash on every call: the reference's Graph is a plain
//     value type whose storage may be reused by a different graph);
//   * one cb_partition per distinct owner array (same keying);
//   * an LRU of sampling plans keyed by graph, partition, shape and a
//     power-of-two seed capacity, instead of a plan per call.
// All entry points serialise on one mutex (the reference runs some of them
// from parallel_for worker threads, analysis.cpp:93).
#pragma once

#include <cstdint>
#include <mutex>
#include <span>
#include <string>
#include <vector>

#include "coopbatch/cache.hpp"
#include "coopbatch/coop.hpp"
#include "coopbatch/partition.hpp"
#include "coopbatch/samplers.hpp"
#include "coopbatch_cuda.h"

namespace coopbatch::b200 {

// C-ABI status -> the reference's exception types (common.hpp:12-31).
[[noreturn]] void raise(int rc);
inline void check(int rc) {
  if (rc != CB_OK) raise(rc);
}

std::recursive_mutex& api_mutex();
using Lock = std::lock_guard<std::recursive_mutex>;
int device();

// Device images of host inputs.
cb_graph* graph_handle(const Graph& g);
cb_partition* partition_handle(const Graph& g, const PartitionMap& pm);

// Sampling plans. parts > 1 without pm: independent parts (indep mode).
struct PlanSpec {
  const Graph* g = nullptr;
  const PartitionMap* pm = nullptr;
  std::uint32_t parts = 1;
  int layers = 1;
  const SamplerConfig* cfg = nullptr;
  std::uint64_t max_seeds = 1;
};
cb_plan* plan_for(const PlanSpec& s);

cb_sched to_sched(const SeedSchedule& s);
cb_variates to_variates(const VariateSource& v);

// Results of part `part`, layer `l` of the plan's last batch.
BipartiteBlock download_block(cb_plan* pl, std::uint32_t part, int l, int layer_label);
void layer_sizes(cb_plan* pl, std::uint32_t part, int l, std::uint64_t sz[6]);

// Host rows mapped into the device for the duration of one call: the
// reference's FeatureStore keeps its f64 rows in host memory (coop.hpp:140-155);
// the device reads them in place over the host link (the paper's storage
// channel) instead of copying the table.
// A large host f64 table kept registered (pinned, mapped, read in place)
// across calls, keyed by (address, rows, dim) and a sampled fingerprint (a
// table freed and reallocated at the same address with other contents is
// re-registered). Rows are read in place, so writes to a registered table are
// seen by the next call. (Registering 2 GB of pages per call cost ~0.3 s.)
cb_features* cached_host_table(const double* rows, std::uint64_t n_rows, std::uint32_t dim);

class MappedHostTable {
 public:
  MappedHostTable(const double* rows, std::uint64_t n_rows, std::uint32_t dim);
  ~MappedHostTable();
  MappedHostTable(const MappedHostTable&) = delete;
  MappedHostTable& operator=(const MappedHostTable&) = delete;
  cb_features* get() const { return f_; }

 private:
  cb_features* f_ = nullptr;
};

}  // namespace coopbatch::b200
