// Internal header of the C-ABI translation units (capi*.cu): handle
// definitions, the error guard, device arenas, and the orchestration helpers
// of capi.cu that the cache / peer-exchange / training-step units reuse.
// Nothing here crosses the C-ABI (include/coopbatch_cuda.h).
#pragma once
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/coopbatch_cuda.h"
#include "cb_internal.h"
#include "exchange.h"
#include "gather.h"
#include "dist.h"
#include "cache.h"
#include "clock_cache.h"
#include "train.h"

using namespace cb;
using cbdev::Variates;

using namespace cb;
using cbdev::Variates;

namespace cb {
namespace capi {

extern thread_local std::string g_err;

// NVTX range per host-side stage (nsys / ncu --nvtx); free without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return CB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return CB_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CB_INTERNAL;
  }
}

struct Arena {
  std::vector<void*> ptrs;
  template <typename T>
  T* alloc(uint64_t count) {
    void* p = nullptr;
    CB_CUDA(cudaMalloc(&p, std::max<uint64_t>(count, 1) * sizeof(T) + 64));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  ~Arena() { release(); }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    CB_CUDA(cudaGetDevice(&prev));
    if (prev != dev) CB_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a != 0 && b > UINT64_MAX / a) return UINT64_MAX;
  return a * b;
}

}  // namespace capi
}  // namespace cb
using namespace cb::capi;

// ------------------------------------------------------------------ handles --
struct cb_graph {
  DeviceGraph g;
  std::unique_ptr<Arena> weights_mem;  // g.weights (RW on weighted graphs)
  ~cb_graph() {
    if (g.indptr) cudaFree(g.indptr);
    if (g.indices) cudaFree(g.indices);
  }
};

struct cb_partition {
  int device = 0;
  uint64_t n = 0;
  uint32_t parts = 1;
  Arena mem;
  uint32_t* owner = nullptr;    // [n]
  uint32_t* row_map = nullptr;  // [n] global table row of v (shard-major)
  uint32_t* members = nullptr;  // [n] vertex of each global row
  std::vector<uint64_t> shard_off;  // [parts+1]
};

struct cb_features {
  int device = 0;
  uint32_t dim = 0;
  int dtype = CB_F32;
  uint64_t seed = 0;            // FeatureStore::synth seed (values and labels)
  uint64_t row_bytes = 0;
  uint64_t n_rows = 0;
  Arena mem;
  void* table = nullptr;
  uint32_t* row_map = nullptr;  // nullptr = identity (P = 1)
  uint64_t shard_rows = 0;      // rows actually held (sharded tables)
  uint64_t shard_r0 = 0;        // first global row of the shard
  void* host_base = nullptr;    // pinned mapped host copy (host tier) or nullptr
  void* hbm_table = nullptr;    // the HBM table while the host tier is active
  uint32_t* labels = nullptr;   // [n_rows] explicit labels (cb_features_set_labels) or null
  void* registered = nullptr;   // caller's host rows mapped in place (cb_features_wrap_host)
  // cb_op_load_rows scratch, reused across calls (a cudaMalloc / cudaFree and
  // a stream per call cost more than the gather)
  cudaStream_t op_stream = nullptr;
  void* op_ids = nullptr;
  void* op_out = nullptr;
  uint64_t op_cap = 0;
  ~cb_features() {
    if (host_base) cudaFreeHost(host_base);
    if (registered) cudaHostUnregister(registered);
    if (op_ids) cudaFree(op_ids);
    if (op_out) cudaFree(op_out);
    if (op_stream) cudaStreamDestroy(op_stream);
  }
};

struct cb_ccache {
  std::unique_ptr<ClockCache> cc;
  cudaStream_t stream = nullptr;
  ~cb_ccache() {
    if (stream) cudaStreamDestroy(stream);
  }
};

struct cb_cache {
  std::unique_ptr<DeviceLru> lru;
  cudaStream_t stream = nullptr;
  ~cb_cache() {
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace cb {
namespace capi {

struct PeWork {
  std::vector<LayerBufs> L;
  Bitmap bm[2];
  Sync sync;
  std::vector<uint32_t*> loc_part, loc_row;  // [layer] cap_src
  uint32_t* owner_final = nullptr;            // coop: S^L_p
  uint64_t cap_final = 0;
  void* rows = nullptr;
  uint64_t cap_rows = 0;
  uint64_t rows_row_bytes = 0;
};

// Multi-process peer exchange state (one part per rank): this rank's
// IPC-exportable exchange region (2 layer slots of bitmap + summary + word
// ranks) and every rank's mapping of it.
struct PxState {
  uint32_t rank = 0, world = 0;
  const uint32_t* owner = nullptr;  // pm->owner (device)
  void* region = nullptr;           // local cudaMalloc, exported
  uint64_t region_bytes = 0;
  static constexpr int kSlots = 4;  // eager steps use 0/1; captured steps all 4
  Bitmap slot[kSlots];              // local views of the region
  PxPeers peers[kSlots];            // per slot, every rank's pointers
  std::vector<void*> opened;        // IPC mappings to close
  unsigned long long* send = nullptr;  // [L * world] this rank's send_counts rows
  uint64_t layer_ctr = 0;           // slot of a layer = ctr & 1 (alternates across batches)
  std::vector<int> slot_of;         // [L]
  // features: virtual bases of every rank's shard (device array) + mappings
  const unsigned char** d_fbase = nullptr;
  std::vector<const unsigned char*> fbase;
  std::vector<void*> fopened;
  uint64_t frow_bytes = 0;
  // owner staging (cb_px_setup_staging): the owner's rows of its set S^L_q
  // staged in an exported buffer, pulled by the requesters; optional cache
  cb_cache* cache = nullptr;
  cb_ccache* ccache = nullptr;  // CLOCK cache in front of the owner's staging (capturable)
  const cb_features* stage_store = nullptr;
  // requester-side cache (cb_px_set_requester_cache): rows owned by other
  // ranks; compaction buffers of the remote requests
  cb_cache* rcache = nullptr;
  uint32_t* r_ids = nullptr;
  uint32_t* r_pos = nullptr;
  const void** r_miss = nullptr;
  void* r_rows = nullptr;
  unsigned long long* r_n = nullptr;
  uint64_t r_cap = 0, r_row_bytes = 0;
  uint64_t r_last[3] = {0, 0, 0};  // last step: remote rows, hits, misses
  void* rstage = nullptr;
  uint64_t rstage_rows = 0;
  const unsigned char** d_rstage = nullptr;  // [kMaxParts] every rank's staging
  std::vector<const unsigned char*> rstage_of;
  std::vector<void*> ropened;
  // device barrier: flag array at region + flag_off on every rank
  uint64_t flag_off = 0;
  uint32_t* bar_ctr = nullptr;  // [0] epoch counter, [1] timeout flag
  PxBarrier bar{};
  // the captured step: graph i % n_exec for replay i (the exchange slots
  // rotate mod 4 over the layers, the barrier value alternates 1/2)
  cudaGraphExec_t exec[4] = {nullptr, nullptr, nullptr, nullptr};
  int n_exec = 0;
  uint64_t replays = 0;
  bool eager_since_capture = false;
  bool memop = false;  // captured barriers: signal kernel + cuStreamWaitValue32
  uint64_t cap_seeds = 0;
  bool cap_rows = false, cap_smooth = false;
  uint64_t cap_launches = 0;
  void drop_graphs() {
    for (auto& e : exec) {
      if (e) cudaGraphExecDestroy(e);
      e = nullptr;
    }
    n_exec = 0;
  }
  ~PxState() {
    drop_graphs();
    for (void* p : ropened) cudaIpcCloseMemHandle(p);
    if (rstage) cudaFree(rstage);
    for (void* p : {static_cast<void*>(r_ids), static_cast<void*>(r_pos),
                    static_cast<void*>(r_miss), r_rows, static_cast<void*>(r_n)})
      if (p) cudaFree(p);
    if (d_rstage) cudaFree(d_rstage);
    if (bar_ctr) cudaFree(bar_ctr);
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    for (void* p : fopened) cudaIpcCloseMemHandle(p);
    if (region) cudaFree(region);
    if (send) cudaFree(send);
    if (d_fbase) cudaFree(d_fbase);
  }
};

}  // namespace capi
}  // namespace cb

struct cb_plan {
  int device = 0;
  const cb_graph* g = nullptr;
  const cb_partition* pm = nullptr;
  uint32_t P = 1;
  int L = 1;
  int kind = CB_LABOR0;
  std::vector<uint32_t> fanouts;
  uint64_t max_seeds = 0;
  double grow = 1.0;
  cudaStream_t stream = nullptr;
  Arena mem;       // capacity-dependent buffers
  Arena rows_mem;  // gathered rows
  std::vector<PeWork> pe;
  LayerMeta* meta = nullptr;                // [P*(L+1)]
  unsigned long long* send_counts = nullptr;  // [L*P*P]
  Variates* var = nullptr;
  double* ext_vtab = nullptr;  // caller variate table r_t (sample_labor0), n entries
  int layer_base = 0;          // block l hashes as layer l + layer_base (sample_block at any layer)
  // captured sample + gather graph: the last layer's relabel of part 0 is
  // launched fused with the gather (launch_relabel_gather)
  bool defer_relabel = false;
  bool has_deferred = false;
  cb::RelabelArgs deferred{};
  uint64_t deferred_work = 0;
  uint32_t* seeds = nullptr;
  uint64_t seeds_cap = 0;
  int mode = -1;          // mode of the last batch
  int dirty_mode = -1;    // mode whose final bitmap still holds bits (-1: clean)
  uint32_t dist_world = 0;  // >0: one part of a multi-process cooperative step
  unsigned long long* scratch = nullptr;  // small device counters (dist ops)
  bool smooth = false;    // kernels of the last enqueue used smoothed variates
  bool trace_on = false;   // globaltimer stamps per CTA (debug, CB_TRACE=1)
  unsigned long long* trace = nullptr;  // [kTraceSlots]
  std::vector<cudaEvent_t>* prof = nullptr;  // per-launch events (cb_plan_profile)
  bool prof_external = false;                 // record as graph event nodes
  std::vector<cudaEvent_t> graph_events;      // of exec_prof
  cudaGraphExec_t exec_prof = nullptr;
  bool cap_smooth = false;
  bool have_batch = false;
  bool have_rows = false;
  std::optional<Variates> var_source;  // cb_plan_set_variate_source override
  // smoothed decisions inside the guard band, resolved on the host
  // (resolve_batch in capi.cu; DESIGN.md §Smoothed variates)
  double guard = cbdev::kGuard;
  int perturb = 0;
  bool strict = true;
  cbdev::Resolve* d_rs = nullptr;
  uint64_t* rs_k1 = nullptr;
  uint64_t* rs_k2 = nullptr;
  double* rs_val = nullptr;
  uint32_t rs_cap = 0;
  cbdev::ResolvePend* rs_pend = nullptr;
  unsigned long long* rs_npend = nullptr;
  uint64_t rs_resolved = 0, rs_reruns = 0;  // of the last cb_sample_sync
  uint64_t rows_limit = 0;    // row-buffer cap in rows (0: the src capacity)
  void* meta_host = nullptr;  // pinned staging of cb_plan_result_copy's counts
  void* pack = nullptr;       // cb_plan_result_pack's packed result (device)
  uint64_t pack_bytes = 0;
  uint64_t pack_version = ~0ULL;  // plan->batches when packed
  uint32_t pack_part = 0;
  uint64_t batches = 0;  // device epoch bumps (count_epoch_bumps)
  uint64_t launches = 0;  // kernels enqueued by the last cb_sample (+ cb_gather)
  double* vtab = nullptr;  // smoothed LABOR r_t table [n] (nullptr: per position)
  uint32_t rw_length = 3, rw_walks = 100;  // samplers.hpp:19-22 defaults
  double rw_restart = 0.5;
  std::unique_ptr<PxState> px;  // multi-process peer exchange (dist plans)
  std::vector<uint64_t> seeds_off;
  // CUDA graphs of one batch (sample) and its gather, replayed per step
  cudaGraphExec_t exec_sample = nullptr;
  cudaGraphExec_t exec_gather = nullptr;
  cudaGraphExec_t exec_all = nullptr;  // sample + gather in one graph
  int cap_mode = -1;
  std::vector<uint64_t> cap_off;
  uint64_t cap_launches_sample = 0, cap_launches_gather = 0, cap_launches_all = 0;

  void drop_graphs() {
    if (exec_sample) cudaGraphExecDestroy(exec_sample);
    if (exec_gather) cudaGraphExecDestroy(exec_gather);
    if (exec_all) cudaGraphExecDestroy(exec_all);
    if (exec_prof) cudaGraphExecDestroy(exec_prof);
    for (auto e : graph_events) cudaEventDestroy(e);
    graph_events.clear();
    exec_sample = exec_gather = exec_all = exec_prof = nullptr;
  }
  // parts of a multi-part plan run concurrently, one stream each, joined
  // before every cross-part step (part_st empty: one after another)
  std::vector<cudaStream_t> part_st;
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_join;
  bool part_concurrent = false;
  ~cb_plan() {
    drop_graphs();
    for (cudaStream_t s : part_st) cudaStreamDestroy(s);
    for (cudaEvent_t e : ev_join) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ext_vtab) cudaFree(ext_vtab);
    if (meta_host) cudaFreeHost(meta_host);
    if (pack) cudaFree(pack);
    for (void* q : {static_cast<void*>(d_rs), static_cast<void*>(rs_k1),
                    static_cast<void*>(rs_k2), static_cast<void*>(rs_val),
                    static_cast<void*>(rs_pend), static_cast<void*>(rs_npend)})
      if (q) cudaFree(q);
  }

  LayerMeta* meta_at(uint32_t p, int l) { return meta + p * (L + 1) + l; }
  bool coop_active() const { return mode == CB_MODE_COOP && P > 1; }
  bool own_dst() const { return coop_active() || dist_world > 0; }
};


namespace cb {
namespace capi {
// capi.cu helpers shared with the other C-ABI translation units
Variates make_variates(const cb_sched* s);
bool smooth_of(const cb_plan* pl, const cb_sched* s);
void upload_variates(cb_plan* pl, const cb_sched* s, uint32_t n_sched, cudaStream_t st);
ExtractArgs extract_args(PeWork& w, const Bitmap& bm, const Bitmap* zero_bm, uint32_t* out,
                         uint64_t cap, unsigned long long* c1, unsigned long long* c2,
                         int ticket, int slot);
RelabelArgs relabel_args(const Bitmap& bm, const LayerBufs& b, const uint32_t* D,
                         const LayerMeta* me);
uint64_t enqueue_layer(cb_plan* pl, PeWork& w, uint32_t p, int l, const uint32_t* D,
                       uint64_t cap_dst, uint64_t n_dst_param, Bitmap& set_bm,
                       const RelabelArgs& fused, uint64_t fused_work, bool smooth,
                       const ExtractArgs& ex, cudaStream_t stream = nullptr);
void check_overflow(cb_plan* pl, bool strict_smooth = true);
const LayerMeta host_meta(cb_plan* pl, uint32_t p, int l);
void require_batch(const cb_plan* pl, uint32_t p, int l);
void count_epoch_bumps(cb_plan* pl, cudaStream_t st, uint64_t bumps);
// Arbitrary ids may be gathered only from a table that holds every row: a
// single-part shard (cb_features_synth_shard) keeps n_rows = n for its
// row_map but allocates only its own rows.
inline void require_full_table(const cb_features* f) {
  require(f->shard_rows == 0,
          "this gather needs a full feature table (got a single-part shard)");
}
// Sizes the plan's row buffers for f. any_row: the gather reads f at any
// vertex (not only this shard's own rows).
void prepare_rows(cb_plan* pl, const cb_features* f, bool any_row = true);
void enqueue_gather(cb_plan* pl, const cb_features* f);
}  // namespace capi
}  // namespace cb
