// libcoopbatch_b200 C-ABI (include/coopbatch_cuda.h) and the C++ orchestrator
// behind it: handle lifetimes, capacity planning, and the per-batch launch
// sequence of expand / indep_sample / coop_sample (samplers.cpp:340-354,
// coop.cpp:68-119) and the fused load_rows + all_to_all_forward gather
// (coop.cpp:145-159, 378-388). Every launch is asynchronous on the plan's
// stream; counts stay on the device (LayerMeta) so a batch never waits on the
// host. Contract violations raise cb::Error(kInput) -> CB_INPUT, mirroring
// coopbatch::InputError (common.hpp:12-15).
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/coopbatch_cuda.h"
#include "cb_internal.h"
#include "exchange.h"
#include "gather.h"
#include "dist.h"
#include "cache.h"
#include "train.h"

using namespace cb;
using cbdev::Variates;

namespace {

thread_local std::string g_err;

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

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a != 0 && b > UINT64_MAX / a) return UINT64_MAX;
  return a * b;
}

}  // namespace

namespace cb {
std::atomic<unsigned long long> g_kernel_launches{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CB_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}
}  // namespace cb

// ------------------------------------------------------------------ handles --
struct cb_graph {
  DeviceGraph g;
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
  ~cb_features() {
    if (host_base) cudaFreeHost(host_base);
  }
};

struct cb_cache {
  std::unique_ptr<DeviceLru> lru;
  cudaStream_t stream = nullptr;
  ~cb_cache() {
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

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
  Bitmap slot[2];                   // local views of the region
  PxPeers peers[2];                 // per slot, every rank's pointers
  std::vector<void*> opened;        // IPC mappings to close
  unsigned long long* send = nullptr;  // [L * world] this rank's send_counts rows
  uint64_t layer_ctr = 0;           // slot of a layer = ctr & 1 (alternates across batches)
  std::vector<int> slot_of;         // [L]
  // features: virtual bases of every rank's shard (device array) + mappings
  const unsigned char** d_fbase = nullptr;
  std::vector<const unsigned char*> fbase;
  std::vector<void*> fopened;
  uint64_t frow_bytes = 0;
  ~PxState() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    for (void* p : fopened) cudaIpcCloseMemHandle(p);
    if (region) cudaFree(region);
    if (send) cudaFree(send);
    if (d_fbase) cudaFree(d_fbase);
  }
};

}  // namespace

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
  uint64_t batches = 0;
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
  uint64_t cap_launches_sample = 0, cap_launches_gather = 0;

  void drop_graphs() {
    if (exec_sample) cudaGraphExecDestroy(exec_sample);
    if (exec_gather) cudaGraphExecDestroy(exec_gather);
    if (exec_all) cudaGraphExecDestroy(exec_all);
    if (exec_prof) cudaGraphExecDestroy(exec_prof);
    for (auto e : graph_events) cudaEventDestroy(e);
    graph_events.clear();
    exec_sample = exec_gather = exec_all = exec_prof = nullptr;
  }
  ~cb_plan() { drop_graphs(); }

  LayerMeta* meta_at(uint32_t p, int l) { return meta + p * (L + 1) + l; }
  bool coop_active() const { return mode == CB_MODE_COOP && P > 1; }
  bool own_dst() const { return coop_active() || dist_world > 0; }
};

namespace {

void make_bitmap(Arena& a, Bitmap& b, uint64_t n) {
  b.words = ceil_div(n, 32);
  b.words_padded = ceil_div(std::max<uint64_t>(b.words, 1), kExtractTileWords) * kExtractTileWords;
  b.bits = a.alloc<uint32_t>(b.words_padded);
  b.wprefix = a.alloc<uint32_t>(b.words_padded);
  CB_CUDA(cudaMemset(b.bits, 0, b.words_padded * sizeof(uint32_t)));
  if (b.words_padded > kExtractBigWords) {  // summary only where extract uses it
    b.summ = a.alloc<uint32_t>(b.words_padded / 32);
    CB_CUDA(cudaMemset(b.summ, 0, b.words_padded / 32 * sizeof(uint32_t)));
  }
}

// Capacity plan (host): upper bounds sized from the seeds and fanouts; any
// overflow is detected on the device and retried with grow *= 2.
void plan_alloc(cb_plan* pl) {
  pl->drop_graphs();
  pl->mem.release();
  pl->rows_mem.release();
  pl->have_rows = false;
  const DeviceGraph& g = pl->g->g;
  const uint64_t n = g.n, m = g.m, maxdeg = std::max<uint64_t>(g.max_degree, 1);
  const uint32_t P = pl->P;
  const int L = pl->L;
  pl->pe.assign(P, PeWork());
  for (uint32_t p = 0; p < P; ++p) {
    PeWork& w = pl->pe[p];
    w.L.resize(L);
    uint64_t cd = std::max<uint64_t>(pl->max_seeds, 1);
    uint64_t max_tiles = 2;
    for (int l = 0; l < L; ++l) {
      const uint64_t k = pl->fanouts[l];
      // scan space: layer-0 seeds may repeat, so its bound is m * grow (an
      // overflow is flagged on the device and retried with grow * 2); later
      // frontiers are unique vertex sets, so m bounds them
      const uint64_t m_grow = sat_mul(std::max<uint64_t>(m, 1),
                                      static_cast<uint64_t>(std::ceil(pl->grow)));
      const uint64_t sum_deg =
          std::min((l == 0) ? m_grow : m, sat_mul(cd, maxdeg));
      uint64_t est;
      if (pl->kind == CB_FULL) est = sum_deg;
      else if (pl->kind == CB_NS || pl->kind == CB_RW) est = sat_mul(cd, k);
      else est = sat_mul(cd, 2 * k) + 4096;
      if (pl->kind != CB_FULL) est = static_cast<uint64_t>(std::ceil(est * pl->grow));
      uint64_t cap_e = std::max<uint64_t>(1, std::min(est, sum_deg));
      if (pl->kind == CB_NS || pl->kind == CB_RW) cap_e = std::min(cap_e, sat_mul(cd, k));
      if (pl->kind == CB_RW) cap_e = std::max<uint64_t>(sat_mul(cd, k), 1);
      LayerBufs& b = w.L[l];
      b.cap_dst = cd;
      b.cap_edges = std::max<uint64_t>(cap_e, 1);
      b.cap_src = std::min(n, cd + b.cap_edges);
      if (l == 0) b.dst = nullptr;  // seeds live in pl->seeds
      else b.dst = pl->mem.alloc<uint32_t>(cd);
      b.act = pl->mem.alloc<ActRec>(cd + 1);
      const bool nsrw = pl->kind == CB_NS || pl->kind == CB_RW;
      b.out_prefix = nsrw ? pl->mem.alloc<uint64_t>(cd + 1) : nullptr;
      b.slots = nsrw ? pl->mem.alloc<uint32_t>(b.cap_edges) : nullptr;
      b.edges = pl->mem.alloc<uint2>(b.cap_edges);
      b.src = pl->mem.alloc<uint32_t>(b.cap_src);
      b.dst_pos = pl->mem.alloc<uint32_t>(cd);
      max_tiles = std::max(max_tiles, ceil_div(sum_deg, kLaborTile) + 2);
      max_tiles = std::max(max_tiles, ceil_div(cd, kFrontierTile) + 2);
      if (P > 1 || pl->dist_world > 0) {
        w.loc_part.push_back(pl->mem.alloc<uint32_t>(b.cap_src));
        w.loc_row.push_back(pl->mem.alloc<uint32_t>(b.cap_src));
      }
      // next layer's frontier: indep -> this src; coop -> owner set
      const uint64_t mult = std::max<uint64_t>(P, pl->dist_world);
      const uint64_t next = (mult > 1) ? std::min(n, sat_mul(mult, b.cap_src)) : b.cap_src;
      cd = std::max(next, b.cap_src);
    }
    w.cap_final = cd;
    w.owner_final = (P > 1 || pl->dist_world > 0) ? pl->mem.alloc<uint32_t>(cd) : nullptr;
    make_bitmap(pl->mem, w.bm[0], n);
    make_bitmap(pl->mem, w.bm[1], n);
    max_tiles = std::max(max_tiles, w.bm[0].words_padded / kExtractTileWords + 2);
    w.sync.max_tiles = max_tiles;
    for (int l = 0; l < L; ++l) {
      w.L[l].tile_first = pl->mem.alloc<uint32_t>(max_tiles + 1);
      CB_CUDA(cudaMemset(w.L[l].tile_first, 0, (max_tiles + 1) * 4));
    }
    w.sync.epoch = pl->mem.alloc<unsigned>(1);
    w.sync.tickets = pl->mem.alloc<unsigned>(2 * Sync::kMaxTickets);
    CB_CUDA(cudaMemset(w.sync.tickets, 0, 2 * Sync::kMaxTickets * sizeof(unsigned)));
    w.sync.overflow = pl->mem.alloc<unsigned>(1);
    w.sync.keep_words = pl->mem.alloc<uint32_t>(max_tiles * kLaborTile / 32 + 1);
    w.sync.status_a = pl->mem.alloc<unsigned long long>(max_tiles);
    w.sync.status_b = pl->mem.alloc<unsigned long long>(max_tiles);
    w.sync.status_c = pl->mem.alloc<unsigned long long>(max_tiles);
    CB_CUDA(cudaMemset(w.sync.epoch, 0, sizeof(unsigned)));
    CB_CUDA(cudaMemset(w.sync.status_a, 0, max_tiles * 8));
    CB_CUDA(cudaMemset(w.sync.status_b, 0, max_tiles * 8));
    CB_CUDA(cudaMemset(w.sync.status_c, 0, max_tiles * 8));
  }
  // kept-edge stage: parts run one after another on the plan stream, so one
  // buffer (the largest scan space) serves all of them
  uint64_t stage_tiles = 0;
  for (const PeWork& w : pl->pe) stage_tiles = std::max(stage_tiles, w.sync.max_tiles);
  uint2* stage = pl->mem.alloc<uint2>(stage_tiles * kLaborTile + 32);
  for (PeWork& w : pl->pe) w.sync.stage = stage;
  // smoothed LABOR variate table (shared by the parts like the stage)
  pl->vtab = (pl->kind == CB_LABOR0 && n <= kVtabMaxVerts) ? pl->mem.alloc<double>(n) : nullptr;
  pl->meta = pl->mem.alloc<LayerMeta>(static_cast<uint64_t>(P) * (L + 1));
  CB_CUDA(cudaMemset(pl->meta, 0, sizeof(LayerMeta) * P * (L + 1)));
  pl->send_counts = pl->mem.alloc<unsigned long long>(static_cast<uint64_t>(L) * P * P);
  pl->var = pl->mem.alloc<Variates>(1);
  pl->seeds_cap = static_cast<uint64_t>(P) * std::max<uint64_t>(pl->max_seeds, 1);
  pl->seeds = pl->mem.alloc<uint32_t>(pl->seeds_cap);
  pl->scratch = pl->mem.alloc<unsigned long long>(8);
  if (pl->trace_on) {
    pl->trace = pl->mem.alloc<unsigned long long>(kTraceSlots);
    CB_CUDA(cudaMemset(pl->trace, 0, kTraceSlots * 8));
  }
  pl->have_batch = false;
  pl->dirty_mode = -1;
  CB_CUDA(cudaDeviceSynchronize());
}

Variates make_variates(const cb_sched* s) {
  // VariateSource::from_schedule (samplers.hpp:75-93): cos/sin on the host,
  // exact 1/0 at the endpoints.
  Variates v{};
  v.z1 = s->z1;
  v.z2 = s->z2;
  double c = 0.0;
  if (s->kappa != cbdev::kKappaInf)
    c = static_cast<double>(s->iteration % s->kappa) / static_cast<double>(s->kappa);
  v.smoothed = (s->kappa != cbdev::kKappaInf && s->kappa >= 2) ? 1 : 0;
  if (c == 0.0) {
    v.cos_c = 1.0;
    v.sin_c = 0.0;
  } else if (c == 1.0) {
    v.cos_c = 0.0;
    v.sin_c = 1.0;
  } else {
    const double angle = c * 1.5707963267948966192;
    v.cos_c = std::cos(angle);
    v.sin_c = std::sin(angle);
  }
  return v;
}

void check_seeds_host(const cb_plan* pl, const uint32_t* flat, const uint64_t* off) {
  const uint64_t n = pl->g->g.n;
  for (uint32_t p = 0; p < pl->P; ++p) {
    require(off[p + 1] >= off[p], "seed offsets must be nondecreasing");
    require(off[p + 1] - off[p] <= pl->max_seeds,
            "part " + std::to_string(p) + " has more seeds than the plan's max_seeds_per_part");
    for (uint64_t i = off[p]; i < off[p + 1]; ++i)
      require(flat[i] < n, "vertex id " + std::to_string(flat[i]) + " out of range [0, " +
                               std::to_string(n) + ")");
  }
}

void check_ownership_host(const cb_plan* pl, const uint32_t* flat, const uint64_t* off) {
  // coop_sample: every seed must be owned by its claimed part (coop.cpp:75-81)
  if (pl->P <= 1) return;
  const uint64_t total = off[pl->P];
  std::vector<uint32_t> owners(total);
  std::vector<uint32_t> seeds(flat, flat + total);
  // gather owner[seed] on the device: tiny (one value per seed)
  uint32_t* d_ids = nullptr;
  uint32_t* d_out = nullptr;
  CB_CUDA(cudaMalloc(&d_ids, total * 4 + 4));
  CB_CUDA(cudaMalloc(&d_out, total * 4 + 4));
  CB_CUDA(cudaMemcpy(d_ids, seeds.data(), total * 4, cudaMemcpyHostToDevice));
  // reuse the feature gather kernel with a 4-byte "row" = owner[v]
  unsigned long long* d_cnt = nullptr;
  CB_CUDA(cudaMalloc(&d_cnt, 8));
  const unsigned long long t = total;
  CB_CUDA(cudaMemcpy(d_cnt, &t, 8, cudaMemcpyHostToDevice));
  launch_gather(pl->pm->owner, 4, 4, d_ids, d_cnt, total, nullptr, d_out, pl->stream);
  CB_CUDA(cudaStreamSynchronize(pl->stream));
  CB_CUDA(cudaMemcpy(owners.data(), d_out, total * 4, cudaMemcpyDeviceToHost));
  cudaFree(d_ids);
  cudaFree(d_out);
  cudaFree(d_cnt);
  for (uint32_t p = 0; p < pl->P; ++p)
    for (uint64_t i = off[p]; i < off[p + 1]; ++i)
      require(owners[i] == p, "coop_sample: seed " + std::to_string(flat[i]) +
                                  " is not owned by part " + std::to_string(p));
}

void prof_mark(cb_plan* pl) {
  if (!pl->prof) return;
  cudaEvent_t e;
  CB_CUDA(cudaEventCreate(&e));
  if (pl->prof_external)
    CB_CUDA(cudaEventRecordWithFlags(e, pl->stream, cudaEventRecordExternal));
  else
    CB_CUDA(cudaEventRecord(e, pl->stream));
  pl->prof->push_back(e);
}

// Which bitmap still holds bits after a batch of `mode`, and the id list
// (with its device count) that names every set word.
struct Dirty {
  uint32_t* bits = nullptr;
  uint32_t* summ = nullptr;
  const uint32_t* list = nullptr;
  const unsigned long long* count = nullptr;
  uint64_t cap = 0;
};

Dirty dirty_of(cb_plan* pl, uint32_t p, int mode) {
  Dirty d;
  if (mode < 0) return d;
  PeWork& w = pl->pe[p];
  const int L = pl->L;
  if (mode == CB_MODE_COOP && pl->P > 1) {
    d.bits = w.bm[1].bits;
    d.summ = w.bm[1].summ;
    d.list = w.owner_final;
    d.count = &pl->meta_at(p, L)->n_dst;
    d.cap = w.cap_final;
  } else {
    d.bits = w.bm[(L - 1) & 1].bits;
    d.summ = w.bm[(L - 1) & 1].summ;
    d.list = w.L[L - 1].src;
    d.count = &pl->meta_at(p, L - 1)->n_src;
    d.cap = w.L[L - 1].cap_src;
  }
  return d;
}

ExtractArgs extract_args(PeWork& w, const Bitmap& bm, const Bitmap* zero_bm, uint32_t* out,
                         uint64_t cap, unsigned long long* c1, unsigned long long* c2,
                         int ticket, int slot) {
  ExtractArgs e{};
  e.bits = bm.bits;
  e.summ = bm.summ;
  e.wprefix = bm.wprefix;
  e.zero_bits = zero_bm ? zero_bm->bits : nullptr;
  e.zero_summ = zero_bm ? zero_bm->summ : nullptr;
  e.words_padded = bm.words_padded;
  e.out = out;
  e.cap_out = cap;
  e.count_out = c1;
  e.count_out2 = c2;
  e.ticket = w.sync.tickets + ticket;
  e.exit_ctr = w.sync.tickets + Sync::kMaxTickets + ticket;
  e.status = w.sync.status_a;
  e.epoch = w.sync.epoch;
  e.slot = slot;
  e.overflow = w.sync.overflow;
  return e;
}

RelabelArgs relabel_args(const Bitmap& bm, const LayerBufs& b, const uint32_t* D,
                         const LayerMeta* me) {
  RelabelArgs r{};
  r.bits = bm.bits;
  r.wprefix = bm.wprefix;
  r.meta = me;
  r.edges = b.edges;
  r.cap_edges = b.cap_edges;
  r.D = D;
  r.dst_pos = b.dst_pos;
  return r;
}

FrontierArgs frontier_args(cb_plan* pl, PeWork& w, uint32_t p, int l, const uint32_t* D,
                           uint64_t n_dst_param, Bitmap& set_bm) {
  const LayerBufs& b = w.L[l];
  FrontierArgs fa{};
  fa.D = D;
  fa.meta = pl->meta_at(p, l);
  fa.n_dst_param = n_dst_param;
  fa.indptr = pl->g->g.indptr;
  fa.kind = pl->kind;
  fa.k = pl->fanouts[l];
  fa.layer = l;
  fa.var = pl->var;
  fa.set_bits = set_bm.bits;
  fa.set_summ = set_bm.summ;
  fa.act = b.act;
  fa.tile_first = b.tile_first;
  fa.out_prefix = b.out_prefix;
  fa.slots = b.slots;
  fa.cap_edges = b.cap_edges;
  fa.cap_tiles = w.sync.max_tiles - 1;
  fa.ticket = w.sync.tickets + 3 * l;
  fa.exit_ctr = w.sync.tickets + Sync::kMaxTickets + 3 * l;
  fa.st_a = w.sync.status_a;
  fa.st_b = w.sync.status_b;
  fa.st_c = w.sync.status_c;
  fa.epoch = w.sync.epoch;
  fa.slot = 8 * l;
  fa.overflow = w.sync.overflow;
  fa.trace = pl->trace ? pl->trace + (3 * l) * kTraceKernel : nullptr;
  return fa;
}

LaborArgs labor_args(cb_plan* pl, PeWork& w, uint32_t p, int l, const uint32_t* D,
                     Bitmap& set_bm) {
  const LayerBufs& b = w.L[l];
  LaborArgs la{};
  la.meta = pl->meta_at(p, l);
  la.act = b.act;
  la.tile_first = b.tile_first;
  la.D = D;
  la.indices = pl->g->g.indices;
  la.kind = pl->kind;
  la.k = pl->fanouts[l];
  la.layer = l;
  la.var = pl->var;
  la.bits = set_bm.bits;
  la.summ = set_bm.summ;
  la.edges = b.edges;
  la.slots = b.slots;
  la.keep_words = w.sync.keep_words;
  la.stage = w.sync.stage;
  la.vtab = pl->vtab;
  la.n_vert = pl->g->g.n;
  la.cap_edges = b.cap_edges;
  la.ticket = w.sync.tickets + 3 * l + 1;
  la.exit_ctr = w.sync.tickets + Sync::kMaxTickets + 3 * l + 1;
  la.status = w.sync.status_b;  // emit runs concurrently with extract (status_a)
  la.epoch = w.sync.epoch;
  la.slot = 8 * l + 3;
  la.overflow = w.sync.overflow;
  la.trace = pl->trace ? pl->trace + (3 * l + 1) * kTraceKernel : nullptr;
  return la;
}

// Frontier + sampling of one layer of one part (sample.cu kernels).
uint64_t enqueue_layer(cb_plan* pl, PeWork& w, uint32_t p, int l, const uint32_t* D,
                       uint64_t cap_dst, uint64_t n_dst_param, Bitmap& set_bm,
                       const RelabelArgs& fused, uint64_t fused_work, bool smooth,
                       const ExtractArgs& ex) {
  NvtxRange nvtx_("cb.layer");
  const DeviceGraph& g = pl->g->g;
  const LayerBufs& b = w.L[l];
  cudaStream_t st = pl->stream;
  launch_frontier(frontier_args(pl, w, p, l, D, n_dst_param, set_bm), fused, cap_dst,
                  fused_work, st);
  prof_mark(pl);
  const LaborArgs la = labor_args(pl, w, p, l, D, set_bm);
  if (pl->kind == CB_NS) {
    launch_ns(la, D, b.out_prefix, g.indptr, g.indices, cap_dst, smooth, st);
    prof_mark(pl);
    launch_extract(ex, st);
    prof_mark(pl);
    return 4;
  }
  if (pl->kind == CB_RW) {
    RwArgs ra{};
    ra.D = D;
    ra.meta = la.meta;
    ra.indptr = g.indptr;
    ra.indices = g.indices;
    ra.layer = l;
    ra.k = pl->fanouts[l];
    ra.walks = pl->rw_walks;
    ra.length = pl->rw_length;
    ra.restart = pl->rw_restart;
    ra.var = pl->var;
    ra.bits = set_bm.bits;
    ra.summ = set_bm.summ;
    ra.slots = b.slots;
    ra.cnt = b.out_prefix;
    ra.edges = b.edges;
    ra.cap_edges = b.cap_edges;
    ra.status = w.sync.status_c;
    ra.epoch = w.sync.epoch;
    ra.slot = 8 * l + 6;
    ra.ticket = w.sync.tickets + 3 * l + 1;
    ra.overflow = w.sync.overflow;
    launch_rw(ra, cap_dst, smooth, st);
    prof_mark(pl);
    launch_extract(ex, st);
    prof_mark(pl);
    return 4;
  }
  launch_labor(la, w.sync.max_tiles, smooth, st);  // labor_mark
  prof_mark(pl);
  ExtractArgs ext = ex;
  ext.trace = pl->trace ? pl->trace + (3 * l + 2) * kTraceKernel : nullptr;
  launch_labor_post(la, w.sync.max_tiles, ext, st);  // emit || extract
  prof_mark(pl);
  return (smooth && pl->kind == CB_LABOR0 && pl->vtab) ? 4 : 3;  // (+ variate table)
}

// The per-batch launch sequence. d_seeds: P seed lists back to back (device).
void enqueue_batch(cb_plan* pl, int mode, const uint32_t* d_seeds, const uint64_t* off,
                   const cb_sched* sched, bool capturing = false) {
  const uint32_t P = pl->P;
  const int L = pl->L;
  cudaStream_t st = pl->stream;
  uint64_t launches = 0;
  if (!capturing) {
    const Variates v = make_variates(sched);
    CB_CUDA(cudaMemcpyAsync(pl->var, &v, sizeof(Variates), cudaMemcpyHostToDevice, st));
  }
  pl->mode = mode;
  pl->seeds_off.assign(off, off + P + 1);
  if (!capturing && ++pl->batches % (1u << 17) == 0) {  // epoch wrap (18-bit epochs)
    for (auto& w : pl->pe) {
      CB_CUDA(cudaMemsetAsync(w.sync.status_a, 0, w.sync.max_tiles * 8, st));
      CB_CUDA(cudaMemsetAsync(w.sync.status_b, 0, w.sync.max_tiles * 8, st));
      CB_CUDA(cudaMemsetAsync(w.sync.status_c, 0, w.sync.max_tiles * 8, st));
    }
  }
  const bool coop = (mode == CB_MODE_COOP) && P > 1;
  const bool smooth = sched->kappa != cbdev::kKappaInf && sched->kappa >= 2;
  pl->smooth = smooth;
  // during capture the graph must clear what a batch of its own mode leaves
  const int dm = capturing ? mode : pl->dirty_mode;
  const RelabelArgs none{};
  for (uint32_t p = 0; p < P; ++p) {
    const Dirty d = dirty_of(pl, p, dm);
    launch_batch_begin(pl->pe[p].sync, d.bits, d.summ, d.list, d.count, d.cap,
                       pl->pe[p].bm[0].words_padded, st);
    ++launches;
    prof_mark(pl);
  }

  if (!coop) {
    for (uint32_t p = 0; p < P; ++p) {
      PeWork& w = pl->pe[p];
      for (int l = 0; l < L; ++l) {
        const uint32_t* D = (l == 0) ? d_seeds + off[p] : w.L[l - 1].src;
        const uint64_t cap_dst = (l == 0) ? w.L[0].cap_dst : w.L[l - 1].cap_src;
        RelabelArgs fused = none;
        uint64_t fused_work = 0;
        if (l > 0) {
          const uint32_t* Dp = (l == 1) ? d_seeds + off[p] : w.L[l - 2].src;
          fused = relabel_args(w.bm[(l - 1) & 1], w.L[l - 1], Dp, pl->meta_at(p, l - 1));
          fused_work = w.L[l - 1].cap_edges;
        }
        launches += enqueue_layer(
            pl, w, p, l, D, cap_dst, l == 0 ? off[p + 1] - off[p] : ~0ULL, w.bm[l & 1], fused,
            fused_work, smooth,
            extract_args(w, w.bm[l & 1], &w.bm[(l + 1) & 1], w.L[l].src, w.L[l].cap_src,
                         &pl->meta_at(p, l)->n_src, &pl->meta_at(p, l + 1)->n_dst, 3 * l + 2,
                         8 * l + 4));
      }
      const uint32_t* Dl = (L == 1) ? d_seeds + off[p] : w.L[L - 2].src;
      launch_relabel(relabel_args(w.bm[(L - 1) & 1], w.L[L - 1], Dl, pl->meta_at(p, L - 1)),
                     std::max(w.L[L - 1].cap_edges, w.L[L - 1].cap_dst), st);
      ++launches;
      prof_mark(pl);
    }
  } else {
    CB_CUDA(cudaMemsetAsync(pl->send_counts, 0, sizeof(unsigned long long) * L * P * P, st));
    for (int l = 0; l < L; ++l) {
      uint64_t max_src = 1;
      for (uint32_t p = 0; p < P; ++p) {
        PeWork& w = pl->pe[p];
        const uint32_t* D = (l == 0) ? d_seeds + off[p] : w.L[l].dst;
        launches += enqueue_layer(
            pl, w, p, l, D, w.L[l].cap_dst, l == 0 ? off[p + 1] - off[p] : ~0ULL, w.bm[0], none,
            0, smooth,
            extract_args(w, w.bm[0], &w.bm[1], w.L[l].src, w.L[l].cap_src,
                         &pl->meta_at(p, l)->n_src, nullptr, 3 * l + 2, 8 * l + 4));
        launch_relabel(relabel_args(w.bm[0], w.L[l], D, pl->meta_at(p, l)),
                       std::max(w.L[l].cap_edges, w.L[l].cap_dst), st);
        launches += 1;
        max_src = std::max(max_src, w.L[l].cap_src);
      }
      PartPtrs pp{};
      for (uint32_t p = 0; p < P; ++p) {
        PeWork& w = pl->pe[p];
        pp.src[p] = w.L[l].src;
        pp.count[p] = &pl->meta_at(p, l)->n_src;
        pp.clear_bits[p] = w.bm[0].bits;
        pp.clear_summ[p] = w.bm[0].summ;
        pp.xbits[p] = w.bm[1].bits;
        pp.xsumm[p] = w.bm[1].summ;
        pp.xprefix[p] = w.bm[1].wprefix;
        pp.loc_part[p] = w.loc_part[l];
        pp.loc_row[p] = w.loc_row[l];
      }
      launch_route(pp, pl->pm->owner, P,
                   pl->send_counts + static_cast<uint64_t>(l) * P * P, max_src, st);
      ++launches;
      for (uint32_t q = 0; q < P; ++q) {
        PeWork& w = pl->pe[q];
        uint32_t* next = (l + 1 < L) ? w.L[l + 1].dst : w.owner_final;
        const uint64_t cap = (l + 1 < L) ? w.L[l + 1].cap_dst : w.cap_final;
        launch_extract(extract_args(w, w.bm[1], nullptr, next, cap,
                                    &pl->meta_at(q, l + 1)->n_dst, nullptr, 3 * L + l,
                                    8 * l + 5),
                       st);
        ++launches;
      }
      launch_locate(pp, pl->pm->owner, P, max_src, st);
      ++launches;
    }
  }
  pl->launches = launches;
  pl->have_batch = true;
  pl->have_rows = false;
  pl->dirty_mode = mode;
}

void check_overflow(cb_plan* pl) {
  CB_CUDA(cudaStreamSynchronize(pl->stream));
  for (auto& w : pl->pe) {
    unsigned o = 0;
    CB_CUDA(cudaMemcpy(&o, w.sync.overflow, 4, cudaMemcpyDeviceToHost));
    if (o) throw Error(kOverflow, "capacity bound exceeded on device (retry with larger plan)");
  }
}

void sample_host(cb_plan* pl, int mode, const uint32_t* flat, const uint64_t* off,
                 const cb_sched* sched) {
  require(mode == CB_MODE_COOP || mode == CB_MODE_INDEP, "unknown sampling mode");
  require(sched != nullptr, "null schedule");
  require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
  check_seeds_host(pl, flat, off);
  if (mode == CB_MODE_COOP) check_ownership_host(pl, flat, off);
  const uint64_t total = off[pl->P];
  if (total)
    CB_CUDA(cudaMemcpyAsync(pl->seeds, flat, total * 4, cudaMemcpyHostToDevice, pl->stream));
  enqueue_batch(pl, mode, pl->seeds, off, sched);
}

const LayerMeta host_meta(cb_plan* pl, uint32_t p, int l) {
  LayerMeta m{};
  CB_CUDA(cudaStreamSynchronize(pl->stream));
  CB_CUDA(cudaMemcpy(&m, pl->meta_at(p, l), sizeof(LayerMeta), cudaMemcpyDeviceToHost));
  return m;
}

void require_batch(const cb_plan* pl, uint32_t p, int l) {
  require(pl->have_batch, "no sampled batch in this plan");
  require(p < pl->P, "part index out of range");
  require(l >= 0 && l < pl->L, "layer index out of range");
}

void prepare_rows(cb_plan* pl, const cb_features* f) {
  require(f->n_rows == pl->g->g.n, "feature table does not match the graph");
  for (uint32_t p = 0; p < pl->P; ++p) {
    PeWork& w = pl->pe[p];
    const LayerBufs& b = w.L[pl->L - 1];
    if (!w.rows || w.rows_row_bytes != f->row_bytes || w.cap_rows < b.cap_src) {
      w.rows = pl->rows_mem.alloc<unsigned char>(b.cap_src * f->row_bytes);
      w.cap_rows = b.cap_src;
      w.rows_row_bytes = f->row_bytes;
    }
  }
}

void enqueue_gather(cb_plan* pl, const cb_features* f) {
  NvtxRange nvtx_("cb.gather");
  const int vb = vec_bytes_for(f->row_bytes);
  for (uint32_t p = 0; p < pl->P; ++p) {
    PeWork& w = pl->pe[p];
    const LayerBufs& b = w.L[pl->L - 1];
    launch_gather(f->table, vb, f->row_bytes, b.src, &pl->meta_at(p, pl->L - 1)->n_src,
                  w.cap_rows, f->row_map, w.rows, pl->stream);
    pl->launches += 1;
    prof_mark(pl);
  }
  pl->have_rows = true;
}

}  // namespace

// ===================================================================== C-ABI ==
extern "C" {

const char* cb_last_error(void) { return g_err.c_str(); }
const char* cb_version(void) { return "coopbatch_b200 0.1 (sm_100a)"; }

int cb_device_count(int* out) {
  return guard([&] { CB_CUDA(cudaGetDeviceCount(out)); });
}

int cb_graph_create_from_csr(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                             uint64_t m, int device, cb_graph** out) {
  return guard([&] {
    require(indptr != nullptr && (m == 0 || indices != nullptr), "null CSR arrays");
    require(n < (1ULL << 32), "vertex ids must fit 32 bits");
    // validate_csr (graph.cpp:267-284)
    require(indptr[0] == 0, "csr: indptr[0] != 0");
    require(indptr[n] == m, "csr: indptr[n] != num edges");
    for (uint64_t v = 0; v < n; ++v)
      require(indptr[v] <= indptr[v + 1],
              "csr: indptr not nondecreasing at " + std::to_string(v));
    for (uint64_t e = 0; e < m; ++e) require(indices[e] < n, "csr: index out of range");
    DeviceGuard dg(device);
    auto h = std::make_unique<cb_graph>();
    h->g.device = device;
    h->g.n = n;
    h->g.m = m;
    CB_CUDA(cudaMalloc(&h->g.indptr, (n + 1) * 8));
    CB_CUDA(cudaMalloc(&h->g.indices, std::max<uint64_t>(m, 1) * 4));
    CB_CUDA(cudaMemcpy(h->g.indptr, indptr, (n + 1) * 8, cudaMemcpyHostToDevice));
    if (m) CB_CUDA(cudaMemcpy(h->g.indices, indices, m * 4, cudaMemcpyHostToDevice));
    uint64_t md = 0;
    for (uint64_t v = 0; v < n; ++v) md = std::max(md, indptr[v + 1] - indptr[v]);
    h->g.max_degree = md;
    *out = h.release();
  });
}

// CBCS binary CSR (graph.hpp:78-80, graph.cpp:196-265): "CBCS", u32 version 1,
// u64 n, u64 m, u64 indptr[n+1], u32 indices[m], u8 flags, f32 weights[m] if
// flags & 1. Little-endian. Weights are validated (> 0) and not kept: the
// device path samples unweighted (LABOR-0 / NS / FULL).
int cb_graph_load_cbcs(const char* path, int device, cb_graph** out) {
  return guard([&] {
    require(path != nullptr && out != nullptr, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw Error(kIo, std::string("cannot open: ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, &std::fclose);
    auto rd = [&](void* dst, size_t bytes, const char* what) {
      if (bytes && std::fread(dst, 1, bytes, f) != bytes)
        throw Error(kFormat, std::string("csr file truncated reading ") + what);
    };
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CBCS", 4) != 0)
      throw Error(kFormat, std::string("not a CBCS file: ") + path);
    uint32_t version = 0;
    rd(&version, 4, "version");
    if (version != 1) throw Error(kFormat, "unsupported CBCS version " + std::to_string(version));
    uint64_t n = 0, m = 0;
    rd(&n, 8, "num_vertices");
    rd(&m, 8, "num_edges");
    std::vector<uint64_t> indptr(n + 1);
    std::vector<uint32_t> indices(m);
    rd(indptr.data(), (n + 1) * 8, "indptr");
    rd(indices.data(), m * 4, "indices");
    uint8_t flags = 0;
    rd(&flags, 1, "flags");
    if (flags & 1) {
      std::vector<float> w(m);
      rd(w.data(), m * 4, "weights");
      for (float x : w) require(x > 0.0f, "csr: weights must be > 0");
    }
    const int rc = cb_graph_create_from_csr(indptr.data(), indices.data(), n, m, device, out);
    if (rc != CB_OK) throw Error(static_cast<Status>(rc), g_err);
  });
}

int cb_graph_save_cbcs(const cb_graph* g, const char* path) {
  return guard([&] {
    require(g != nullptr && path != nullptr, "null argument");
    std::vector<uint64_t> indptr(g->g.n + 1);
    std::vector<uint32_t> indices(g->g.m);
    {
      DeviceGuard dg(g->g.device);
      CB_CUDA(cudaMemcpy(indptr.data(), g->g.indptr, (g->g.n + 1) * 8, cudaMemcpyDeviceToHost));
      if (g->g.m)
        CB_CUDA(cudaMemcpy(indices.data(), g->g.indices, g->g.m * 4, cudaMemcpyDeviceToHost));
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(kIo, std::string("cannot open for write: ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, &std::fclose);
    const uint32_t version = 1;
    const uint64_t n = g->g.n, m = g->g.m;
    const uint8_t flags = 0;
    bool ok = std::fwrite("CBCS", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&m, 8, 1, f) == 1 &&
              std::fwrite(indptr.data(), 8, n + 1, f) == n + 1 &&
              (m == 0 || std::fwrite(indices.data(), 4, m, f) == m) &&
              std::fwrite(&flags, 1, 1, f) == 1;
    if (!ok) throw Error(kIo, std::string("write failed: ") + path);
  });
}

int cb_graph_generate_rmat(uint64_t n, uint64_t m, uint64_t seed, int device, cb_graph** out) {
  return guard([&] {
    DeviceGuard dg(device);
    auto h = std::make_unique<cb_graph>();
    h->g.device = device;
    cudaStream_t st;
    CB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      graph_generate_rmat(h->g, n, m, seed, st);
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    CB_CUDA(cudaStreamDestroy(st));
    *out = h.release();
  });
}

int cb_graph_info(const cb_graph* g, uint64_t* n, uint64_t* m, uint64_t* max_degree) {
  return guard([&] {
    require(g != nullptr, "null graph");
    if (n) *n = g->g.n;
    if (m) *m = g->g.m;
    if (max_degree) *max_degree = g->g.max_degree;
  });
}

int cb_graph_download(const cb_graph* g, uint64_t* indptr, uint32_t* indices) {
  return guard([&] {
    require(g != nullptr, "null graph");
    DeviceGuard dg(g->g.device);
    if (indptr)
      CB_CUDA(cudaMemcpy(indptr, g->g.indptr, (g->g.n + 1) * 8, cudaMemcpyDeviceToHost));
    if (indices && g->g.m)
      CB_CUDA(cudaMemcpy(indices, g->g.indices, g->g.m * 4, cudaMemcpyDeviceToHost));
  });
}

void cb_graph_destroy(cb_graph* g) {
  if (!g) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->g.device);
  delete g;
  cudaSetDevice(prev);
}

static void finish_partition(cb_partition* pm) {
  // members = vertices grouped by owner, ascending within a part (part_members,
  // partition.cpp:99-105); row_map[v] = global row of v. Stable key sort.
  const uint64_t n = pm->n;
  pm->row_map = pm->mem.alloc<uint32_t>(n);
  pm->members = pm->mem.alloc<uint32_t>(n);
  uint32_t* keys2 = pm->mem.alloc<uint32_t>(n);
  uint32_t* ids = pm->mem.alloc<uint32_t>(n);
  cudaStream_t st;
  CB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<uint32_t> iota(n);
  for (uint64_t v = 0; v < n; ++v) iota[v] = static_cast<uint32_t>(v);
  CB_CUDA(cudaMemcpy(ids, iota.data(), n * 4, cudaMemcpyHostToDevice));
  uint32_t* keys = pm->mem.alloc<uint32_t>(n);
  CB_CUDA(cudaMemcpy(keys, pm->owner, n * 4, cudaMemcpyDeviceToDevice));
  // the copies above run on the legacy stream (D2D and staged pageable H2D
  // return before completion); st is non-blocking, so order them explicitly
  CB_CUDA(cudaDeviceSynchronize());
  int bits = 1;
  while ((1u << bits) < pm->parts) ++bits;
  cub::DoubleBuffer<uint32_t> kb(keys, keys2), vb(ids, pm->members);
  size_t tmp_bytes = 0;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, (int64_t)n, 0, bits, st));
  void* tmp = nullptr;
  CB_CUDA(cudaMalloc(&tmp, tmp_bytes + 16));
  CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, (int64_t)n, 0, bits, st));
  CB_CUDA(cudaStreamSynchronize(st));
  cudaFree(tmp);
  std::vector<uint32_t> members(n), sorted_keys(n);
  CB_CUDA(cudaMemcpy(members.data(), vb.Current(), n * 4, cudaMemcpyDeviceToHost));
  CB_CUDA(cudaMemcpy(sorted_keys.data(), kb.Current(), n * 4, cudaMemcpyDeviceToHost));
  pm->shard_off.assign(pm->parts + 1, 0);
  for (uint64_t i = 0; i < n; ++i) pm->shard_off[sorted_keys[i] + 1]++;
  for (uint32_t q = 0; q < pm->parts; ++q) pm->shard_off[q + 1] += pm->shard_off[q];
  std::vector<uint32_t> row_map(n);
  for (uint64_t i = 0; i < n; ++i) row_map[members[i]] = static_cast<uint32_t>(i);
  CB_CUDA(cudaMemcpy(pm->members, members.data(), n * 4, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(pm->row_map, row_map.data(), n * 4, cudaMemcpyHostToDevice));
  CB_CUDA(cudaStreamDestroy(st));
}

int cb_partition_random(const cb_graph* g, uint32_t parts, uint64_t seed, cb_partition** out) {
  return guard([&] {
    require(g != nullptr, "null graph");
    require(parts >= 1, "partition_random: parts must be >= 1");
    require(parts <= kMaxParts, "at most 16 parts per device");
    DeviceGuard dg(g->g.device);
    auto pm = std::make_unique<cb_partition>();
    pm->device = g->g.device;
    pm->n = g->g.n;
    pm->parts = parts;
    pm->owner = pm->mem.alloc<uint32_t>(pm->n);
    partition_random_device(pm->n, parts, seed, pm->owner, nullptr);
    CB_CUDA(cudaDeviceSynchronize());
    finish_partition(pm.get());
    *out = pm.release();
  });
}

int cb_partition_create(const cb_graph* g, const uint32_t* owner, uint32_t parts,
                        cb_partition** out) {
  return guard([&] {
    require(g != nullptr && owner != nullptr, "null argument");
    require(parts >= 1, "partition: zero parts");
    require(parts <= kMaxParts, "at most 16 parts per device");
    for (uint64_t v = 0; v < g->g.n; ++v)
      require(owner[v] < parts, "partition: owner id out of range");
    DeviceGuard dg(g->g.device);
    auto pm = std::make_unique<cb_partition>();
    pm->device = g->g.device;
    pm->n = g->g.n;
    pm->parts = parts;
    pm->owner = pm->mem.alloc<uint32_t>(pm->n);
    CB_CUDA(cudaMemcpy(pm->owner, owner, pm->n * 4, cudaMemcpyHostToDevice));
    finish_partition(pm.get());
    *out = pm.release();
  });
}

int cb_partition_download(const cb_partition* pm, uint32_t* owner) {
  return guard([&] {
    require(pm != nullptr && owner != nullptr, "null argument");
    DeviceGuard dg(pm->device);
    CB_CUDA(cudaMemcpy(owner, pm->owner, pm->n * 4, cudaMemcpyDeviceToHost));
  });
}

int cb_cross_edge_ratio(const cb_graph* g, const cb_partition* pm, uint64_t* cross,
                        double* ratio) {
  return guard([&] {
    require(g != nullptr && pm != nullptr, "null argument");
    require(pm->n == g->g.n, "partition: owner array does not cover all vertices");
    DeviceGuard dg(g->g.device);
    const uint64_t c = cross_edges(g->g, pm->owner, nullptr);
    if (cross) *cross = c;
    if (ratio) *ratio = g->g.m ? static_cast<double>(c) / static_cast<double>(g->g.m) : 0.0;
  });
}

int cb_partition_members(const cb_partition* pm, uint32_t* members, uint64_t* shard_off) {
  return guard([&] {
    require(pm != nullptr, "null partition");
    DeviceGuard dg(pm->device);
    if (members) CB_CUDA(cudaMemcpy(members, pm->members, pm->n * 4, cudaMemcpyDeviceToHost));
    if (shard_off)
      for (uint32_t q = 0; q <= pm->parts; ++q) shard_off[q] = pm->shard_off[q];
  });
}

void cb_partition_destroy(cb_partition* pm) {
  if (!pm) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(pm->device);
  delete pm;
  cudaSetDevice(prev);
}

int cb_features_synth(const cb_graph* g, const cb_partition* pm, uint32_t dim, int dtype,
                      uint64_t seed, cb_features** out) {
  return guard([&] {
    require(g != nullptr, "null graph");
    require(dim >= 1, "feature dim must be >= 1");
    require(dtype == CB_F64 || dtype == CB_F32 || dtype == CB_F16, "unknown dtype");
    require(pm == nullptr || pm->n == g->g.n, "partition does not cover the graph");
    DeviceGuard dg(g->g.device);
    auto f = std::make_unique<cb_features>();
    f->device = g->g.device;
    f->dim = dim;
    f->dtype = dtype;
    f->seed = seed;
    const uint64_t es = dtype == CB_F64 ? 8 : (dtype == CB_F32 ? 4 : 2);
    f->row_bytes = es * dim;
    f->n_rows = g->g.n;
    f->table = f->mem.alloc<unsigned char>(f->n_rows * f->row_bytes);
    const bool sharded = pm != nullptr && pm->parts > 1;
    if (sharded) {
      f->row_map = f->mem.alloc<uint32_t>(g->g.n);
      CB_CUDA(cudaMemcpy(f->row_map, pm->row_map, g->g.n * 4, cudaMemcpyDeviceToDevice));
    }
    launch_synth(seed, dim, dtype, f->n_rows, sharded ? pm->members : nullptr, 0, f->table,
                 nullptr);
    CB_CUDA(cudaDeviceSynchronize());
    *out = f.release();
  });
}

int cb_features_info(const cb_features* f, uint32_t* dim, int* dtype, uint64_t* row_bytes) {
  return guard([&] {
    require(f != nullptr, "null features");
    if (dim) *dim = f->dim;
    if (dtype) *dtype = f->dtype;
    if (row_bytes) *row_bytes = f->row_bytes;
  });
}

void cb_features_destroy(cb_features* f) {
  if (!f) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(f->device);
  delete f;
  cudaSetDevice(prev);
}

int cb_plan_create(const cb_graph* g, const cb_partition* pm, int num_layers, int kind,
                   const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out) {
  return guard([&] {
    require(g != nullptr, "null graph");
    require(num_layers >= 1, "expand: num_layers must be >= 1");
    require(num_layers <= 8, "at most 8 layers");
    require(kind == CB_FULL || kind == CB_NS || kind == CB_LABOR0 || kind == CB_RW,
            "sample_block: unknown sampler kind");
    require(fanouts != nullptr || kind == CB_FULL, "null fanouts");
    require(pm == nullptr || pm->n == g->g.n, "partition does not cover the graph");
    DeviceGuard dg(g->g.device);
    auto pl = std::make_unique<cb_plan>();
    pl->device = g->g.device;
    pl->g = g;
    pl->pm = pm;
    pl->P = pm ? pm->parts : 1;
    pl->L = num_layers;
    pl->kind = kind;
    for (int l = 0; l < num_layers; ++l) {
      const uint32_t k = fanouts ? fanouts[l] : 1;
      if (kind != CB_FULL)
        require(k >= 1, kind == CB_NS ? "sample_ns: fanout must be >= 1"
                                      : "sample_labor0: fanout must be >= 1");
      pl->fanouts.push_back(k);
    }
    pl->max_seeds = std::max<uint64_t>(max_seeds_per_part, 1);
    if (const char* e = std::getenv("CB_TRACE")) pl->trace_on = std::atoi(e) != 0;
    CB_CUDA(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
    plan_alloc(pl.get());
    *out = pl.release();
  });
}

void cb_plan_destroy(cb_plan* plan) {
  if (!plan) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  cudaStreamSynchronize(plan->stream);
  cudaStreamDestroy(plan->stream);
  delete plan;
  cudaSetDevice(prev);
}

int cb_plan_num_parts(const cb_plan* plan, uint32_t* parts) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    *parts = plan->P;
  });
}

void* cb_plan_stream(const cb_plan* plan) { return plan ? plan->stream : nullptr; }

int cb_sample(cb_plan* plan, int mode, const uint32_t* seeds_flat, const uint64_t* seeds_off,
              const cb_sched* sched) {
  NvtxRange nvtx_("cb.sample");
  return guard([&] {
    require(plan != nullptr && seeds_off != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    sample_host(plan, mode, seeds_flat, seeds_off, sched);
  });
}

int cb_sample_sync(cb_plan* plan, int mode, const uint32_t* seeds_flat,
                   const uint64_t* seeds_off, const cb_sched* sched) {
  NvtxRange nvtx_("cb.sample_sync");
  return guard([&] {
    require(plan != nullptr && seeds_off != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    for (int attempt = 0;; ++attempt) {
      sample_host(plan, mode, seeds_flat, seeds_off, sched);
      try {
        check_overflow(plan);
        return;
      } catch (const Error& e) {
        if (e.code != kOverflow || attempt >= 12) throw;
        plan->grow *= 2.0;
        plan_alloc(plan);
      }
    }
  });
}

int cb_sample_device(cb_plan* plan, int mode, const uint32_t* d_seeds_flat,
                     const uint64_t* seeds_off, const cb_sched* sched) {
  return guard([&] {
    require(plan != nullptr && seeds_off != nullptr && sched != nullptr, "null argument");
    require(mode == CB_MODE_COOP || mode == CB_MODE_INDEP, "unknown sampling mode");
    for (uint32_t p = 0; p < plan->P; ++p)
      require(seeds_off[p + 1] - seeds_off[p] <= plan->max_seeds,
              "more seeds than the plan's max_seeds_per_part");
    DeviceGuard dg(plan->device);
    enqueue_batch(plan, mode, d_seeds_flat, seeds_off, sched);
  });
}

int cb_gather(cb_plan* plan, const cb_features* f) {
  return guard([&] {
    require(plan != nullptr && f != nullptr, "null argument");
    require(plan->have_batch, "no sampled batch in this plan");
    DeviceGuard dg(plan->device);
    prepare_rows(plan, f);
    enqueue_gather(plan, f);
  });
}

int cb_plan_capture(cb_plan* plan, int mode, const uint64_t* seeds_off, const cb_features* f,
                    const cb_sched* sched) {
  return guard([&] {
    require(plan != nullptr && seeds_off != nullptr && sched != nullptr, "null argument");
    require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    require(mode == CB_MODE_COOP || mode == CB_MODE_INDEP, "unknown sampling mode");
    for (uint32_t p = 0; p < plan->P; ++p)
      require(seeds_off[p + 1] - seeds_off[p] <= plan->max_seeds,
              "more seeds than the plan's max_seeds_per_part");
    DeviceGuard dg(plan->device);
    plan->drop_graphs();
    if (f) prepare_rows(plan, f);
    const cb_sched& dummy = *sched;
    // one eager batch first: sets kernel attributes outside capture
    enqueue_batch(plan, mode, plan->seeds, seeds_off, &dummy);
    if (f) enqueue_gather(plan, f);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    cudaGraph_t graph;
    CB_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
    enqueue_batch(plan, mode, plan->seeds, seeds_off, &dummy, true);
    CB_CUDA(cudaStreamEndCapture(plan->stream, &graph));
    CB_CUDA(cudaGraphInstantiate(&plan->exec_sample, graph, 0));
    CB_CUDA(cudaGraphDestroy(graph));
    plan->cap_launches_sample = plan->launches;
    if (f) {
      CB_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
      plan->launches = 0;
      enqueue_gather(plan, f);
      CB_CUDA(cudaStreamEndCapture(plan->stream, &graph));
      CB_CUDA(cudaGraphInstantiate(&plan->exec_gather, graph, 0));
      CB_CUDA(cudaGraphDestroy(graph));
      plan->cap_launches_gather = plan->launches;
      CB_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
      enqueue_batch(plan, mode, plan->seeds, seeds_off, &dummy, true);
      enqueue_gather(plan, f);
      CB_CUDA(cudaStreamEndCapture(plan->stream, &graph));
      CB_CUDA(cudaGraphInstantiate(&plan->exec_all, graph, 0));
      CB_CUDA(cudaGraphDestroy(graph));
    }
    // profiling twin: same launches with external event-record nodes between
    {
      plan->prof = &plan->graph_events;
      plan->prof_external = true;
      CB_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
      prof_mark(plan);
      enqueue_batch(plan, mode, plan->seeds, seeds_off, &dummy, true);
      if (f) enqueue_gather(plan, f);
      CB_CUDA(cudaStreamEndCapture(plan->stream, &graph));
      plan->prof = nullptr;
      plan->prof_external = false;
      CB_CUDA(cudaGraphInstantiate(&plan->exec_prof, graph, 0));
      CB_CUDA(cudaGraphDestroy(graph));
    }
    plan->cap_mode = mode;
    plan->cap_smooth = plan->smooth;
    plan->cap_off.assign(seeds_off, seeds_off + plan->P + 1);
    plan->have_batch = false;
  });
}

int cb_plan_replay(cb_plan* plan, const uint32_t* seeds_flat, int seeds_on_device,
                   const cb_sched* sched, int what) {
  NvtxRange nvtx_("cb.replay");
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(plan->exec_sample != nullptr, "no captured batch (call cb_plan_capture)");
    DeviceGuard dg(plan->device);
    cudaStream_t st = plan->stream;
    if (what & 1) {
      require(sched != nullptr, "null schedule");
      require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
      const bool sm = sched->kappa != cbdev::kKappaInf && sched->kappa >= 2;
      require(sm == plan->cap_smooth,
              "schedule smoothing differs from the captured batch (re-capture)");
      const uint64_t total = plan->cap_off[plan->P];
      if (seeds_flat && total)
        CB_CUDA(cudaMemcpyAsync(plan->seeds, seeds_flat, total * 4,
                                seeds_on_device ? cudaMemcpyDeviceToDevice
                                                : cudaMemcpyHostToDevice,
                                st));
      const Variates v = make_variates(sched);
      CB_CUDA(cudaMemcpyAsync(plan->var, &v, sizeof(Variates), cudaMemcpyHostToDevice, st));
      if (++plan->batches % (1u << 17) == 0) {
        for (auto& w : plan->pe) {
          CB_CUDA(cudaMemsetAsync(w.sync.status_a, 0, w.sync.max_tiles * 8, st));
          CB_CUDA(cudaMemsetAsync(w.sync.status_b, 0, w.sync.max_tiles * 8, st));
          CB_CUDA(cudaMemsetAsync(w.sync.status_c, 0, w.sync.max_tiles * 8, st));
        }
      }
      if (plan->dirty_mode >= 0 && plan->dirty_mode != plan->cap_mode) {
        for (uint32_t p = 0; p < plan->P; ++p) {
          const Dirty d = dirty_of(plan, p, plan->dirty_mode);
          launch_batch_begin(plan->pe[p].sync, d.bits, d.summ, d.list, d.count, d.cap,
                             plan->pe[p].bm[0].words_padded, st);
        }
      }
      const bool all = (what & 2) && plan->exec_all;
      CB_CUDA(cudaGraphLaunch(all ? plan->exec_all : plan->exec_sample, st));
      plan->dirty_mode = plan->cap_mode;
      plan->mode = plan->cap_mode;
      plan->seeds_off = plan->cap_off;
      plan->have_batch = true;
      plan->have_rows = all;
      plan->launches = plan->cap_launches_sample + (all ? plan->cap_launches_gather : 0);
      if (all) return;
    }
    if (what & 2) {
      require(plan->exec_gather != nullptr, "no captured gather");
      require(plan->have_batch, "no sampled batch in this plan");
      CB_CUDA(cudaGraphLaunch(plan->exec_gather, st));
      plan->have_rows = true;
      plan->launches += plan->cap_launches_gather;
    }
  });
}

int cb_synchronize(cb_plan* plan) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
  });
}

int cb_layer_sizes(cb_plan* plan, uint32_t part, int layer, uint64_t* sizes) {
  return guard([&] {
    require(plan != nullptr && sizes != nullptr, "null argument");
    require_batch(plan, part, layer);
    DeviceGuard dg(plan->device);
    const LayerMeta m = host_meta(plan, part, layer);
    sizes[0] = m.n_dst;
    sizes[1] = m.n_src;
    sizes[2] = m.n_edges;
    sizes[3] = m.uncertified;
    sizes[4] = m.scan_total;
    sizes[5] = m.n_active;
  });
}

int cb_download_block(cb_plan* plan, uint32_t part, int layer, uint32_t* dst, uint32_t* src,
                      uint32_t* edges, uint32_t* dst_pos) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require_batch(plan, part, layer);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const LayerMeta m = host_meta(plan, part, layer);
    PeWork& w = plan->pe[part];
    const uint32_t* d_dst;
    if (layer == 0) d_dst = plan->seeds + plan->seeds_off[part];
    else if (!plan->own_dst()) d_dst = w.L[layer - 1].src;
    else d_dst = w.L[layer].dst;
    const LayerBufs& b = w.L[layer];
    if (dst && m.n_dst) CB_CUDA(cudaMemcpy(dst, d_dst, m.n_dst * 4, cudaMemcpyDeviceToHost));
    if (src && m.n_src) CB_CUDA(cudaMemcpy(src, b.src, m.n_src * 4, cudaMemcpyDeviceToHost));
    if (edges && m.n_edges)
      CB_CUDA(cudaMemcpy(edges, b.edges, m.n_edges * 8, cudaMemcpyDeviceToHost));
    if (dst_pos && m.n_dst)
      CB_CUDA(cudaMemcpy(dst_pos, b.dst_pos, m.n_dst * 4, cudaMemcpyDeviceToHost));
  });
}

int cb_owner_set_size(cb_plan* plan, uint32_t part, uint64_t* n) {
  return guard([&] {
    require(plan != nullptr && n != nullptr, "null argument");
    require_batch(plan, part, 0);
    DeviceGuard dg(plan->device);
    if (plan->coop_active()) *n = host_meta(plan, part, plan->L).n_dst;
    else *n = host_meta(plan, part, plan->L - 1).n_src;
  });
}

int cb_download_owner_set(cb_plan* plan, uint32_t part, uint32_t* ids) {
  return guard([&] {
    require(plan != nullptr && ids != nullptr, "null argument");
    require_batch(plan, part, 0);
    require(plan->mode == CB_MODE_COOP, "owner sets exist only for cooperative batches");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    PeWork& w = plan->pe[part];
    if (plan->coop_active()) {
      const uint64_t n = host_meta(plan, part, plan->L).n_dst;
      if (n) CB_CUDA(cudaMemcpy(ids, w.owner_final, n * 4, cudaMemcpyDeviceToHost));
    } else {  // P = 1: the owner set is the last src list (coop.cpp:44-51)
      const uint64_t n = host_meta(plan, part, plan->L - 1).n_src;
      if (n) CB_CUDA(cudaMemcpy(ids, w.L[plan->L - 1].src, n * 4, cudaMemcpyDeviceToHost));
    }
  });
}

int cb_download_exchange(cb_plan* plan, int layer, uint64_t* send_counts,
                         uint64_t* owner_row_counts, uint32_t* loc_part, uint64_t* loc_row) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require_batch(plan, 0, layer);
    require(plan->mode == CB_MODE_COOP, "exchange records exist only for cooperative batches");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const uint32_t P = plan->P;
    if (!plan->coop_active()) {  // P = 1: everything stays local
      const LayerMeta m = host_meta(plan, 0, layer);
      if (send_counts) send_counts[0] = m.n_src;
      if (owner_row_counts) owner_row_counts[0] = m.n_src;
      for (uint64_t j = 0; j < m.n_src; ++j) {
        if (loc_part) loc_part[j] = 0;
        if (loc_row) loc_row[j] = j;
      }
      return;
    }
    std::vector<unsigned long long> sc(static_cast<size_t>(P) * P);
    CB_CUDA(cudaMemcpy(sc.data(), plan->send_counts + static_cast<uint64_t>(layer) * P * P,
                       sc.size() * 8, cudaMemcpyDeviceToHost));
    if (send_counts)
      for (size_t i = 0; i < sc.size(); ++i) send_counts[i] = sc[i];
    if (owner_row_counts)
      for (uint32_t q = 0; q < P; ++q)
        owner_row_counts[q] = host_meta(plan, q, layer + 1).n_dst;
    uint64_t o = 0;
    for (uint32_t p = 0; p < P; ++p) {
      const uint64_t n = host_meta(plan, p, layer).n_src;
      if (loc_part && n)
        CB_CUDA(cudaMemcpy(loc_part + o, plan->pe[p].loc_part[layer], n * 4,
                           cudaMemcpyDeviceToHost));
      if (loc_row && n) {
        std::vector<uint32_t> tmp(n);
        CB_CUDA(cudaMemcpy(tmp.data(), plan->pe[p].loc_row[layer], n * 4,
                           cudaMemcpyDeviceToHost));
        for (uint64_t j = 0; j < n; ++j) loc_row[o + j] = tmp[j];
      }
      o += n;
    }
  });
}

int cb_download_rows(cb_plan* plan, uint32_t part, void* out) {
  return guard([&] {
    require(plan != nullptr && out != nullptr, "null argument");
    require(plan->have_rows, "no gathered rows (call cb_gather)");
    require(part < plan->P, "part index out of range");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const uint64_t n = host_meta(plan, part, plan->L - 1).n_src;
    PeWork& w = plan->pe[part];
    if (n)
      CB_CUDA(cudaMemcpy(out, w.rows, n * w.rows_row_bytes, cudaMemcpyDeviceToHost));
  });
}

int cb_rows_device(cb_plan* plan, uint32_t part, void** ptr, uint64_t* rows) {
  return guard([&] {
    require(plan != nullptr && ptr != nullptr, "null argument");
    require(plan->have_rows, "no gathered rows (call cb_gather)");
    require(part < plan->P, "part index out of range");
    DeviceGuard dg(plan->device);
    *ptr = plan->pe[part].rows;
    if (rows) *rows = host_meta(plan, part, plan->L - 1).n_src;
  });
}

int cb_plan_profile(cb_plan* plan, int mode, const uint32_t* seeds_flat,
                    const uint64_t* seeds_off, const cb_sched* sched, const cb_features* f,
                    float* ms, int max_n, int* n) {
  return guard([&] {
    require(plan != nullptr && ms != nullptr && n != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    std::vector<cudaEvent_t> ev;
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    plan->prof = &ev;
    try {
      prof_mark(plan);
      sample_host(plan, mode, seeds_flat, seeds_off, sched);
      if (f) {
        prepare_rows(plan, f);
        enqueue_gather(plan, f);
      }
    } catch (...) {
      plan->prof = nullptr;
      for (auto e : ev) cudaEventDestroy(e);
      throw;
    }
    plan->prof = nullptr;
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    int k = 0;
    for (size_t i = 1; i < ev.size() && k < max_n; ++i, ++k)
      CB_CUDA(cudaEventElapsedTime(&ms[k], ev[i - 1], ev[i]));
    *n = k;
    for (auto e : ev) cudaEventDestroy(e);
  });
}

int cb_plan_create_dist(const cb_graph* g, uint32_t world, int num_layers, int kind,
                        const uint32_t* fanouts, uint64_t max_seeds, cb_plan** out) {
  return guard([&] {
    require(g != nullptr && out != nullptr, "null argument");
    require(world >= 1 && world <= kDistMaxParts, "world size must be in [1, 64]");
    require(num_layers >= 1, "coop_sample: num_layers must be >= 1");
    require(num_layers <= 8, "at most 8 layers");
    require(kind == CB_FULL || kind == CB_NS || kind == CB_LABOR0 || kind == CB_RW,
            "sample_block: unknown sampler kind");
    DeviceGuard dg(g->g.device);
    auto pl = std::make_unique<cb_plan>();
    pl->device = g->g.device;
    pl->g = g;
    pl->P = 1;
    pl->dist_world = world;
    pl->L = num_layers;
    pl->kind = kind;
    for (int l = 0; l < num_layers; ++l) {
      const uint32_t k = fanouts ? fanouts[l] : 1;
      if (kind != CB_FULL) require(k >= 1, "fanout must be >= 1");
      pl->fanouts.push_back(k);
    }
    pl->max_seeds = std::max<uint64_t>(max_seeds, 1);
    CB_CUDA(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
    plan_alloc(pl.get());
    pl->mode = CB_MODE_COOP;
    *out = pl.release();
  });
}

int cb_plan_sample_layer(cb_plan* plan, int layer, const uint32_t* d_dst, uint64_t n_dst,
                         const cb_sched* sched, uint64_t* n_src) {
  return guard([&] {
    require(plan != nullptr && sched != nullptr && n_src != nullptr, "null argument");
    require(plan->P == 1, "per-layer sampling needs a single-part plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    LayerBufs& b = w.L[layer];
    uint32_t* D = (layer == 0) ? plan->seeds : b.dst;
    const uint64_t cap = (layer == 0) ? plan->max_seeds : b.cap_dst;
    if (n_dst > cap)
      throw Error(kOverflow, "frontier of layer " + std::to_string(layer) +
                                 " exceeds the plan capacity (" + std::to_string(cap) + ")");
    cudaStream_t st = plan->stream;
    if (n_dst)
      CB_CUDA(cudaMemcpyAsync(D, d_dst, n_dst * 4, cudaMemcpyDeviceToDevice, st));
    if (layer == 0) {
      const Variates v = make_variates(sched);
      CB_CUDA(cudaMemcpyAsync(plan->var, &v, sizeof(Variates), cudaMemcpyHostToDevice, st));
      plan->seeds_off.assign({0, n_dst});
      plan->mode = CB_MODE_COOP;
    }
    const bool smooth = sched->kappa != cbdev::kKappaInf && sched->kappa >= 2;
    launch_batch_begin(w.sync, nullptr, nullptr, nullptr, nullptr, 0, 0, st);
    const RelabelArgs none{};
    enqueue_layer(plan, w, 0, layer, D, cap, n_dst, w.bm[0], none, 0, smooth,
                  extract_args(w, w.bm[0], nullptr, b.src, b.cap_src,
                               &plan->meta_at(0, layer)->n_src, nullptr, 3 * layer + 2,
                               8 * layer + 4));
    launch_relabel(relabel_args(w.bm[0], b, D, plan->meta_at(0, layer)),
                   std::max(b.cap_edges, b.cap_dst), st);
    launch_clear(w.bm[0], b.src, &plan->meta_at(0, layer)->n_src, st);
    check_overflow(plan);
    *n_src = host_meta(plan, 0, layer).n_src;
    plan->have_batch = true;
    plan->dirty_mode = -1;
  });
}

int cb_plan_layer_src(cb_plan* plan, int layer, uint32_t** d_src) {
  return guard([&] {
    require(plan != nullptr && d_src != nullptr, "null argument");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    *d_src = plan->pe[0].L[layer].src;
  });
}

int cb_bucket_by_owner(cb_plan* plan, const uint32_t* d_ids, uint64_t n, const uint32_t* d_owner,
                       uint32_t parts, uint32_t* d_out, uint32_t* d_perm, uint64_t* counts) {
  return guard([&] {
    require(plan != nullptr && counts != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    bucket_by_owner(d_ids, n, d_owner, parts, d_out, d_perm, counts, plan->stream);
  });
}

int cb_merge_owned(cb_plan* plan, int layer, const uint32_t* d_recv, uint64_t n_recv,
                   uint32_t* d_next, uint64_t cap_next, uint64_t* n_next, uint32_t* d_rank) {
  return guard([&] {
    require(plan != nullptr && n_next != nullptr, "null argument");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    cudaStream_t st = plan->stream;
    unsigned long long* cnt = plan->scratch;
    launch_batch_begin(w.sync, nullptr, nullptr, nullptr, nullptr, 0, 0, st);
    mark_ids(d_recv, n_recv, w.bm[1].bits, w.bm[1].summ, st);
    launch_extract(extract_args(w, w.bm[1], nullptr, d_next, cap_next, cnt, nullptr,
                                3 * plan->L + layer, 8 * layer + 5),
                   st);
    CB_CUDA(cudaMemcpyAsync(cnt + 1, &n_recv, 8, cudaMemcpyHostToDevice, st));
    launch_rank(w.bm[1], d_recv, cnt + 1, d_rank, st);
    launch_clear(w.bm[1], d_next, cnt, st);
    check_overflow(plan);
    unsigned long long h = 0;
    CB_CUDA(cudaMemcpy(&h, cnt, 8, cudaMemcpyDeviceToHost));
    *n_next = h;
  });
}

int cb_scatter_u32(cb_plan* plan, const uint32_t* d_in, const uint32_t* d_perm, uint64_t n,
                   uint32_t* d_out) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    scatter_u32(d_in, d_perm, n, d_out, plan->stream);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int cb_scatter_rows(cb_plan* plan, const void* d_in, const uint32_t* d_perm, uint64_t n,
                    uint64_t row_bytes, void* d_out) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    scatter_rows(d_in, d_perm, n, row_bytes, d_out, plan->stream);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int cb_features_synth_shard(const cb_graph* g, const cb_partition* pm, uint32_t part,
                            uint32_t dim, int dtype, uint64_t seed, cb_features** out) {
  return guard([&] {
    require(g != nullptr && pm != nullptr && out != nullptr, "null argument");
    require(part < pm->parts, "part index out of range");
    require(dim >= 1, "feature dim must be >= 1");
    require(dtype == CB_F64 || dtype == CB_F32 || dtype == CB_F16, "unknown dtype");
    DeviceGuard dg(g->g.device);
    auto f = std::make_unique<cb_features>();
    f->device = g->g.device;
    f->dim = dim;
    f->dtype = dtype;
    f->seed = seed;
    const uint64_t es = dtype == CB_F64 ? 8 : (dtype == CB_F32 ? 4 : 2);
    f->row_bytes = es * dim;
    const uint64_t r0 = pm->shard_off[part], r1 = pm->shard_off[part + 1];
    f->n_rows = g->g.n;  // addressable by global row id of owned vertices
    f->shard_rows = r1 - r0;
    f->shard_r0 = r0;
    unsigned char* shard = f->mem.alloc<unsigned char>((r1 - r0) * f->row_bytes);
    f->table = shard - r0 * f->row_bytes;  // virtual base: row_map[v] indexes it
    f->row_map = f->mem.alloc<uint32_t>(g->g.n);
    CB_CUDA(cudaMemcpy(f->row_map, pm->row_map, g->g.n * 4, cudaMemcpyDeviceToDevice));
    launch_synth(seed, dim, dtype, r1 - r0, pm->members + r0, 0, shard, nullptr);
    CB_CUDA(cudaDeviceSynchronize());
    *out = f.release();
  });
}

int cb_gather_rows(const cb_features* f, const uint32_t* d_ids, uint64_t n, void* d_out,
                   void* stream) {
  return guard([&] {
    require(f != nullptr, "null features");
    DeviceGuard dg(f->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    launch_gather(f->table, vec_bytes_for(f->row_bytes), f->row_bytes, d_ids, nullptr, n,
                  f->row_map, d_out, st);
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

int cb_memcpy(void* dst, const void* src, uint64_t bytes, int device) {
  return guard([&] {
    if (!bytes) return;
    DeviceGuard dg(device);
    CB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  });
}

int cb_plan_graph_profile(cb_plan* plan, const uint32_t* d_seeds, const cb_sched* sched,
                          float* ms, int max_n, int* n) {
  return guard([&] {
    require(plan != nullptr && sched != nullptr && ms != nullptr && n != nullptr,
            "null argument");
    require(plan->exec_prof != nullptr, "no captured batch (call cb_plan_capture)");
    DeviceGuard dg(plan->device);
    cudaStream_t st = plan->stream;
    const uint64_t total = plan->cap_off[plan->P];
    if (d_seeds && total)
      CB_CUDA(cudaMemcpyAsync(plan->seeds, d_seeds, total * 4, cudaMemcpyDefault, st));
    const Variates v = make_variates(sched);
    CB_CUDA(cudaMemcpyAsync(plan->var, &v, sizeof(Variates), cudaMemcpyHostToDevice, st));
    if (plan->dirty_mode >= 0 && plan->dirty_mode != plan->cap_mode)
      for (uint32_t p = 0; p < plan->P; ++p) {
        const Dirty d = dirty_of(plan, p, plan->dirty_mode);
        launch_batch_begin(plan->pe[p].sync, d.bits, d.summ, d.list, d.count, d.cap,
                           plan->pe[p].bm[0].words_padded, st);
      }
    CB_CUDA(cudaGraphLaunch(plan->exec_prof, st));
    CB_CUDA(cudaStreamSynchronize(st));
    plan->dirty_mode = plan->cap_mode;
    plan->have_batch = true;
    plan->have_rows = true;
    int k = 0;
    const auto& ev = plan->graph_events;
    for (size_t i = 1; i < ev.size() && k < max_n; ++i, ++k)
      CB_CUDA(cudaEventElapsedTime(&ms[k], ev[i - 1], ev[i]));
    *n = k;
  });
}

int cb_plan_trace(cb_plan* plan, uint64_t* out, uint64_t n) {
  return guard([&] {
    require(plan != nullptr && out != nullptr, "null argument");
    require(plan->trace != nullptr, "tracing off (set CB_TRACE=1 before creating the plan)");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    CB_CUDA(cudaMemcpy(out, plan->trace, std::min<uint64_t>(n, kTraceSlots) * 8,
                       cudaMemcpyDeviceToHost));
  });
}

int cb_plan_launch_count(const cb_plan* plan, int mode, int with_gather, uint64_t* n) {
  return guard([&] {
    require(plan != nullptr && n != nullptr, "null argument");
    const uint64_t samp = (plan->kind == CB_NS || plan->kind == CB_RW) ? 4 : 3;  // incl. extract
    const uint64_t P = plan->P;
    const uint64_t L = plan->L;
    uint64_t k;
    if (mode == CB_MODE_COOP && P > 1)
      k = P + L * (P * (samp + 1) + 1 + P + 1);
    else
      k = P * (1 + L * samp + 1);
    if (with_gather) k += P;
    *n = k;
  });
}

// ------------------------------------------------------------- LRU cache --
int cb_cache_create(int device, uint64_t n_keys, uint64_t capacity, uint64_t row_bytes,
                    cb_cache** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(capacity >= 1, "LruCache: capacity must be >= 1");
    DeviceGuard dg(device);
    auto c = std::make_unique<cb_cache>();
    c->lru = std::make_unique<DeviceLru>(device, n_keys, capacity, row_bytes);
    CB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c.release();
  });
}

void cb_cache_destroy(cb_cache* c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->lru->device());
  delete c;
  cudaSetDevice(prev);
}

int cb_cache_access_trace(cb_cache* c, const uint32_t* keys, uint64_t n, uint8_t* miss) {
  return guard([&] {
    require(c != nullptr && (n == 0 || (keys != nullptr && miss != nullptr)), "null argument");
    DeviceGuard dg(c->lru->device());
    c->lru->access_trace(keys, n, miss, c->stream);
  });
}

int cb_cache_access_ids(cb_cache* c, const uint32_t* d_ids, uint64_t n, uint64_t order_key,
                        const cb_partition* pm, uint32_t part, const cb_features* backing,
                        void* d_rows_out, uint64_t* kept, void* stream) {
  NvtxRange nvtx_("cb.cache_access");
  return guard([&] {
    require(c != nullptr, "null cache");
    require(pm == nullptr || part < pm->parts, "part index out of range");
    require(d_rows_out == nullptr || backing != nullptr, "rows requested without a table");
    require(backing == nullptr || c->lru->row_bytes() == 0 ||
                backing->row_bytes == c->lru->row_bytes(),
            "cache row size does not match the feature table");
    DeviceGuard dg(c->lru->device());
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    CacheGatherSrc src;
    if (backing && d_rows_out) {
      src.table = backing->table;
      src.row_map = backing->row_map;
      src.rows_out = d_rows_out;
    }
    const uint64_t k = c->lru->access_ids(d_ids, n, order_key, pm ? pm->owner : nullptr,
                                          part, src, st);
    if (kept) *kept = k;
  });
}

int cb_cache_access_plan(cb_cache* c, cb_plan* plan, uint32_t part, uint64_t order_key,
                         const cb_partition* pm, uint32_t owner_part,
                         const cb_features* backing, void* d_rows_out, uint64_t* kept) {
  NvtxRange nvtx_("cb.cache_access_plan");
  return guard([&] {
    require(c != nullptr && plan != nullptr, "null argument");
    require_batch(plan, part, plan->L - 1);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const uint64_t n = host_meta(plan, part, plan->L - 1).n_src;
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    const uint32_t* ids = plan->pe[part].L[plan->L - 1].src;
    if (backing && !d_rows_out) {  // rows land in the plan's own row buffer
      require(pm == nullptr, "plan row buffer holds all input rows: no owner filter");
      prepare_rows(plan, backing);
      d_rows_out = plan->pe[part].rows;
      plan->have_rows = true;
    }
    CacheGatherSrc src;
    if (backing && d_rows_out) {
      require(c->lru->row_bytes() == 0 || backing->row_bytes == c->lru->row_bytes(),
              "cache row size does not match the feature table");
      src.table = backing->table;
      src.row_map = backing->row_map;
      src.rows_out = d_rows_out;
    }
    const uint64_t k = c->lru->access_ids(ids, n, order_key, pm ? pm->owner : nullptr,
                                          owner_part, src, plan->stream);
    if (kept) *kept = k;
  });
}

int cb_cache_access_host_ids(cb_cache* c, const uint32_t* ids, uint64_t n, uint64_t order_key,
                             const cb_partition* pm, uint32_t part, uint64_t* kept) {
  return guard([&] {
    require(c != nullptr && (n == 0 || ids != nullptr), "null argument");
    require(pm == nullptr || part < pm->parts, "part index out of range");
    DeviceGuard dg(c->lru->device());
    uint32_t* d = nullptr;
    CB_CUDA(cudaMalloc(&d, n * 4 + 16));
    uint64_t k = 0;
    try {
      CB_CUDA(cudaMemcpy(d, ids, n * 4, cudaMemcpyHostToDevice));
      k = c->lru->access_ids(d, n, order_key, pm ? pm->owner : nullptr, part, CacheGatherSrc{},
                             c->stream);
    } catch (...) {
      cudaFree(d);
      throw;
    }
    cudaFree(d);
    if (kept) *kept = k;
  });
}

int cb_cache_stats(const cb_cache* c, uint64_t* hits, uint64_t* misses, uint64_t* size) {
  return guard([&] {
    require(c != nullptr, "null cache");
    if (hits) *hits = c->lru->hits();
    if (misses) *misses = c->lru->misses();
    if (size) *size = c->lru->size();
  });
}

int cb_cache_reset_counters(cb_cache* c) {
  return guard([&] {
    require(c != nullptr, "null cache");
    c->lru->reset_counters();
  });
}

int cb_cache_resident(cb_cache* c, uint32_t* out, uint64_t cap_out, uint64_t* n) {
  return guard([&] {
    require(c != nullptr && n != nullptr, "null argument");
    DeviceGuard dg(c->lru->device());
    std::vector<uint32_t> r;
    c->lru->resident(r);
    require(out == nullptr || cap_out >= r.size(), "output buffer too small");
    if (out) std::memcpy(out, r.data(), r.size() * 4);
    *n = r.size();
  });
}

int cb_cache_storage(const cb_cache* c, const void** d_rows) {
  return guard([&] {
    require(c != nullptr && d_rows != nullptr, "null argument");
    *d_rows = c->lru->storage();
  });
}

// stack_fingerprint (cache.cpp:123-133): sequential mix64 fold over the
// downloaded blocks of part p, computed on the host.
int cb_stack_fingerprint(cb_plan* plan, uint32_t part, uint64_t* out) {
  return guard([&] {
    require(plan != nullptr && out != nullptr, "null argument");
    require_batch(plan, part, 0);
    uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int l = 0; l < plan->L; ++l) {
      uint64_t sz[6];
      if (cb_layer_sizes(plan, part, l, sz) != CB_OK) throw Error(kCuda, g_err);
      std::vector<uint32_t> dst(sz[0]), src(sz[1]), edges(2 * sz[2]);
      if (cb_download_block(plan, part, l, dst.data(), src.data(), edges.data(), nullptr) !=
          CB_OK)
        throw Error(kCuda, g_err);
      h = cbdev::mix64(h ^ static_cast<uint64_t>(l));
      for (uint32_t v : dst) h = cbdev::mix64(h ^ v);
      for (uint32_t v : src) h = cbdev::mix64(h ^ (0x100000000ULL | v));
      for (uint64_t e = 0; e < sz[2]; ++e)
        h = cbdev::mix64(h ^ ((static_cast<uint64_t>(edges[2 * e]) << 32) | edges[2 * e + 1]));
    }
    *out = h;
  });
}

// Fixed training order of run_dependent_experiment (cache.cpp:155-162):
// Fisher-Yates with j = (u64)(hash_uniform(seed, {kStreamSeedDraw, i}) * i).
int cb_shuffled_order(uint64_t n, uint64_t seed, uint32_t* out) {
  return guard([&] {
    require(out != nullptr || n == 0, "null argument");
    for (uint64_t v = 0; v < n; ++v) out[v] = static_cast<uint32_t>(v);
    const uint64_t pfx = cbdev::hstep(cbdev::hinit(seed), 8ULL);
    for (uint64_t i = n; i > 1; --i) {
      const double u = cbdev::ufb(cbdev::hstep(pfx, i));
      const uint64_t j = static_cast<uint64_t>(u * static_cast<double>(i));
      std::swap(out[i - 1], out[std::min(j, i - 1)]);
    }
  });
}

// Storage tier of a feature table: 1 = pinned host memory mapped into the
// device address space (rows then cross the host link on every miss),
// 0 = HBM. The row layout is unchanged.
int cb_features_set_tier(cb_features* f, int host) {
  return guard([&] {
    require(f != nullptr, "null features");
    DeviceGuard dg(f->device);
    require(f->shard_rows == 0, "host tier of a single-part shard table is not supported");
    const uint64_t rows = f->n_rows;
    const uint64_t bytes = rows * f->row_bytes;
    const bool on_host = f->host_base != nullptr;
    if (static_cast<bool>(host) == on_host) return;
    CB_CUDA(cudaDeviceSynchronize());
    if (host) {
      void* h = nullptr;
      CB_CUDA(cudaHostAlloc(&h, bytes + 64, cudaHostAllocMapped | cudaHostAllocPortable));
      CB_CUDA(cudaMemcpy(h, f->table, bytes, cudaMemcpyDeviceToHost));
      void* d = nullptr;
      CB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
      f->hbm_table = f->table;
      f->host_base = h;
      f->table = d;
    } else {
      CB_CUDA(cudaMemcpy(f->hbm_table, f->host_base, bytes, cudaMemcpyHostToDevice));
      CB_CUDA(cudaFreeHost(f->host_base));
      f->host_base = nullptr;
      f->table = f->hbm_table;
      f->hbm_table = nullptr;
    }
  });
}

int cb_plan_set_rw(cb_plan* plan, uint32_t rw_length, double rw_restart, uint32_t rw_walks) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(rw_length >= 1 && rw_walks >= 1, "sample_rw: rw_length and rw_walks must be >= 1");
    require(rw_restart >= 0.0 && rw_restart < 1.0, "sample_rw: rw_restart must be in [0, 1)");
    require(static_cast<uint64_t>(rw_length) * rw_walks <= kRwMaxVisits,
            "rw_walks * rw_length must be <= 512 on the device");
    plan->rw_length = rw_length;
    plan->rw_restart = rw_restart;
    plan->rw_walks = rw_walks;
    plan->drop_graphs();
  });
}

int cb_plan_meta_async(cb_plan* plan, void* host_dst, uint64_t* bytes) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    const uint64_t nb = sizeof(LayerMeta) * plan->P * (plan->L + 1);
    if (bytes) *bytes = nb;
    if (!host_dst) return;
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaMemcpyAsync(host_dst, plan->meta, nb, cudaMemcpyDeviceToHost, plan->stream));
  });
}

int cb_kernel_launches(uint64_t* n) {
  return guard([&] {
    require(n != nullptr, "null argument");
    *n = g_kernel_launches.load();
  });
}

int cb_plan_input_ids(cb_plan* plan, uint32_t part, const uint32_t** d_ids, uint64_t* n) {
  return guard([&] {
    require(plan != nullptr && d_ids != nullptr && n != nullptr, "null argument");
    require_batch(plan, part, plan->L - 1);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    *n = host_meta(plan, part, plan->L - 1).n_src;
    *d_ids = plan->pe[part].L[plan->L - 1].src;
  });
}

// ------------------------------------------------ multi-process peer exchange --
// One part per rank (cb_plan_create_dist). Per layer l, with a cross-rank
// barrier (the caller's: an NCCL all-reduce on cb_plan_stream, or a host
// barrier) between the three calls:
//   cb_px_layer(l)  : sample layer l, then OR every src id into its owner's
//                     exchange bitmap over peer memory (build_exchange,
//                     coop.cpp:35-51) -- no counts, no host sync
//   cb_px_owner(l)  : the owner's sorted unique set S^{l+1}_q + word ranks
//                     (coop.cpp:44-51), next layer's frontier
//   cb_px_locate(l) : src_location from the owners' bitmaps (coop.cpp:53-62)
// and cb_px_gather pulls the input rows from the owners' shards
// (all_to_all_forward, coop.cpp:145-159). Everything is stream-ordered on the
// plan stream.
namespace {

PxState& px_of(cb_plan* pl) {
  require(pl->px != nullptr, "peer exchange not set up (cb_px_setup)");
  return *pl->px;
}

}  // namespace

int cb_px_setup(cb_plan* plan, const cb_partition* pm, uint32_t rank, void* handle_out) {
  return guard([&] {
    require(plan != nullptr && pm != nullptr && handle_out != nullptr, "null argument");
    require(plan->dist_world > 0, "peer exchange needs a dist plan (cb_plan_create_dist)");
    require(pm->parts == plan->dist_world, "partition part count != world size");
    require(plan->dist_world <= static_cast<uint32_t>(kMaxParts), "peer exchange: world <= 16");
    require(rank < plan->dist_world, "rank out of range");
    DeviceGuard dg(plan->device);
    auto px = std::make_unique<PxState>();
    px->rank = rank;
    px->world = plan->dist_world;
    px->owner = pm->owner;
    const uint64_t n = plan->g->g.n;
    const uint64_t words = ceil_div(n, 32);
    const uint64_t wp = ceil_div(std::max<uint64_t>(words, 1), kExtractTileWords) * kExtractTileWords;
    const bool summ = wp > kExtractBigWords;
    const uint64_t per = (2 * wp + (summ ? wp / 32 : 0)) * 4;
    px->region_bytes = 2 * per;
    CB_CUDA(cudaMalloc(&px->region, px->region_bytes));
    CB_CUDA(cudaMemset(px->region, 0, px->region_bytes));
    for (int s = 0; s < 2; ++s) {
      uint32_t* base = reinterpret_cast<uint32_t*>(static_cast<char*>(px->region) + s * per);
      Bitmap& b = px->slot[s];
      b.words = words;
      b.words_padded = wp;
      b.bits = base;
      b.wprefix = base + wp;
      b.summ = summ ? base + 2 * wp : nullptr;
      px->peers[s] = PxPeers{};
      px->peers[s].bits[rank] = b.bits;
      px->peers[s].summ[rank] = b.summ;
      px->peers[s].pre[rank] = b.wprefix;
    }
    CB_CUDA(cudaMalloc(&px->send, plan->L * px->world * 8 + 8));
    CB_CUDA(cudaMemset(px->send, 0, plan->L * px->world * 8 + 8));
    CB_CUDA(cudaMalloc(&px->d_fbase, kMaxParts * sizeof(void*)));
    px->fbase.assign(kMaxParts, nullptr);
    px->slot_of.assign(plan->L, 0);
    cudaIpcMemHandle_t h;
    CB_CUDA(cudaIpcGetMemHandle(&h, px->region));
    std::memcpy(handle_out, &h, sizeof(h));
    plan->px = std::move(px);
  });
}

int cb_px_connect(cb_plan* plan, uint32_t q, const void* handle) {
  return guard([&] {
    require(plan != nullptr && handle != nullptr, "null argument");
    PxState& px = px_of(plan);
    require(q < px.world && q != px.rank, "peer rank out of range (or self)");
    DeviceGuard dg(plan->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    CB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    px.opened.push_back(p);
    const uint64_t per = px.region_bytes / 2;
    for (int s = 0; s < 2; ++s) {
      uint32_t* base = reinterpret_cast<uint32_t*>(static_cast<char*>(p) + s * per);
      const uint64_t wp = px.slot[s].words_padded;
      px.peers[s].bits[q] = base;
      px.peers[s].pre[q] = base + wp;
      px.peers[s].summ[q] = px.slot[s].summ ? base + 2 * wp : nullptr;
    }
  });
}

int cb_px_layer(cb_plan* plan, int layer, const uint32_t* seeds, uint64_t n_seeds,
                const cb_sched* sched) {
  NvtxRange nvtx_("cb.px_layer");
  return guard([&] {
    require(plan != nullptr && sched != nullptr, "null argument");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    LayerBufs& b = w.L[layer];
    cudaStream_t st = plan->stream;
    uint32_t* D = (layer == 0) ? plan->seeds : b.dst;
    const uint64_t cap = (layer == 0) ? plan->max_seeds : b.cap_dst;
    if (layer == 0) {
      require(seeds != nullptr || n_seeds == 0, "null seeds");
      require(n_seeds <= plan->max_seeds, "more seeds than the plan's max_seeds_per_part");
      if (n_seeds)
        CB_CUDA(cudaMemcpyAsync(D, seeds, n_seeds * 4, cudaMemcpyDefault, st));
      const Variates v = make_variates(sched);
      CB_CUDA(cudaMemcpyAsync(plan->var, &v, sizeof(Variates), cudaMemcpyHostToDevice, st));
      CB_CUDA(cudaMemsetAsync(px.send, 0, plan->L * px.world * 8, st));
      plan->seeds_off.assign({0, n_seeds});
      plan->mode = CB_MODE_COOP;
    }
    const bool smooth = sched->kappa != cbdev::kKappaInf && sched->kappa >= 2;
    const int s = static_cast<int>(px.layer_ctr++ & 1);
    px.slot_of[layer] = s;
    launch_batch_begin(w.sync, nullptr, nullptr, nullptr, nullptr, 0, 0, st);
    const RelabelArgs none{};
    enqueue_layer(plan, w, 0, layer, D, cap, layer == 0 ? n_seeds : ~0ULL, w.bm[0], none, 0,
                  smooth,
                  extract_args(w, w.bm[0], nullptr, b.src, b.cap_src,
                               &plan->meta_at(0, layer)->n_src, nullptr, 3 * layer + 2,
                               8 * layer + 4));
    launch_relabel(relabel_args(w.bm[0], b, D, plan->meta_at(0, layer)),
                   std::max(b.cap_edges, b.cap_dst), st);
    launch_clear(w.bm[0], b.src, &plan->meta_at(0, layer)->n_src, st);
    launch_px_route(b.src, &plan->meta_at(0, layer)->n_src, b.cap_src, px.owner, px.peers[s],
                    px.send + static_cast<uint64_t>(layer) * px.world, st);
    plan->have_batch = true;
    plan->have_rows = false;
    plan->dirty_mode = -1;
  });
}

int cb_px_owner(cb_plan* plan, int layer) {
  NvtxRange nvtx_("cb.px_owner");
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    const int s = px.slot_of[layer];
    uint32_t* next = (layer + 1 < plan->L) ? w.L[layer + 1].dst : w.owner_final;
    const uint64_t cap = (layer + 1 < plan->L) ? w.L[layer + 1].cap_dst : w.cap_final;
    // the other slot was last read by the previous layer's locates, which
    // every rank finished before the barrier that precedes this call
    launch_extract(extract_args(w, px.slot[s], &px.slot[s ^ 1], next, cap,
                                &plan->meta_at(0, layer + 1)->n_dst, nullptr,
                                3 * plan->L + layer, 8 * layer + 5),
                   plan->stream);
  });
}

int cb_px_locate(cb_plan* plan, int layer) {
  NvtxRange nvtx_("cb.px_locate");
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    LayerBufs& b = w.L[layer];
    launch_px_locate(b.src, &plan->meta_at(0, layer)->n_src, b.cap_src, px.owner,
                     px.peers[px.slot_of[layer]], w.loc_part[layer], w.loc_row[layer],
                     plan->stream);
  });
}

int cb_px_finish(cb_plan* plan) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
  });
}

int cb_px_sizes(cb_plan* plan, int layer, uint64_t* n_src, uint64_t* n_owned) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    if (n_src) *n_src = host_meta(plan, 0, layer).n_src;
    if (n_owned) *n_owned = host_meta(plan, 0, layer + 1).n_dst;
  });
}

int cb_px_download(cb_plan* plan, int layer, uint64_t* send_row, uint32_t* loc_part,
                   uint32_t* loc_row, uint32_t* owned) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    PeWork& w = plan->pe[0];
    const uint64_t n = host_meta(plan, 0, layer).n_src;
    const uint64_t no = host_meta(plan, 0, layer + 1).n_dst;
    if (send_row) {
      std::vector<unsigned long long> h(px.world);
      CB_CUDA(cudaMemcpy(h.data(), px.send + static_cast<uint64_t>(layer) * px.world,
                         px.world * 8, cudaMemcpyDeviceToHost));
      for (uint32_t q = 0; q < px.world; ++q) send_row[q] = h[q];
    }
    if (loc_part && n) CB_CUDA(cudaMemcpy(loc_part, w.loc_part[layer], n * 4, cudaMemcpyDeviceToHost));
    if (loc_row && n) CB_CUDA(cudaMemcpy(loc_row, w.loc_row[layer], n * 4, cudaMemcpyDeviceToHost));
    if (owned && no) {
      const uint32_t* d = (layer + 1 < plan->L) ? w.L[layer + 1].dst : w.owner_final;
      CB_CUDA(cudaMemcpy(owned, d, no * 4, cudaMemcpyDeviceToHost));
    }
  });
}

int cb_features_export(const cb_features* f, void* handle_out, uint64_t* shard_r0) {
  return guard([&] {
    require(f != nullptr && handle_out != nullptr, "null argument");
    require(f->shard_rows > 0, "export needs a single-part shard table (cb_features_synth_shard)");
    require(f->host_base == nullptr, "export of a host-tier table is not supported");
    DeviceGuard dg(f->device);
    void* base = static_cast<unsigned char*>(f->table) + f->shard_r0 * f->row_bytes;
    cudaIpcMemHandle_t h;
    CB_CUDA(cudaIpcGetMemHandle(&h, base));
    std::memcpy(handle_out, &h, sizeof(h));
    if (shard_r0) *shard_r0 = f->shard_r0;
  });
}

int cb_px_connect_features(cb_plan* plan, uint32_t q, const void* handle, uint64_t shard_r0,
                           const cb_features* local) {
  return guard([&] {
    require(plan != nullptr && local != nullptr, "null argument");
    PxState& px = px_of(plan);
    require(q < px.world, "peer rank out of range");
    DeviceGuard dg(plan->device);
    px.frow_bytes = local->row_bytes;
    if (q == px.rank) {
      px.fbase[q] = static_cast<const unsigned char*>(local->table);
    } else {
      require(handle != nullptr, "null handle");
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handle, sizeof(h));
      void* p = nullptr;
      CB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      px.fopened.push_back(p);
      px.fbase[q] = static_cast<const unsigned char*>(p) - shard_r0 * local->row_bytes;
    }
    CB_CUDA(cudaMemcpy(px.d_fbase, px.fbase.data(), kMaxParts * sizeof(void*),
                       cudaMemcpyHostToDevice));
  });
}

int cb_px_gather(cb_plan* plan, const cb_features* local) {
  NvtxRange nvtx_("cb.px_gather");
  return guard([&] {
    require(plan != nullptr && local != nullptr, "null argument");
    require(plan->have_batch, "no sampled batch in this plan");
    PxState& px = px_of(plan);
    for (uint32_t q = 0; q < px.world; ++q)
      require(px.fbase[q] != nullptr, "feature shard of a rank not connected");
    DeviceGuard dg(plan->device);
    prepare_rows(plan, local);
    PeWork& w = plan->pe[0];
    const int L = plan->L;
    launch_px_gather(px.d_fbase, px.owner, local->row_map, local->row_bytes, w.L[L - 1].src,
                     &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, plan->stream);
    plan->have_rows = true;
  });
}

}  // extern "C"

// ------------------------------------------------- GCN training step (f1) --
// GcnModel (coop.hpp:105-135) on the device and coop_train_step /
// indep_train_step (coop.cpp:438-610) over the plan's last batch: the
// forward pass mean-aggregates each block's sampled in-neighbours, applies
// W and tanh (identity at block 0), moves hidden rows to the requesters with
// the batch's exchange records (all_to_all_forward), takes the softmax
// cross-entropy of the seeds, and runs the backward pass with the owner-side
// gradient sums (all_to_all_reverse_sum). FP64 in the reference's
// accumulation order (train.cu).
struct cb_model {
  int device = 0;
  int L = 0;
  bool tanh_hidden = true;
  std::vector<uint32_t> rows, cols;
  std::vector<double*> w;
  ~cb_model() {
    for (double* p : w) if (p) cudaFree(p);
  }
};

namespace {

struct TmpArena {
  std::vector<void*> ptrs;
  template <typename T>
  T* get(uint64_t n) {
    void* p = nullptr;
    CB_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T) + 16));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~TmpArena() {
    for (void* p : ptrs) cudaFree(p);
  }
};

struct U32ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// out[0..n] = exclusive prefix of the u32 counts (out[n] = total)
void scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* out, TmpArena& A, cudaStream_t st) {
  auto it = thrust::make_transform_iterator(cnt, U32ToU64{});
  size_t bytes = 0;
  CB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, static_cast<int64_t>(n + 1), st));
  void* tmp = A.get<unsigned char>(bytes);
  CB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, it, out, static_cast<int64_t>(n + 1), st));
}

__global__ void src_hist_kernel(const uint2* __restrict__ edges, uint64_t n, uint32_t* cnt,
                                uint32_t* key, uint32_t* val) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&cnt[edges[e].x], 1u);
    key[e] = edges[e].x;
    val[e] = static_cast<uint32_t>(e);
  }
}

__global__ void owner_key_kernel(const uint32_t* __restrict__ part, const uint32_t* __restrict__ row,
                                 uint64_t n, const uint64_t* __restrict__ owner_base,
                                 uint64_t g0, uint32_t* cnt, uint64_t* key, uint64_t* val) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = owner_base[part[j]] + row[j];
    atomicAdd(&cnt[k], 1u);
    key[g0 + j] = k;
    val[g0 + j] = g0 + j;
  }
}

int grid_of_n(uint64_t n) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)));
}

}  // namespace

extern "C" {

int cb_gcn_model_init(int device, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                      int num_layers, uint64_t seed, cb_model** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(num_layers >= 1, "GcnModel: num_layers must be >= 1");
    require(in_dim >= 1 && hidden >= 1 && classes >= 1, "GcnModel: dims must be >= 1");
    DeviceGuard dg(device);
    auto m = std::make_unique<cb_model>();
    m->device = device;
    m->L = num_layers;
    for (int l = 0; l < num_layers; ++l) {
      // GcnModel::init (coop.cpp:334-357): weights[l] is used at block l
      const uint32_t rows = (l == num_layers - 1) ? in_dim : hidden;
      const uint32_t cols = (l == 0) ? classes : hidden;
      std::vector<double> w(static_cast<uint64_t>(rows) * cols);
      const double scale = 1.0 / std::sqrt(static_cast<double>(rows));
      const uint64_t pfx = cbdev::hstep(cbdev::hstep(cbdev::hinit(seed), 11ULL),
                                        static_cast<uint64_t>(l));
      for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
          const double u = cbdev::ufb(cbdev::hstep(cbdev::hstep(pfx, i), j));
          volatile double t = 2.0 * u;  // no contraction: (2u - 1) * scale as two roundings
          w[i * cols + j] = (t - 1.0) * scale;
        }
      double* d = nullptr;
      CB_CUDA(cudaMalloc(&d, w.size() * 8));
      CB_CUDA(cudaMemcpy(d, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
      m->rows.push_back(rows);
      m->cols.push_back(cols);
      m->w.push_back(d);
    }
    *out = m.release();
  });
}

int cb_gcn_model_weights(cb_model* m, int layer, double* host, int upload, uint64_t* rows,
                         uint64_t* cols) {
  return guard([&] {
    require(m != nullptr, "null model");
    require(layer >= 0 && layer < m->L, "layer index out of range");
    DeviceGuard dg(m->device);
    const uint64_t n = static_cast<uint64_t>(m->rows[layer]) * m->cols[layer];
    if (rows) *rows = m->rows[layer];
    if (cols) *cols = m->cols[layer];
    if (!host) return;
    if (upload) CB_CUDA(cudaMemcpy(m->w[layer], host, n * 8, cudaMemcpyHostToDevice));
    else CB_CUDA(cudaMemcpy(host, m->w[layer], n * 8, cudaMemcpyDeviceToHost));
  });
}

void cb_gcn_model_destroy(cb_model* m) {
  if (!m) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  delete m;
  cudaSetDevice(prev);
}

int cb_train_step(cb_plan* pl, const cb_features* f, uint32_t classes, cb_model* m,
                  double* loss_out, double* grad_w_out) {
  NvtxRange nvtx_("cb.train_step");
  return guard([&] {
    require(pl != nullptr && f != nullptr && m != nullptr && loss_out != nullptr,
            "null argument");
    require(pl->have_batch, "no sampled batch in this plan");
    require(f->dtype == CB_F64, "train step: the feature table must be f64 (FeatureStore)");
    require(m->L == pl->L, "train step: model depth does not match layer count");
    require(m->rows[pl->L - 1] == f->dim, "train step: model input dim does not match store");
    require(classes >= 1 && m->cols[0] == classes, "train step: class count mismatch");
    DeviceGuard dg(pl->device);
    check_overflow(pl);
    const uint32_t P = pl->P;
    const int L = pl->L;
    const bool coop = pl->coop_active();
    cudaStream_t st = pl->stream;
    TmpArena A;
    // counts of the batch (one host read)
    std::vector<std::vector<LayerMeta>> M(P, std::vector<LayerMeta>(L + 1));
    for (uint32_t p = 0; p < P; ++p)
      CB_CUDA(cudaMemcpy(M[p].data(), pl->meta_at(p, 0), sizeof(LayerMeta) * (L + 1),
                         cudaMemcpyDeviceToHost));
    uint64_t total_seeds = 0;
    for (uint32_t p = 0; p < P; ++p) total_seeds += M[p][0].n_dst;
    require(total_seeds > 0, coop ? "coop_train_step: no seeds" : "indep_train_step: no seeds");
    auto dst_of = [&](uint32_t p, int l) -> const uint32_t* {
      if (l == 0) return pl->seeds + pl->seeds_off[p];
      return pl->own_dst() ? pl->pe[p].L[l].dst : pl->pe[p].L[l - 1].src;
    };
    // input rows of every part, requester-aligned (load_rows + all_to_all_forward)
    prepare_rows(pl, f);
    enqueue_gather(pl, f);
    std::vector<std::vector<double*>> hin(L, std::vector<double*>(P)), agg(L, std::vector<double*>(P)),
        out(L, std::vector<double*>(P));
    std::vector<std::vector<uint32_t*>> deg(L, std::vector<uint32_t*>(P));
    for (int l = L - 1; l >= 0; --l) {
      const uint32_t din = m->rows[l], dout = m->cols[l];
      const bool act = (l > 0) && m->tanh_hidden;
      for (uint32_t p = 0; p < P; ++p) {
        const LayerBufs& b = pl->pe[p].L[l];
        const uint64_t nd = M[p][l].n_dst, ne = M[p][l].n_edges;
        if (l == L - 1) hin[l][p] = static_cast<double*>(pl->pe[p].rows);
        else if (!coop) hin[l][p] = out[l + 1][p];
        deg[l][p] = A.get<uint32_t>(nd);
        CB_CUDA(cudaMemsetAsync(deg[l][p], 0, std::max<uint64_t>(nd, 1) * 4, st));
        launch_in_degrees(b.edges, ne, deg[l][p], st);
        uint64_t* off = A.get<uint64_t>(nd + 1);
        scan_counts(deg[l][p], nd, off, A, st);
        agg[l][p] = A.get<double>(nd * din);
        launch_aggregate(b.edges, deg[l][p], off, b.dst_pos, nd, hin[l][p], din, agg[l][p], st);
        out[l][p] = A.get<double>(nd * dout);
        launch_dense(agg[l][p], nd, din, m->w[l], dout, act, out[l][p], st);
      }
      if (coop && l > 0) {  // all_to_all_forward of block l's outputs to block l-1's sources
        const double** owners = A.get<const double*>(P);
        std::vector<const double*> h(out[l].begin(), out[l].end());
        CB_CUDA(cudaMemcpyAsync(owners, h.data(), P * sizeof(void*), cudaMemcpyHostToDevice, st));
        CB_CUDA(cudaStreamSynchronize(st));
        for (uint32_t p = 0; p < P; ++p) {
          const uint64_t ns = M[p][l - 1].n_src;
          hin[l - 1][p] = A.get<double>(ns * dout);
          launch_row_forward(owners, pl->pe[p].loc_part[l - 1], pl->pe[p].loc_row[l - 1], ns,
                             dout, hin[l - 1][p], st);
        }
      }
    }
    // loss on the seeds, gradient rows scaled by the global mean
    const double scale = 1.0 / static_cast<double>(total_seeds);
    const uint32_t C = classes;
    std::vector<std::vector<double*>> grad(L + 1, std::vector<double*>(P, nullptr));
    double loss_sum = 0.0;
    for (uint32_t p = 0; p < P; ++p) {
      const uint64_t n0 = M[p][0].n_dst;
      double* rl = A.get<double>(n0);
      grad[0][p] = A.get<double>(n0 * C);
      launch_softmax_ce(out[0][p], n0, C, dst_of(p, 0), f->seed, scale, rl, grad[0][p], st);
      std::vector<double> h(n0);
      if (n0) CB_CUDA(cudaMemcpyAsync(h.data(), rl, n0 * 8, cudaMemcpyDeviceToHost, st));
      CB_CUDA(cudaStreamSynchronize(st));
      for (double x : h) loss_sum += x;
    }
    *loss_out = loss_sum * scale;
    // backward with owner-side gradient accumulation between layers
    uint64_t gw_off = 0;
    for (int l = 0; l < L; ++l) {
      const uint32_t din = m->rows[l], dout = m->cols[l];
      const bool act = (l > 0) && m->tanh_hidden;
      const uint64_t nw = static_cast<uint64_t>(din) * dout;
      double* gw = A.get<double>(nw);
      CB_CUDA(cudaMemsetAsync(gw, 0, nw * 8, st));
      double* gwp = A.get<double>(nw);
      uint64_t req_total = 0;
      std::vector<uint64_t> req_off(P + 1, 0);
      for (uint32_t p = 0; p < P; ++p) req_off[p + 1] = req_off[p] + M[p][l].n_src;
      req_total = req_off[P];
      double* gh_all = A.get<double>(req_total * din);
      for (uint32_t p = 0; p < P; ++p) {
        const LayerBufs& b = pl->pe[p].L[l];
        const uint64_t nd = M[p][l].n_dst, ne = M[p][l].n_edges, ns = M[p][l].n_src;
        double* dp = grad[l][p];
        if (act) launch_tanh_grad(out[l][p], nd * dout, dp, st);
        launch_grad_w(agg[l][p], dp, nd, din, dout, gwp, st);
        launch_add(gw, gwp, nw, st);  // parts in order (the simulated all-reduce)
        double* dagg = A.get<double>(nd * din);
        launch_grad_agg(dp, m->w[l], nd, din, dout, dagg, st);
        // sources' edges in edge order (stable CSC) + the isolated dst of each source
        uint32_t* cnt = A.get<uint32_t>(ns);
        CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(ns, 1) * 4, st));
        uint32_t* key = A.get<uint32_t>(ne);
        uint32_t* val = A.get<uint32_t>(ne);
        uint32_t* key2 = A.get<uint32_t>(ne);
        uint32_t* val2 = A.get<uint32_t>(ne);
        if (ne) src_hist_kernel<<<grid_of_n(ne), 256, 0, st>>>(b.edges, ne, cnt, key, val);
        CB_LAUNCH("src_hist");
        uint64_t* soff = A.get<uint64_t>(ns + 1);
        scan_counts(cnt, ns, soff, A, st);
        cub::DoubleBuffer<uint32_t> kb(key, key2), vb(val, val2);
        size_t bytes = 0;
        CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, static_cast<int64_t>(ne), 0,
                                                32, st));
        void* tmp = A.get<unsigned char>(bytes);
        CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int64_t>(ne), 0, 32,
                                                st));
        int64_t* iso = A.get<int64_t>(ns);
        CB_CUDA(cudaMemsetAsync(iso, 0xff, std::max<uint64_t>(ns, 1) * 8, st));
        launch_iso_dst(deg[l][p], b.dst_pos, nd, iso, st);
        launch_grad_h_in(b.edges, vb.Current(), soff, deg[l][p], iso, ns, dagg, din,
                         gh_all + req_off[p] * din, st);
      }
      if (grad_w_out)
        CB_CUDA(cudaMemcpyAsync(grad_w_out + gw_off, gw, nw * 8, cudaMemcpyDeviceToHost, st));
      gw_off += nw;
      if (l + 1 < L) {
        if (!coop) {
          for (uint32_t p = 0; p < P; ++p) grad[l + 1][p] = gh_all + req_off[p] * din;
        } else {  // all_to_all_reverse_sum over the exchange of layer l
          std::vector<uint64_t> obase(P + 1, 0);
          for (uint32_t q = 0; q < P; ++q) obase[q + 1] = obase[q] + M[q][l + 1].n_dst;
          const uint64_t no = obase[P];
          uint64_t* d_obase = A.get<uint64_t>(P + 1);
          CB_CUDA(cudaMemcpyAsync(d_obase, obase.data(), (P + 1) * 8, cudaMemcpyHostToDevice, st));
          uint32_t* cnt = A.get<uint32_t>(no);
          CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(no, 1) * 4, st));
          uint64_t* key = A.get<uint64_t>(req_total);
          uint64_t* val = A.get<uint64_t>(req_total);
          uint64_t* key2 = A.get<uint64_t>(req_total);
          uint64_t* val2 = A.get<uint64_t>(req_total);
          for (uint32_t p = 0; p < P; ++p) {
            const uint64_t ns = M[p][l].n_src;
            if (ns)
              owner_key_kernel<<<grid_of_n(ns), 256, 0, st>>>(
                  pl->pe[p].loc_part[l], pl->pe[p].loc_row[l], ns, d_obase, req_off[p], cnt, key,
                  val);
            CB_LAUNCH("owner_key");
          }
          uint64_t* ooff = A.get<uint64_t>(no + 1);
          scan_counts(cnt, no, ooff, A, st);
          cub::DoubleBuffer<uint64_t> kb(key, key2), vb(val, val2);
          size_t bytes = 0;
          CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb,
                                                  static_cast<int64_t>(req_total), 0, 64, st));
          void* tmp = A.get<unsigned char>(bytes);
          CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb,
                                                  static_cast<int64_t>(req_total), 0, 64, st));
          double* oall = A.get<double>(no * din);
          launch_reverse_sum(ooff, vb.Current(), no, gh_all, din, oall, st);
          for (uint32_t q = 0; q < P; ++q) grad[l + 1][q] = oall + obase[q] * din;
        }
      }
    }
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
