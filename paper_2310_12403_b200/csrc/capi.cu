// libcoopbatch_b200 C-ABI (include/coopbatch_cuda.h) and the C++ orchestrator
// behind it: handle lifetimes, capacity planning, and the per-batch launch
// sequence of expand / indep_sample / coop_sample (samplers.cpp:340-354,
// coop.cpp:68-119) and the fused load_rows + all_to_all_forward gather
// (coop.cpp:145-159, 378-388). Every launch is asynchronous on the plan's
// stream; counts stay on the device (LayerMeta) so a batch never waits on the
// host. Contract violations raise cb::Error(kInput) -> CB_INPUT, mirroring
// coopbatch::InputError (common.hpp:12-15).
#include "capi_internal.h"
#include "result.h"

thread_local std::string cb::capi::g_err;

namespace cb {
std::atomic<unsigned long long> g_kernel_launches{0};
// Off by default: with 8 batches in flight the early-launched (waiting) CTAs
// of the next kernel take SM slots from the other batches' kernels
// (65.4 vs 67.4 us/step at c2, latency 148 vs 150 us). CB_PDL=1 enables it.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CB_PDL");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
}  // namespace cb

namespace cb {
namespace capi {

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
      // the scan space (stage: 8 B per position) is also bounded by a budget
      // that grows with the retries: sum_deg alone is m at large graphs (c4:
      // 1.6B positions = 13 GB of stage per plan for a 48M-position layer)
      const uint64_t scan_cap = std::min(
          sum_deg, sat_mul(kScanBudget, static_cast<uint64_t>(std::ceil(pl->grow))));
      max_tiles = std::max(max_tiles, ceil_div(scan_cap, kLaborTile) + 2);
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
      w.L[l].tile_list = pl->mem.alloc<uint2>(max_tiles);
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
  const bool tab = pl->kind == CB_LABOR0 && n <= kVtabMaxVerts;
  // parts run concurrently (own stage + variate table each) when that fits a
  // modest budget; otherwise one after another on the plan stream, sharing them
  const uint64_t per_part = stage_tiles * kLaborTile * 8 + (tab ? n * 8 : 0);
  pl->part_concurrent = P > 1 && sat_mul(per_part, P) <= (8ULL << 30);
  if (pl->part_concurrent && pl->part_st.size() != P) {
    for (uint32_t p = 0; p < P; ++p) {
      cudaStream_t s;
      cudaEvent_t e;
      CB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      CB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      pl->part_st.push_back(s);
      pl->ev_join.push_back(e);
    }
    CB_CUDA(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming));
  }
  uint2* stage = nullptr;
  double* vt = nullptr;
  for (PeWork& w : pl->pe) {
    if (!stage || pl->part_concurrent) {
      stage = pl->mem.alloc<uint2>(stage_tiles * kLaborTile + 32);
      vt = tab ? pl->mem.alloc<double>(n) : nullptr;
    }
    w.sync.stage = stage;
    w.sync.vtab = vt;
  }
  pl->vtab = vt;
  pl->meta = pl->mem.alloc<LayerMeta>(static_cast<uint64_t>(P) * (L + 1));
  CB_CUDA(cudaMemset(pl->meta, 0, sizeof(LayerMeta) * P * (L + 1)));
  pl->send_counts = pl->mem.alloc<unsigned long long>(static_cast<uint64_t>(L) * P * P);
  pl->var = pl->mem.alloc<Variates>(P);  // one per part (per-part schedules)
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

// The smoothed (FP64 threshold) kernel path: a smoothing schedule, or the
// caller's variate table of cb_plan_set_variate_table.
bool smooth_of(const cb_plan* pl, const cb_sched* s) {
  if (pl->var_source) return pl->ext_vtab != nullptr || pl->var_source->smoothed != 0;
  return pl->ext_vtab != nullptr || (s->kappa != cbdev::kKappaInf && s->kappa >= 2);
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

constexpr uint32_t kResolvePendCap = 1u << 16;

// The resolve buffers of a plan (allocated the first time a smoothed batch
// runs): the device Resolve struct, the pending list and its count.
void resolve_alloc(cb_plan* pl) {
  if (pl->d_rs) return;
  CB_CUDA(cudaMalloc(&pl->d_rs, sizeof(cbdev::Resolve)));
  CB_CUDA(cudaMalloc(&pl->rs_pend, sizeof(cbdev::ResolvePend) * kResolvePendCap));
  CB_CUDA(cudaMalloc(&pl->rs_npend, 8));
  CB_CUDA(cudaMemset(pl->rs_npend, 0, 8));
  cbdev::Resolve r{};
  r.cap_pend = kResolvePendCap;
  r.pend = pl->rs_pend;
  r.n_pend = pl->rs_npend;
  r.perturb = pl->perturb;
  h2d_sync(pl->d_rs, &r, sizeof(r));
}

// The same variates for every part (the reference's single schedule), or one
// schedule per part (cb_sample_multi).
void upload_variates(cb_plan* pl, const cb_sched* s, uint32_t n_sched, cudaStream_t st) {
  std::vector<Variates> v(pl->P);
  for (uint32_t p = 0; p < pl->P; ++p) {
    v[p] = pl->var_source ? *pl->var_source : make_variates(s + (n_sched > 1 ? p : 0));
    if (pl->ext_vtab) v[p].smoothed = 2;  // caller variate table (sample_labor0)
    v[p].guard = pl->guard;
    v[p].part = static_cast<int>(p);
  }
  // in-band decisions are recorded per (part, layer, vertex[, position])
  if (v[0].smoothed == 1) {
    resolve_alloc(pl);
    for (auto& x : v) x.rs = pl->d_rs;
  }
  if (pl->rs_npend) CB_CUDA(cudaMemsetAsync(pl->rs_npend, 0, 8, st));
  CB_CUDA(cudaMemcpyAsync(pl->var, v.data(), sizeof(Variates) * pl->P, cudaMemcpyHostToDevice,
                          st));  // pageable source: staged before the call returns
}

// Seed offsets index the plan's seed buffer (P * max_seeds ids): they start
// at 0, never decrease, and no part exceeds max_seeds.
void check_offsets(const cb_plan* pl, const uint64_t* off) {
  require(off[0] == 0, "seed offsets must start at 0");
  for (uint32_t p = 0; p < pl->P; ++p) {
    require(off[p + 1] >= off[p], "seed offsets must be nondecreasing");
    if (off[p + 1] - off[p] > pl->max_seeds)
      throw Error(kInput, "part " + std::to_string(p) +
                              " has more seeds than the plan's max_seeds_per_part");
  }
}

void check_seeds_host(const cb_plan* pl, const uint32_t* flat, const uint64_t* off) {
  const uint64_t n = pl->g->g.n;
  check_offsets(pl, off);
  for (uint32_t p = 0; p < pl->P; ++p) {
    for (uint64_t i = off[p]; i < off[p + 1]; ++i)
      if (flat[i] >= n)
        throw Error(kInput, "vertex id " + std::to_string(flat[i]) + " out of range [0, " +
                                std::to_string(n) + ")");
  }
}

void require_mode(const cb_plan* pl, int mode) {
  require(mode == CB_MODE_COOP || mode == CB_MODE_INDEP, "unknown sampling mode");
  require(mode != CB_MODE_COOP || pl->P == 1 || pl->pm != nullptr,
          "cooperative sampling needs a partition (plan created without one)");
}

void check_ownership_host(const cb_plan* pl, const uint32_t* flat, const uint64_t* off) {
  // coop_sample: every seed must be owned by its claimed part (coop.cpp:75-81)
  if (pl->P <= 1) return;
  const uint64_t total = off[pl->P];
  std::vector<uint32_t> owners(total);
  std::vector<uint32_t> seeds(flat, flat + total);
  // gather owner[seed] on the device: tiny (one value per seed)
  DevBuf b_ids(total * 4 + 4), b_out(total * 4 + 4), b_cnt(8);
  uint32_t* d_ids = b_ids.as<uint32_t>();
  uint32_t* d_out = b_out.as<uint32_t>();
  // uploads ordered on the plan stream: a pageable cudaMemcpy runs on the
  // legacy stream and may return before its DMA lands
  CB_CUDA(cudaMemcpyAsync(d_ids, seeds.data(), total * 4, cudaMemcpyHostToDevice, pl->stream));
  // reuse the feature gather kernel with a 4-byte "row" = owner[v]
  unsigned long long* d_cnt = b_cnt.as<unsigned long long>();
  const unsigned long long t = total;
  CB_CUDA(cudaMemcpyAsync(d_cnt, &t, 8, cudaMemcpyHostToDevice, pl->stream));
  launch_gather(pl->pm->owner, 4, 4, d_ids, d_cnt, total, nullptr, d_out, pl->stream);
  CB_CUDA(cudaStreamSynchronize(pl->stream));
  CB_CUDA(cudaMemcpy(owners.data(), d_out, total * 4, cudaMemcpyDeviceToHost));
  for (uint32_t p = 0; p < pl->P; ++p)
    for (uint64_t i = off[p]; i < off[p + 1]; ++i)
      if (owners[i] != p)
        throw Error(kInput, "coop_sample: seed " + std::to_string(flat[i]) +
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
  fa.layer = l + pl->layer_base;
  fa.var = pl->var + p;
  fa.set_bits = set_bm.bits;
  fa.set_summ = set_bm.summ;
  fa.act = b.act;
  fa.tile_first = b.tile_first;
  fa.out_prefix = b.out_prefix;
  fa.slots = b.slots;
  fa.cap_edges = b.cap_edges;
  fa.cap_tiles = w.sync.max_tiles - 1;
  const bool lists = pl->kind == CB_LABOR0 || pl->kind == CB_FULL;
  fa.tile_list = lists ? b.tile_list : nullptr;
  fa.list_ctr = w.sync.tickets + Sync::kListTicket + 2 * l;
  fa.list_cap = w.sync.max_tiles;
  fa.ticket = w.sync.tickets + 3 * l;
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
  la.layer = l + pl->layer_base;
  la.var = pl->var + p;
  la.bits = set_bm.bits;
  la.summ = set_bm.summ;
  la.edges = b.edges;
  la.slots = b.slots;
  la.tile_list = (pl->kind == CB_LABOR0 || pl->kind == CB_FULL) ? b.tile_list : nullptr;
  la.list_ctr = w.sync.tickets + Sync::kListTicket + 2 * l;
  la.pure_ticket = w.sync.tickets + Sync::kPureTicket + l;
  la.list_cap = w.sync.max_tiles;
  la.keep_words = w.sync.keep_words;
  la.stage = w.sync.stage;
  la.vtab = pl->ext_vtab ? pl->ext_vtab : w.sync.vtab;
  la.n_vert = pl->ext_vtab ? 0 : pl->g->g.n;  // 0: the table is always used, never rebuilt
  la.cap_edges = b.cap_edges;
  la.ticket = w.sync.tickets + 3 * l + 1;
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
                       const ExtractArgs& ex, cudaStream_t stream) {
  NvtxRange nvtx_("cb.layer");
  const DeviceGraph& g = pl->g->g;
  const LayerBufs& b = w.L[l];
  cudaStream_t st = stream ? stream : pl->stream;
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
    ra.weights = g.weights;
    ra.layer = l + pl->layer_base;
    ra.k = pl->fanouts[l];
    ra.walks = pl->rw_walks;
    ra.length = pl->rw_length;
    ra.restart = pl->rw_restart;
    ra.var = pl->var + p;
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

// Look-back status words carry an 18-bit epoch. Every device epoch bump
// (one batch_begin launch per part, eager, layer-wise or inside a replayed
// graph) is counted here, and the status arrays are cleared, in stream order,
// whenever the count crosses a multiple of 2^17, so a stale status can never
// alias the current epoch.
void count_epoch_bumps(cb_plan* pl, cudaStream_t st, uint64_t bumps) {
  const uint64_t before = pl->batches;
  pl->batches += bumps;
  if ((before >> 17) == (pl->batches >> 17)) return;
  for (auto& w : pl->pe) {
    CB_CUDA(cudaMemsetAsync(w.sync.status_a, 0, w.sync.max_tiles * 8, st));
    CB_CUDA(cudaMemsetAsync(w.sync.status_b, 0, w.sync.max_tiles * 8, st));
    CB_CUDA(cudaMemsetAsync(w.sync.status_c, 0, w.sync.max_tiles * 8, st));
  }
}

// The per-batch launch sequence. d_seeds: P seed lists back to back (device).
void enqueue_batch(cb_plan* pl, int mode, const uint32_t* d_seeds, const uint64_t* off,
                   const cb_sched* sched, bool capturing = false, uint32_t n_sched = 1) {
  const uint32_t P = pl->P;
  const int L = pl->L;
  cudaStream_t st = pl->stream;
  uint64_t launches = 0;
  if (!capturing) upload_variates(pl, sched, n_sched, st);
  pl->mode = mode;
  pl->seeds_off.assign(off, off + P + 1);
  if (!capturing) count_epoch_bumps(pl, st, 1);
  const bool coop = (mode == CB_MODE_COOP) && P > 1;
  const bool smooth = smooth_of(pl, sched);
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

  // parts on their own streams (fork after the batch_begin launches, join
  // before anything that reads another part's results)
  const bool conc = pl->part_concurrent && !pl->prof && P > 1;
  auto pst = [&](uint32_t p) { return conc ? pl->part_st[p] : st; };
  auto fork = [&]() {
    if (!conc) return;
    CB_CUDA(cudaEventRecord(pl->ev_fork, st));
    for (uint32_t p = 0; p < P; ++p) CB_CUDA(cudaStreamWaitEvent(pl->part_st[p], pl->ev_fork, 0));
  };
  auto join = [&]() {
    if (!conc) return;
    for (uint32_t p = 0; p < P; ++p) {
      CB_CUDA(cudaEventRecord(pl->ev_join[p], pl->part_st[p]));
      CB_CUDA(cudaStreamWaitEvent(st, pl->ev_join[p], 0));
    }
  };
  if (!coop) {
    fork();
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
                         8 * l + 4),
            pst(p));
      }
      const uint32_t* Dl = (L == 1) ? d_seeds + off[p] : w.L[L - 2].src;
      const RelabelArgs last = relabel_args(w.bm[(L - 1) & 1], w.L[L - 1], Dl,
                                            pl->meta_at(p, L - 1));
      const uint64_t work = std::max(w.L[L - 1].cap_edges, w.L[L - 1].cap_dst);
      if (pl->defer_relabel && P == 1) {  // launched by enqueue_gather, fused
        pl->deferred = last;
        pl->deferred_work = work;
        pl->has_deferred = true;
      } else {
        launch_relabel(last, work, pst(p));
        ++launches;
        prof_mark(pl);
      }
    }
    join();
  } else {
    CB_CUDA(cudaMemsetAsync(pl->send_counts, 0, sizeof(unsigned long long) * L * P * P, st));
    for (int l = 0; l < L; ++l) {
      uint64_t max_src = 1;
      fork();
      for (uint32_t p = 0; p < P; ++p) {
        PeWork& w = pl->pe[p];
        const uint32_t* D = (l == 0) ? d_seeds + off[p] : w.L[l].dst;
        launches += enqueue_layer(
            pl, w, p, l, D, w.L[l].cap_dst, l == 0 ? off[p + 1] - off[p] : ~0ULL, w.bm[0], none,
            0, smooth,
            extract_args(w, w.bm[0], &w.bm[1], w.L[l].src, w.L[l].cap_src,
                         &pl->meta_at(p, l)->n_src, nullptr, 3 * l + 2, 8 * l + 4),
            pst(p));
        launch_relabel(relabel_args(w.bm[0], w.L[l], D, pl->meta_at(p, l)),
                       std::max(w.L[l].cap_edges, w.L[l].cap_dst), pst(p));
        launches += 1;
        max_src = std::max(max_src, w.L[l].cap_src);
      }
      join();
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

uint64_t pending_count(cb_plan* pl);

void check_overflow(cb_plan* pl, bool strict_smooth) {
  CB_CUDA(cudaStreamSynchronize(pl->stream));
  for (auto& w : pl->pe) {
    unsigned o = 0;
    CB_CUDA(cudaMemcpy(&o, w.sync.overflow, 4, cudaMemcpyDeviceToHost));
    if (o) throw Error(kOverflow, "capacity bound exceeded on device (retry with larger plan)");
  }
  // a smoothed decision inside the guard band that no host pass resolved
  // (asynchronous paths; cb_sample_sync resolves them) fails loudly
  if (strict_smooth && pl->strict && pending_count(pl) != 0)
    throw Error(kUncertified,
                "smoothed variate decisions inside the guard band are unresolved "
                "(sample with cb_sample_sync to resolve them on the host)");
}

// ---- host resolution of smoothed decisions inside the guard band ----------
// The reference's own arithmetic (rng.cpp:7-52, rng.hpp:40-58,
// samplers.hpp:96-100) on the host: glibc erfc/log/log1p/exp/sqrt, no FMA
// (-ffp-contract=off), so the value is the reference's bit for bit.
namespace hostvar {

double phi(double x) { return 0.5 * std::erfc(-x * 0.7071067811865475244); }

double inverse_phi(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - plow) {
    const double q = p - 0.5;
    const double r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = std::sqrt(-2.0 * std::log1p(-p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  const double e = phi(x) - p;
  const double u = e * std::sqrt(2.0 * 3.14159265358979323846) * std::exp(0.5 * x * x);
  return x - u / (1.0 + 0.5 * x * u);
}

double normal_from_bits(uint64_t bits) {
  return inverse_phi((static_cast<double>(bits >> 11) + 0.5) * 0x1.0p-53);
}

// VariateSource::finish (samplers.hpp:96-100), smoothed branch
double finish(const Variates& v, uint64_t b1, uint64_t b2) {
  return phi(v.cos_c * normal_from_bits(b1) + v.sin_c * normal_from_bits(b2));
}

// The exact variate of a recorded decision: LABOR r_t under prefix
// {kStreamLabor, layer} (samplers.cpp:114-129), NS u_i under
// {kStreamNs, layer, s} (samplers.cpp:75-81).
double exact(const Variates& v, uint64_t k1, uint64_t k2) {
  using cbdev::hinit;
  using cbdev::hstep;
  const uint64_t layer = (k1 >> 32) & 0xffffULL;
  const uint64_t id = k1 & 0xffffffffULL;
  if (k1 & cbdev::kResolveLabor) {
    const uint64_t h1 = hstep(hstep(hinit(v.z1), 2ULL), layer);
    const uint64_t h2 = hstep(hstep(hinit(v.z2), 2ULL), layer);
    return finish(v, hstep(h1, id), hstep(h2, id));
  }
  const uint64_t h1 = hstep(hstep(hstep(hinit(v.z1), 1ULL), layer), id);
  const uint64_t h2 = hstep(hstep(hstep(hinit(v.z2), 1ULL), layer), id);
  return finish(v, hstep(h1, k2), hstep(h2, k2));
}

}  // namespace hostvar

void resolve_upload(cb_plan* pl, const std::map<std::pair<uint64_t, uint64_t>, double>& tab,
                    cudaStream_t st) {
  const uint32_t n = static_cast<uint32_t>(tab.size());
  if (n > pl->rs_cap) {
    for (void* q : {static_cast<void*>(pl->rs_k1), static_cast<void*>(pl->rs_k2),
                    static_cast<void*>(pl->rs_val)})
      if (q) CB_CUDA(cudaFree(q));
    pl->rs_cap = std::max<uint32_t>(n, 1024);
    CB_CUDA(cudaMalloc(&pl->rs_k1, 8ULL * pl->rs_cap));
    CB_CUDA(cudaMalloc(&pl->rs_k2, 8ULL * pl->rs_cap));
    CB_CUDA(cudaMalloc(&pl->rs_val, 8ULL * pl->rs_cap));
  }
  std::vector<uint64_t> k1, k2;
  std::vector<double> val;
  for (const auto& [k, x] : tab) {
    k1.push_back(k.first);
    k2.push_back(k.second);
    val.push_back(x);
  }
  if (n) {
    CB_CUDA(cudaMemcpyAsync(pl->rs_k1, k1.data(), 8ULL * n, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaMemcpyAsync(pl->rs_k2, k2.data(), 8ULL * n, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaMemcpyAsync(pl->rs_val, val.data(), 8ULL * n, cudaMemcpyHostToDevice, st));
  }
  cbdev::Resolve r{};
  r.k1 = pl->rs_k1;
  r.k2 = pl->rs_k2;
  r.val = pl->rs_val;
  r.n = n;
  r.cap_pend = kResolvePendCap;
  r.pend = pl->rs_pend;
  r.n_pend = pl->rs_npend;
  r.perturb = pl->perturb;
  CB_CUDA(cudaMemcpyAsync(pl->d_rs, &r, sizeof(r), cudaMemcpyHostToDevice, st));
  CB_CUDA(cudaStreamSynchronize(st));  // r and the key vectors live on this frame
}

uint64_t pending_count(cb_plan* pl) {
  if (!pl->rs_npend) return 0;
  unsigned long long n = 0;
  CB_CUDA(cudaMemcpy(&n, pl->rs_npend, 8, cudaMemcpyDeviceToHost));
  return n;
}

uint64_t uncertified_total(cb_plan* pl) {
  uint64_t u = 0;
  for (uint32_t p = 0; p < pl->P; ++p)
    for (int l = 0; l < pl->L; ++l) u += host_meta(pl, p, l).uncertified;
  return u;
}

void clear_uncertified(cb_plan* pl, cudaStream_t st) {
  for (uint32_t p = 0; p < pl->P; ++p)
    for (int l = 0; l <= pl->L; ++l)
      CB_CUDA(cudaMemsetAsync(&pl->meta_at(p, l)->uncertified, 0, 8, st));
  if (pl->rs_npend) CB_CUDA(cudaMemsetAsync(pl->rs_npend, 0, 8, st));
}

void sample_host(cb_plan* pl, int mode, const uint32_t* flat, const uint64_t* off,
                 const cb_sched* sched, uint32_t n_sched = 1) {
  require(mode == CB_MODE_COOP || mode == CB_MODE_INDEP, "unknown sampling mode");
  require(sched != nullptr, "null schedule");
  for (uint32_t i = 0; i < n_sched; ++i) {
    require(sched[i].kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    const auto smoothed = [](const cb_sched& x) {
      return x.kappa != cbdev::kKappaInf && x.kappa >= 2;
    };
    require(smoothed(sched[i]) == smoothed(sched[0]),
            "per-part schedules must agree on smoothing (kappa in {1, inf} vs 2..)");
  }
  check_seeds_host(pl, flat, off);
  require_mode(pl, mode);
  if (mode == CB_MODE_COOP) check_ownership_host(pl, flat, off);
  const uint64_t total = off[pl->P];
  if (total)
    CB_CUDA(cudaMemcpyAsync(pl->seeds, flat, total * 4, cudaMemcpyHostToDevice, pl->stream));
  enqueue_batch(pl, mode, pl->seeds, off, sched, false, n_sched);
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

void prepare_rows(cb_plan* pl, const cb_features* f, bool any_row) {
  require(f->n_rows == pl->g->g.n, "feature table does not match the graph");
  if (any_row) require_full_table(f);
  for (uint32_t p = 0; p < pl->P; ++p) {
    PeWork& w = pl->pe[p];
    const LayerBufs& b = w.L[pl->L - 1];
    // peer-exchange plans cap their row buffers (their src capacity is the
    // world-times worst case); exceeding the cap flags an overflow
    const uint64_t want = pl->rows_limit ? std::min(b.cap_src, pl->rows_limit) : b.cap_src;
    if (!w.rows || w.rows_row_bytes != f->row_bytes || w.cap_rows < want) {
      w.rows = pl->rows_mem.alloc<unsigned char>(want * f->row_bytes);
      w.cap_rows = want;
      w.rows_row_bytes = f->row_bytes;
    }
  }
}

void enqueue_gather(cb_plan* pl, const cb_features* f) {
  NvtxRange nvtx_("cb.gather");
  const int vb = vec_bytes_for(f->row_bytes);
  const bool conc = pl->part_concurrent && !pl->prof && pl->P > 1;
  if (conc) {  // the parts' gathers are independent: one stream each
    CB_CUDA(cudaEventRecord(pl->ev_fork, pl->stream));
    for (uint32_t p = 0; p < pl->P; ++p)
      CB_CUDA(cudaStreamWaitEvent(pl->part_st[p], pl->ev_fork, 0));
  }
  for (uint32_t p = 0; p < pl->P; ++p) {
    PeWork& w = pl->pe[p];
    const LayerBufs& b = w.L[pl->L - 1];
    if (p == 0 && pl->has_deferred) {
      launch_relabel_gather(pl->deferred, pl->deferred_work, f->table, vb, f->row_bytes, b.src,
                            &pl->meta_at(p, pl->L - 1)->n_src, w.cap_rows, f->row_map, w.rows,
                            conc ? pl->part_st[p] : pl->stream);
      pl->has_deferred = false;
    } else {
      launch_gather(f->table, vb, f->row_bytes, b.src, &pl->meta_at(p, pl->L - 1)->n_src,
                    w.cap_rows, f->row_map, w.rows, conc ? pl->part_st[p] : pl->stream);
    }
    pl->launches += 1;
    prof_mark(pl);
  }
  if (conc)
    for (uint32_t p = 0; p < pl->P; ++p) {
      CB_CUDA(cudaEventRecord(pl->ev_join[p], pl->part_st[p]));
      CB_CUDA(cudaStreamWaitEvent(pl->stream, pl->ev_join[p], 0));
    }
  pl->have_rows = true;
}

}  // namespace capi
}  // namespace cb

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
      if (indptr[v] > indptr[v + 1])
        throw Error(kInput, "csr: indptr not nondecreasing at " + std::to_string(v));
    for (uint64_t e = 0; e < m; ++e) require(indices[e] < n, "csr: index out of range");
    DeviceGuard dg(device);
    auto h = std::make_unique<cb_graph>();
    h->g.device = device;
    h->g.n = n;
    h->g.m = m;
    CB_CUDA(cudaMalloc(&h->g.indptr, (n + 1) * 8));
    // +16 B: labor_mark bulk-copies 16-byte-aligned supersets of id ranges
    CB_CUDA(cudaMalloc(&h->g.indices, std::max<uint64_t>(m, 1) * 4 + 16));
    h2d_sync(h->g.indptr, indptr, (n + 1) * 8);
    if (m) h2d_sync(h->g.indices, indices, m * 4);
    uint64_t md = 0;
    for (uint64_t v = 0; v < n; ++v) md = std::max(md, indptr[v + 1] - indptr[v]);
    h->g.max_degree = md;
    *out = h.release();
  });
}

// Edge weights (graph.hpp:25, one per edge, > 0): kept in HBM next to the
// indices; only the RW sampler reads them (samplers.cpp:139-165).
int cb_graph_set_weights(cb_graph* g, const float* weights) {
  return guard([&] {
    require(g != nullptr, "null graph");
    DeviceGuard dg(g->g.device);
    if (!weights) {
      if (g->weights_mem) g->weights_mem.reset();
      g->g.weights = nullptr;
      return;
    }
    for (uint64_t e = 0; e < g->g.m; ++e)
      require(weights[e] > 0.0f, "csr: weights must be > 0");
    g->weights_mem = std::make_unique<Arena>();
    g->g.weights = g->weights_mem->alloc<float>(std::max<uint64_t>(g->g.m, 1));
    if (g->g.m)
      h2d_sync(g->g.weights, weights, g->g.m * 4);
  });
}

// CBCS binary CSR (graph.hpp:78-80, graph.cpp:196-265): "CBCS", u32 version 1,
// u64 n, u64 m, u64 indptr[n+1], u32 indices[m], u8 flags, f32 weights[m] if
// flags & 1. Little-endian. Weights (validated > 0) go to HBM with the CSR.
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
    std::vector<float> w;
    if (flags & 1) {
      w.resize(m);
      rd(w.data(), m * 4, "weights");
      for (float x : w) require(x > 0.0f, "csr: weights must be > 0");
    }
    const int rc = cb_graph_create_from_csr(indptr.data(), indices.data(), n, m, device, out);
    if (rc != CB_OK) throw Error(static_cast<Status>(rc), g_err);
    if (flags & 1) {
      const int rw = cb_graph_set_weights(*out, w.data());
      if (rw != CB_OK) {
        cb_graph_destroy(*out);
        *out = nullptr;
        throw Error(static_cast<Status>(rw), g_err);
      }
    }
  });
}

int cb_graph_save_cbcs(const cb_graph* g, const char* path) {
  return guard([&] {
    require(g != nullptr && path != nullptr, "null argument");
    std::vector<uint64_t> indptr(g->g.n + 1);
    std::vector<uint32_t> indices(g->g.m);
    std::vector<float> w(g->g.weights ? g->g.m : 0);
    {
      DeviceGuard dg(g->g.device);
      CB_CUDA(cudaMemcpy(indptr.data(), g->g.indptr, (g->g.n + 1) * 8, cudaMemcpyDeviceToHost));
      if (g->g.m)
        CB_CUDA(cudaMemcpy(indices.data(), g->g.indices, g->g.m * 4, cudaMemcpyDeviceToHost));
      if (!w.empty())
        CB_CUDA(cudaMemcpy(w.data(), g->g.weights, g->g.m * 4, cudaMemcpyDeviceToHost));
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(kIo, std::string("cannot open for write: ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, &std::fclose);
    const uint32_t version = 1;
    const uint64_t n = g->g.n, m = g->g.m;
    const uint8_t flags = w.empty() ? 0 : 1;
    bool ok = std::fwrite("CBCS", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&m, 8, 1, f) == 1 &&
              std::fwrite(indptr.data(), 8, n + 1, f) == n + 1 &&
              (m == 0 || std::fwrite(indices.data(), 4, m, f) == m) &&
              std::fwrite(&flags, 1, 1, f) == 1 &&
              (w.empty() || std::fwrite(w.data(), 4, m, f) == m);
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
  h2d_sync(ids, iota.data(), n * 4);
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
  {
    DevBuf tmp(tmp_bytes + 16);
    CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.as<void>(), tmp_bytes, kb, vb, (int64_t)n, 0,
                                            bits, st));
    CB_CUDA(cudaStreamSynchronize(st));
  }
  std::vector<uint32_t> members(n), sorted_keys(n);
  CB_CUDA(cudaMemcpy(members.data(), vb.Current(), n * 4, cudaMemcpyDeviceToHost));
  CB_CUDA(cudaMemcpy(sorted_keys.data(), kb.Current(), n * 4, cudaMemcpyDeviceToHost));
  pm->shard_off.assign(pm->parts + 1, 0);
  for (uint64_t i = 0; i < n; ++i) pm->shard_off[sorted_keys[i] + 1]++;
  for (uint32_t q = 0; q < pm->parts; ++q) pm->shard_off[q + 1] += pm->shard_off[q];
  std::vector<uint32_t> row_map(n);
  for (uint64_t i = 0; i < n; ++i) row_map[members[i]] = static_cast<uint32_t>(i);
  h2d_sync(pm->members, members.data(), n * 4);
  h2d_sync(pm->row_map, row_map.data(), n * 4);
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
    h2d_sync(pm->owner, owner, pm->n * 4);
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

namespace {
int plan_create(const cb_graph* g, const cb_partition* pm, uint32_t parts, int num_layers,
                int kind, const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out) {
  return guard([&] {
    require(g != nullptr && out != nullptr, "null argument");
    require(parts >= 1 && parts <= 64, "part count must be in [1, 64]");
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
    pl->P = pm ? pm->parts : parts;
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
}  // namespace

int cb_plan_create(const cb_graph* g, const cb_partition* pm, int num_layers, int kind,
                   const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out) {
  return plan_create(g, pm, 1, num_layers, kind, fanouts, max_seeds_per_part, out);
}

int cb_plan_create_parts(const cb_graph* g, uint32_t parts, int num_layers, int kind,
                         const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out) {
  return plan_create(g, nullptr, parts, num_layers, kind, fanouts, max_seeds_per_part, out);
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
    const bool smooth = smooth_of(plan, sched) && !plan->ext_vtab &&
                        !(plan->var_source && plan->var_source->smoothed != 1);
    std::map<std::pair<uint64_t, uint64_t>, double> tab;
    plan->rs_resolved = plan->rs_reruns = 0;
    if (smooth) {
      resolve_alloc(plan);
      resolve_upload(plan, tab, plan->stream);
    }
    const Variates var = plan->var_source ? *plan->var_source : make_variates(sched);
    for (int pass = 0;; ++pass) {
      for (int attempt = 0;; ++attempt) {
        sample_host(plan, mode, seeds_flat, seeds_off, sched);
        try {
          check_overflow(plan, false);
          break;
        } catch (const Error& e) {
          if (e.code != kOverflow || attempt >= 12) throw;
          plan->grow *= 2.0;
          plan_alloc(plan);
        }
      }
      if (!smooth) return;
      const uint64_t np = pending_count(plan);
      if (np == 0) return;
      // decisions the device made inside the guard band: evaluate each with
      // the reference's arithmetic; if every one agrees, the batch stands
      std::vector<cbdev::ResolvePend> pend(std::min<uint64_t>(np, kResolvePendCap));
      CB_CUDA(cudaMemcpy(pend.data(), plan->rs_pend, sizeof(cbdev::ResolvePend) * pend.size(),
                         cudaMemcpyDeviceToHost));
      bool differ = np > pend.size();
      for (const auto& e : pend) {
        const double ex = hostvar::exact(var, e.k1, e.k2);
        tab[{e.k1, e.k2}] = ex;
        ++plan->rs_resolved;
        if (e.k1 & cbdev::kResolveLabor) {
          differ |= (ex <= e.aux) != (e.dev <= e.aux);
        } else {
          const double y = ex * static_cast<double>(e.k2 + 1);
          differ |= static_cast<uint64_t>(y) != static_cast<uint64_t>(e.aux);
        }
      }
      if (!differ) {
        clear_uncertified(plan, plan->stream);
        CB_CUDA(cudaStreamSynchronize(plan->stream));
        return;
      }
      // some device decision was wrong: sample again with the exact values
      // (a corrected layer may bring new in-band decisions: repeat)
      if (pass >= 8) throw Error(kInternal, "smoothed decisions did not converge");
      ++plan->rs_reruns;
      resolve_upload(plan, tab, plan->stream);
    }
  });
}

int cb_plan_set_guard(cb_plan* plan, double band, int perturb, int strict) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(band >= 0.0 && band < 1.0, "guard band must be in [0, 1)");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    plan->guard = band;
    plan->perturb = perturb;
    plan->strict = strict != 0;
    if (plan->d_rs) {
      std::map<std::pair<uint64_t, uint64_t>, double> none;
      resolve_upload(plan, none, plan->stream);
    }
  });
}

int cb_plan_resolve_stats(const cb_plan* plan, uint64_t* resolved, uint64_t* reruns) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    if (resolved) *resolved = plan->rs_resolved;
    if (reruns) *reruns = plan->rs_reruns;
  });
}

int cb_plan_set_layer_base(cb_plan* plan, int base) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(base >= 0, "layer index must be >= 0");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    plan->drop_graphs();
    plan->layer_base = base;
  });
}

int cb_plan_set_variate_table(cb_plan* plan, const double* table, int on_device) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(plan->kind == CB_LABOR0 || table == nullptr,
            "a variate table applies to LABOR-0 plans only");
    require(plan->dist_world == 0, "variate tables are not supported on distributed plans");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    plan->drop_graphs();  // captured batches baked the previous variate mode in
    if (!table) {
      if (plan->ext_vtab) cudaFree(plan->ext_vtab);
      plan->ext_vtab = nullptr;
      return;
    }
    const uint64_t n = plan->g->g.n;
    if (!plan->ext_vtab) CB_CUDA(cudaMalloc(&plan->ext_vtab, std::max<uint64_t>(n, 1) * 8));
    CB_CUDA(cudaMemcpyAsync(plan->ext_vtab, table, n * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            plan->stream));
    CB_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

// An explicit VariateSource (samplers.hpp:61-126: z1, z2, cos/sin of the
// contribution, smoothed) for the plan's next batches instead of the one
// SeedSchedule derives; nullptr goes back to the schedule.
int cb_plan_set_variate_source(cb_plan* plan, const cb_variates* v) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    plan->drop_graphs();  // captured batches baked the previous smoothing mode in
    if (!v) {
      plan->var_source.reset();
      return;
    }
    Variates x{};
    x.z1 = v->z1;
    x.z2 = v->z2;
    x.cos_c = v->cos_c;
    x.sin_c = v->sin_c;
    x.smoothed = v->smoothed ? 1 : 0;
    plan->var_source = x;
  });
}

int cb_sample_multi(cb_plan* plan, const uint32_t* seeds_flat, const uint64_t* seeds_off,
                    const cb_sched* scheds) {
  NvtxRange nvtx_("cb.sample_multi");
  return guard([&] {
    require(plan != nullptr && seeds_off != nullptr && scheds != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    for (int attempt = 0;; ++attempt) {
      sample_host(plan, CB_MODE_INDEP, seeds_flat, seeds_off, scheds, plan->P);
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
    require_mode(plan, mode);
    check_offsets(plan, seeds_off);
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
    require_mode(plan, mode);
    check_offsets(plan, seeds_off);
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
      plan->defer_relabel = true;
      try {
        enqueue_batch(plan, mode, plan->seeds, seeds_off, &dummy, true);
      } catch (...) {
        plan->defer_relabel = false;
        throw;
      }
      plan->defer_relabel = false;
      enqueue_gather(plan, f);
      plan->cap_launches_all = plan->launches;
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
      const bool sm = smooth_of(plan, sched);
      require(sm == plan->cap_smooth,
              "schedule smoothing differs from the captured batch (re-capture)");
      const uint64_t total = plan->cap_off[plan->P];
      if (seeds_flat && total)
        CB_CUDA(cudaMemcpyAsync(plan->seeds, seeds_flat, total * 4,
                                seeds_on_device ? cudaMemcpyDeviceToDevice
                                                : cudaMemcpyHostToDevice,
                                st));
      upload_variates(plan, sched, 1, st);
      // the graph bumps the epoch once; a re-clear of another mode's
      // leftovers below bumps it once more
      count_epoch_bumps(plan, st, 1);
      if (plan->dirty_mode >= 0 && plan->dirty_mode != plan->cap_mode) {
        count_epoch_bumps(plan, st, 1);
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
      plan->launches = all ? plan->cap_launches_all : plan->cap_launches_sample;
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

// Result bytes a batch of this plan can need at most (capacities), for
// sizing the pinned buffer of cb_plan_result_async.
int cb_plan_result_bytes(const cb_plan* plan, uint32_t part, uint64_t row_bytes,
                         uint64_t* max_bytes) {
  return guard([&] {
    require(plan != nullptr && max_bytes != nullptr, "null argument");
    require(part < plan->P, "part index out of range");
    require(plan->L <= kResultMaxLayers, "result: too many layers");
    auto pad = [](uint64_t b) { return (b + 15) & ~15ULL; };
    uint64_t t = pad(8ULL * (5 + 3 * plan->L));
    const PeWork& w = plan->pe[part];
    for (int l = 0; l < plan->L; ++l) {
      const LayerBufs& b = w.L[l];
      const uint64_t cd = l == 0 ? plan->max_seeds : b.cap_dst;
      t += 2 * pad(cd * 4) + pad(b.cap_src * 4) + pad(b.cap_edges * 8);
    }
    t += pad(w.L[plan->L - 1].cap_src * row_bytes);
    *max_bytes = t;
  });
}

// The batch's blocks (and gathered rows, when the batch has them) written
// into pinned host memory by one kernel on the plan stream; nothing waits.
// Layout: result.cu. Ordered after the batch; the caller synchronises
// (cb_synchronize / an event) before reading.
int cb_plan_result_async(cb_plan* plan, uint32_t part, void* host_pinned, uint64_t cap_bytes) {
  return guard([&] {
    require(plan != nullptr && host_pinned != nullptr, "null argument");
    require_batch(plan, part, 0);
    require(plan->L <= kResultMaxLayers, "result: too many layers");
    require(cap_bytes >= 8ULL * (5 + 3 * plan->L), "result buffer smaller than its header");
    DeviceGuard dg(plan->device);
    void* dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, host_pinned, 0) != cudaSuccess) {
      cudaGetLastError();  // not sticky: clear it so later launch checks stay clean
      throw Error(kInput, "result buffer is not pinned, device-mapped host memory");
    }
    PeWork& w = plan->pe[part];
    ResultArgs a{};
    a.meta = plan->meta_at(part, 0);
    a.L = plan->L;
    for (int l = 0; l < plan->L; ++l) {
      const LayerBufs& b = w.L[l];
      const uint32_t* d_dst;
      if (l == 0) d_dst = plan->seeds + plan->seeds_off[part];
      else if (!plan->own_dst()) d_dst = w.L[l - 1].src;
      else d_dst = b.dst;
      a.ptr[l][0] = d_dst;
      a.ptr[l][1] = b.src;
      a.ptr[l][2] = b.edges;
      a.ptr[l][3] = b.dst_pos;
    }
    a.rows = plan->have_rows ? w.rows : nullptr;
    a.row_bytes = plan->have_rows ? w.rows_row_bytes : 0;
    a.out = static_cast<unsigned char*>(dptr);
    a.cap = cap_bytes;
    launch_result(a, plan->stream);
  });
}

// Pack part `part`'s batch result (result.cu layout) into the plan's device
// staging buffer, sized from the capacities (cb_plan_result_bytes).
void enqueue_result_pack(cb_plan* plan, uint32_t part) {
  const int L = plan->L;
  PeWork& w = plan->pe[part];
  uint64_t need = 0;
  cb_plan_result_bytes(plan, part, plan->have_rows ? w.rows_row_bytes : 0, &need);
  if (plan->pack_bytes < need) {
    if (plan->pack) CB_CUDA(cudaFree(plan->pack));
    plan->pack_bytes = need;
    CB_CUDA(cudaMalloc(&plan->pack, plan->pack_bytes));
  }
  ResultArgs a{};
  a.meta = plan->meta_at(part, 0);
  a.L = L;
  for (int l = 0; l < L; ++l) {
    const LayerBufs& b = w.L[l];
    const uint32_t* d_dst;
    if (l == 0) d_dst = plan->seeds + plan->seeds_off[part];
    else if (!plan->own_dst()) d_dst = w.L[l - 1].src;
    else d_dst = b.dst;
    a.ptr[l][0] = d_dst;
    a.ptr[l][1] = b.src;
    a.ptr[l][2] = b.edges;
    a.ptr[l][3] = b.dst_pos;
  }
  a.rows = plan->have_rows ? w.rows : nullptr;
  a.row_bytes = plan->have_rows ? w.rows_row_bytes : 0;
  a.out = static_cast<unsigned char*>(plan->pack);
  a.cap = plan->pack_bytes;
  launch_result(a, plan->stream);
  plan->pack_part = part;
  plan->pack_version = plan->batches;
}

int cb_plan_result_pack(cb_plan* plan, uint32_t part) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    require_batch(plan, part, 0);
    require(plan->L <= kResultMaxLayers, "result: too many layers");
    DeviceGuard dg(plan->device);
    enqueue_result_pack(plan, part);
  });
}

// The result moved by a copy engine: the batch packed on the device (by
// cb_plan_result_pack right after the batch, else here), the host waits for
// it, and ONE D2H copy of the packed bytes follows on the plan stream. A copy
// engine sustains ~56 GB/s over the host link where SM stores into mapped
// memory reach ~34 GB/s; the host wait is hidden by a caller that keeps
// several batches in flight.
int cb_plan_result_copy(cb_plan* plan, uint32_t part, void* host_pinned, uint64_t cap_bytes,
                        uint64_t* total_bytes) {
  NvtxRange nvtx_("cb.result_copy");
  return guard([&] {
    require(plan != nullptr && host_pinned != nullptr, "null argument");
    require_batch(plan, part, 0);
    require(plan->L <= kResultMaxLayers, "result: too many layers");
    const int L = plan->L;
    require(cap_bytes >= 8ULL * (5 + 3 * L), "result buffer smaller than its header");
    DeviceGuard dg(plan->device);
    if (plan->pack_version != plan->batches || plan->pack_part != part)
      enqueue_result_pack(plan, part);
    if (!plan->meta_host)
      CB_CUDA(cudaHostAlloc(&plan->meta_host, 64, cudaHostAllocDefault));
    // the packed header (its total size) once the batch and the pack are done
    CB_CUDA(cudaMemcpyAsync(plan->meta_host, plan->pack, 40, cudaMemcpyDeviceToHost,
                            plan->stream));
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    const uint64_t* hd = static_cast<const uint64_t*>(plan->meta_host);
    const uint64_t total = hd[3];
    if (total_bytes) *total_bytes = total;
    const uint64_t n = total <= cap_bytes ? total : 8ULL * (5 + 3 * L);
    CB_CUDA(cudaMemcpyAsync(host_pinned, plan->pack, n, cudaMemcpyDeviceToHost, plan->stream));
    if (total > cap_bytes) {  // header only, flagged truncated, as the kernel form
      CB_CUDA(cudaStreamSynchronize(plan->stream));
      static_cast<uint64_t*>(host_pinned)[4] = 1;
    }
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
      upload_variates(plan, sched, 1, st);
      plan->seeds_off.assign({0, n_dst});
      plan->mode = CB_MODE_COOP;
    }
    const bool smooth = smooth_of(plan, sched);
    count_epoch_bumps(plan, st, 1);
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
    count_epoch_bumps(plan, st, 1);
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
    if (f->shard_rows) {  // a single-part shard serves only its own rows
      DevBuf flag(8);
      require(shard_holds(d_ids, n, f->row_map, f->shard_r0, f->shard_rows,
                          flag.as<unsigned>(), st),
              "gather from a shard table: an id is not owned by the shard");
    }
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
    upload_variates(plan, sched, 1, st);
    count_epoch_bumps(plan, st, 1);
    if (plan->dirty_mode >= 0 && plan->dirty_mode != plan->cap_mode) {
      count_epoch_bumps(plan, st, 1);
      for (uint32_t p = 0; p < plan->P; ++p) {
        const Dirty d = dirty_of(plan, p, plan->dirty_mode);
        launch_batch_begin(plan->pe[p].sync, d.bits, d.summ, d.list, d.count, d.cap,
                           plan->pe[p].bm[0].words_padded, st);
      }
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

int cb_plan_captured_launches(const cb_plan* plan, int what, uint64_t* n) {
  return guard([&] {
    require(plan != nullptr && n != nullptr, "null argument");
    if (what == 4) {  // the captured peer-exchange step (cb_px_capture)
      require(plan->px != nullptr && plan->px->exec[0] != nullptr,
              "no captured step (call cb_px_capture)");
      *n = plan->px->cap_launches;
      return;
    }
    require(plan->exec_sample != nullptr, "no captured batch (call cb_plan_capture)");
    if (what == 1) *n = plan->cap_launches_sample;
    else if (what == 2) *n = plan->cap_launches_gather;
    else {
      require(what == 3 && plan->exec_all != nullptr, "no captured sample + gather graph");
      *n = plan->cap_launches_all;
    }
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

}  // extern "C"
