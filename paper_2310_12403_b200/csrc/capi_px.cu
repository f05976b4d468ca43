// C-ABI: multi-process peer exchange (cb_px_*), one part per rank over CUDA IPC.
#include "capi_internal.h"

#include <cuda.h>

#include <numeric>

extern "C" {

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

// CB_PX_BARRIER_TIMEOUT_MS (default 20000): a barrier wait that long gives up
// and flags the step as failed instead of hanging the device.
constexpr uint64_t kPxRowsLimit = 1ULL << 22;

unsigned long long barrier_timeout_ns() {
  const char* e = std::getenv("CB_PX_BARRIER_TIMEOUT_MS");
  const unsigned long long ms = e ? std::strtoull(e, nullptr, 10) : 20000ULL;
  return (ms ? ms : 20000ULL) * 1000000ULL;
}

void check_barrier(PxState& px) {
  uint32_t err = 0;
  CB_CUDA(cudaMemcpy(&err, px.bar.err, 4, cudaMemcpyDeviceToHost));
  if (err) throw Error(kCuda, "peer barrier timed out (a rank stopped or ran a different step)");
}

// Layer l of the cooperative step on the plan stream: sample, then OR every
// src id into its owner's exchange bitmap (build_exchange, coop.cpp:35-51).
// Layer 0's seeds are already in plan->seeds.
void px_enqueue_layer(cb_plan* plan, int layer, uint64_t n_seeds, bool smooth, int s) {
  PxState& px = *plan->px;
  PeWork& w = plan->pe[0];
  LayerBufs& b = w.L[layer];
  cudaStream_t st = plan->stream;
  uint32_t* D = (layer == 0) ? plan->seeds : b.dst;
  const uint64_t cap = (layer == 0) ? plan->max_seeds : b.cap_dst;
  if (layer == 0) CB_CUDA(cudaMemsetAsync(px.send, 0, plan->L * px.world * 8, st));
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
}

// The owner's sorted unique set S^{l+1}_q + word ranks (coop.cpp:44-51) from
// slot s, clearing slot `clr` (a slot every rank has finished reading).
void px_enqueue_owner(cb_plan* plan, int layer, int s, int clr) {
  PxState& px = *plan->px;
  PeWork& w = plan->pe[0];
  uint32_t* next = (layer + 1 < plan->L) ? w.L[layer + 1].dst : w.owner_final;
  const uint64_t cap = (layer + 1 < plan->L) ? w.L[layer + 1].cap_dst : w.cap_final;
  launch_extract(extract_args(w, px.slot[s], &px.slot[clr], next, cap,
                              &plan->meta_at(0, layer + 1)->n_dst, nullptr,
                              3 * plan->L + layer, 8 * layer + 5),
                 plan->stream);
}

// src_location from the owners' bitmaps (coop.cpp:53-62).
void px_enqueue_locate(cb_plan* plan, int layer) {
  PxState& px = *plan->px;
  PeWork& w = plan->pe[0];
  LayerBufs& b = w.L[layer];
  launch_px_locate(b.src, &plan->meta_at(0, layer)->n_src, b.cap_src, px.owner,
                   px.peers[px.slot_of[layer]], w.loc_part[layer], w.loc_row[layer],
                   plan->stream);
}

// cuStreamWaitValue32 through the runtime's driver entry point (no -lcuda).
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    const char* e = std::getenv("CB_PX_BARRIER");
    if (e && std::string(e) == "spin") return static_cast<WaitValueFn>(nullptr);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WaitValueFn>(nullptr);
    return reinterpret_cast<WaitValueFn>(p);
  }();
  return fn;
}

// Barrier j of a captured step in graph g: this rank's arrival is stored as
// g + 1 into row 1 + j of every peer's flag block, and the stream waits (a
// front-end semaphore wait, no SM spinning) until every peer's entry in the
// local row equals g + 1. Consecutive replays alternate g, and a rank can be
// at most one barrier ahead of any peer, so a row is never overwritten while
// a peer still waits on it.
void px_enqueue_barrier(cb_plan* plan, int j, int g) {
  PxState& px = *plan->px;
  if (!px.memop) {
    launch_px_barrier(px.bar, plan->stream);
    return;
  }
  const uint32_t row = 1 + j, val = 1 + g;
  launch_px_signal(px.bar, row, val, plan->stream);
  for (uint32_t q = 0; q < px.world; ++q) {
    if (q == px.rank) continue;
    const CUdeviceptr a =
        reinterpret_cast<CUdeviceptr>(px.bar.flags[px.rank] + row * kMaxParts + q);
    if (wait_value_fn()(reinterpret_cast<CUstream>(plan->stream), a, val,
                        CU_STREAM_WAIT_VALUE_EQ) != CUDA_SUCCESS)
      throw Error(kCuda, "cuStreamWaitValue32 failed");
  }
}

void px_enqueue_staged_gather(cb_plan* plan, int g);

// The whole cooperative step as captured (coop.cpp:92-102 per layer, then
// all_to_all_forward when f is given), with ONE barrier per layer plus one at
// the end. Layer c of the run (c0 + l) routes into slot c % 4; after barrier
// l the owner extracts slot c % 4 and clears slot (c + 2) % 4, and the
// requester locates layer l - 1 in slot (c - 1) % 4:
//  * slot c % 4 is complete at barrier l (every rank's route l precedes it);
//  * slot (c - 1) % 4 was extracted by every owner before barrier l, and is
//    cleared only by owner c + 1, after barrier l + 1;
//  * slot (c + 2) % 4 = (c - 2) % 4 was last read by locate l - 2, before
//    barrier l, and is next written by route c + 2, after barrier l + 1.
// Graph g signals barrier value g % 2 + 1 (px_enqueue_barrier).
void px_enqueue_step(cb_plan* plan, uint64_t n_seeds, bool smooth, uint64_t c0,
                     const cb_features* f, int g) {
  PxState& px = *plan->px;
  const int L = plan->L;
  for (int l = 0; l < L; ++l) {
    const uint64_t c = c0 + l;
    px_enqueue_layer(plan, l, n_seeds, smooth, static_cast<int>(c % 4));
    px_enqueue_barrier(plan, l, g & 1);
    px_enqueue_owner(plan, l, static_cast<int>(c % 4), static_cast<int>((c + 2) % 4));
    if (l > 0) px_enqueue_locate(plan, l - 1);
  }
  px_enqueue_barrier(plan, L, g & 1);
  px_enqueue_locate(plan, L - 1);
  if (f && px.rstage) {
    px_enqueue_staged_gather(plan, g);
  } else if (f) {
    PeWork& w = plan->pe[0];
    launch_px_gather(px.d_fbase, px.owner, f->row_map, f->row_bytes, w.L[L - 1].src,
                     &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, plan->stream);
  }
}

// access order key of the requester cache (a different stream than the
// owner's, so the two caches see independent orders)
uint64_t requester_key(uint64_t order_key) { return cbdev::hstep(order_key, 0x5245515545ULL); }

void require_staging(const PxState& px) {
  require(px.rstage != nullptr, "no staging buffer (cb_px_setup_staging)");
  for (uint32_t q = 0; q < px.world; ++q)
    require(px.rstage_of[q] != nullptr, "staging buffer of a rank not connected");
}

// Owner q gathers the rows of S^L_q from its shard into its staging buffer
// (device count), barrier, requesters pull from the owners' staging.
void px_enqueue_staged_gather(cb_plan* plan, int g) {
  PxState& px = *plan->px;
  PeWork& w = plan->pe[0];
  const int L = plan->L;
  const cb_features* f = px.stage_store;
  if (px.ccache) {  // owner-side CLOCK cache: hits from HBM, misses from the shard
    px.ccache->cc->gather(f->table, f->row_map, w.owner_final, &plan->meta_at(0, L)->n_dst,
                          px.rstage_rows, px.rstage, plan->stream);
  } else {
    launch_gather(f->table, vec_bytes_for(f->row_bytes), f->row_bytes, w.owner_final,
                  &plan->meta_at(0, L)->n_dst, px.rstage_rows, f->row_map, px.rstage,
                  plan->stream);
  }
  if (g < 0) launch_px_barrier(px.bar, plan->stream);
  else px_enqueue_barrier(plan, L + 1, g & 1);
  PxCaps caps;
  caps.count2 = &plan->meta_at(0, L)->n_dst;
  caps.cap2 = px.rstage_rows;
  caps.overflow = w.sync.overflow;
  launch_px_gather_staged(px.d_rstage, w.loc_part[L - 1], w.loc_row[L - 1], f->row_bytes,
                          &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, caps,
                          plan->stream);
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
    px->flag_off = PxState::kSlots * per;
    px->region_bytes = px->flag_off + kBarRows * kMaxParts * 4;
    CB_CUDA(cudaMalloc(&px->region, px->region_bytes));
    CB_CUDA(cudaMemset(px->region, 0, px->region_bytes));
    for (int s = 0; s < PxState::kSlots; ++s) {
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
    CB_CUDA(cudaMalloc(&px->bar_ctr, 8));
    CB_CUDA(cudaMemset(px->bar_ctr, 0, 8));
    px->bar.ctr = px->bar_ctr;
    px->bar.err = px->bar_ctr + 1;
    px->bar.rank = rank;
    px->bar.world = px->world;
    px->bar.timeout_ns = barrier_timeout_ns();
    px->bar.flags[rank] =
        reinterpret_cast<uint32_t*>(static_cast<char*>(px->region) + px->flag_off);
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
    const uint64_t per = px.flag_off / PxState::kSlots;
    px.bar.flags[q] = reinterpret_cast<uint32_t*>(static_cast<char*>(p) + px.flag_off);
    for (int s = 0; s < PxState::kSlots; ++s) {
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
    cudaStream_t st = plan->stream;
    if (layer == 0) {
      require(seeds != nullptr || n_seeds == 0, "null seeds");
      require(n_seeds <= plan->max_seeds, "more seeds than the plan's max_seeds_per_part");
      if (n_seeds)
        CB_CUDA(cudaMemcpyAsync(plan->seeds, seeds, n_seeds * 4, cudaMemcpyDefault, st));
      upload_variates(plan, sched, 1, st);
      plan->seeds_off.assign({0, n_seeds});
      plan->mode = CB_MODE_COOP;
    }
    require(px.replays == 0,
            "captured peer-exchange steps ran on this plan (eager steps need a new plan)");
    const bool smooth = smooth_of(plan, sched);
    const int s = static_cast<int>(px.layer_ctr++ & 1);
    px.eager_since_capture = true;
    count_epoch_bumps(plan, st, 1);
    px_enqueue_layer(plan, layer, layer == 0 ? n_seeds : 0, smooth, s);
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
    // eager steps alternate slots 0/1: the other one was last read by the
    // previous layer's locates, finished before the caller's barrier
    const int s = px.slot_of[layer];
    px_enqueue_owner(plan, layer, s, s ^ 1);
  });
}

int cb_px_locate(cb_plan* plan, int layer) {
  NvtxRange nvtx_("cb.px_locate");
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(layer >= 0 && layer < plan->L, "layer index out of range");
    px_of(plan);
    DeviceGuard dg(plan->device);
    px_enqueue_locate(plan, layer);
  });
}

int cb_px_finish(cb_plan* plan) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    if (plan->px) check_barrier(*plan->px);
  });
}

int cb_px_barrier(cb_plan* plan) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    launch_px_barrier(px.bar, plan->stream);
  });
}

int cb_px_capture(cb_plan* plan, uint64_t n_seeds, const cb_sched* sched,
                  const cb_features* local) {
  return guard([&] {
    require(plan != nullptr && sched != nullptr, "null argument");
    require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    require(n_seeds <= plan->max_seeds, "more seeds than the plan's max_seeds_per_part");
    PxState& px = px_of(plan);
    if (local && !px.rstage) {  // direct pull from the peers' shards
      for (uint32_t q = 0; q < px.world; ++q)
        require(px.fbase[q] != nullptr, "feature shard of a rank not connected");
    }
    DeviceGuard dg(plan->device);
    px.drop_graphs();
    if (local) prepare_rows(plan, local, false);
    const bool smooth = smooth_of(plan, sched);
    // kernel attributes are set by the eager layer calls every rank has made
    // before capturing (the caller's warm-up step); capture is local only
    require(plan->L + 3 <= kBarRows, "peer exchange capture: too many layers");
    if (local && px.rstage) require_staging(px);
    px.memop = wait_value_fn() != nullptr;
    px_preload();
    // captured steps rotate all four slots: start from clean ones (the caller
    // keeps every rank quiet around the capture, dist.PeerCoop.capture)
    CB_CUDA(cudaStreamSynchronize(plan->stream));
    CB_CUDA(cudaMemset(px.region, 0, px.flag_off));
    CB_CUDA(cudaDeviceSynchronize());
    const int period = 4 / std::gcd(plan->L, 4);  // steps until the slots realign
    px.n_exec = std::max(period, 2);               // and the barrier value alternates
    const unsigned long long k0 = g_kernel_launches.load();
    for (int g = 0; g < px.n_exec; ++g) {
      cudaGraph_t graph;
      CB_CUDA(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
      try {
        px_enqueue_step(plan, n_seeds, smooth, static_cast<uint64_t>(g) * plan->L, local, g);
      } catch (...) {
        cudaStreamEndCapture(plan->stream, &graph);
        throw;
      }
      CB_CUDA(cudaStreamEndCapture(plan->stream, &graph));
      CB_CUDA(cudaGraphInstantiate(&px.exec[g], graph, 0));
      CB_CUDA(cudaGraphDestroy(graph));
    }
    px.cap_launches = (g_kernel_launches.load() - k0) / px.n_exec;
    px.replays = 0;
    px.eager_since_capture = false;
    px.cap_seeds = n_seeds;
    px.cap_rows = local != nullptr;
    px.cap_smooth = smooth;
  });
}

int cb_px_replay(cb_plan* plan, const uint32_t* seeds, int seeds_on_device,
                 const cb_sched* sched) {
  NvtxRange nvtx_("cb.px_replay");
  return guard([&] {
    require(plan != nullptr && sched != nullptr, "null argument");
    require(sched->kappa != 0, "SeedSchedule: kappa must be >= 1 (or infinity)");
    PxState& px = px_of(plan);
    require(px.exec[0] != nullptr, "no captured step (call cb_px_capture)");
    require(smooth_of(plan, sched) == px.cap_smooth,
            "schedule smoothing differs from the captured step (re-capture)");
    require(seeds != nullptr || px.cap_seeds == 0, "null seeds");
    DeviceGuard dg(plan->device);
    cudaStream_t st = plan->stream;
    if (px.cap_seeds)
      CB_CUDA(cudaMemcpyAsync(plan->seeds, seeds, px.cap_seeds * 4,
                              seeds_on_device ? cudaMemcpyDeviceToDevice
                                              : cudaMemcpyHostToDevice,
                              st));
    upload_variates(plan, sched, 1, st);
    require(!px.eager_since_capture, "eager peer-exchange steps ran since the capture (re-capture)");
    const int g = static_cast<int>(px.replays % px.n_exec);
    count_epoch_bumps(plan, st, plan->L);
    CB_CUDA(cudaGraphLaunch(px.exec[g], st));
    for (int l = 0; l < plan->L; ++l)
      px.slot_of[l] = static_cast<int>((static_cast<uint64_t>(g) * plan->L + l) % 4);
    ++px.replays;
    plan->seeds_off.assign({0, px.cap_seeds});
    plan->mode = CB_MODE_COOP;
    plan->have_batch = true;
    plan->have_rows = px.cap_rows;
    plan->dirty_mode = -1;
    plan->launches = px.cap_launches;
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
    h2d_sync(px.d_fbase, px.fbase.data(), kMaxParts * sizeof(void*));
  });
}

int cb_px_gather(cb_plan* plan, const cb_features* local) {
  NvtxRange nvtx_("cb.px_gather");
  return guard([&] {
    require(plan != nullptr && local != nullptr, "null argument");
    require(plan->have_batch, "no sampled batch in this plan");
    PxState& px = px_of(plan);
    DeviceGuard dg(plan->device);
    prepare_rows(plan, local, false);  // rows come from the owners' shards
    plan->have_rows = true;
    if (px.rstage) {  // through the owners' staging buffers
      require_staging(px);
      px_enqueue_staged_gather(plan, -1);
      return;
    }
    for (uint32_t q = 0; q < px.world; ++q)
      require(px.fbase[q] != nullptr, "feature shard of a rank not connected");
    PeWork& w = plan->pe[0];
    const int L = plan->L;
    launch_px_gather(px.d_fbase, px.owner, local->row_map, local->row_bytes, w.L[L - 1].src,
                     &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, plan->stream);
    plan->have_rows = true;
  });
}

// ---- owner staging: the feature fetch through the owners -------------------
// all_to_all_forward (coop.cpp:145-159) the way the reference does it: owner
// q loads the rows of its set S^L_q (every requested row it owns, sorted) from
// its own shard into a staging buffer exported through CUDA IPC; after a
// barrier each requester pulls row loc_row[j] of rank loc_part[j]'s staging
// buffer. Reading a peer's whole shard in place instead costs a translation
// miss per row once the shards are large (c4: 1.2 ms vs 24 us per step for two
// ranks sharing one B200), and each owned row crosses the storage channel
// once however many ranks requested it.
//
// With a cache (cb_px_set_cache; the per-GPU cache of the dependent-
// minibatch reuse at the OWNER) S^L_q goes through the owner's LRU in
// access_order(S^L_q, order_key) -- feature_load_sim's per-part loop
// (cache.cpp:100-110) with S^L_q as part q's accesses: hits come from the
// cache's HBM rows, misses from the shard (HBM or the pinned host tier).
int cb_px_setup_staging(cb_plan* plan, const cb_features* local, void* handle_out) {
  return guard([&] {
    require(plan != nullptr && local != nullptr && handle_out != nullptr, "null argument");
    PxState& px = px_of(plan);
    require(local->shard_rows > 0, "staging needs this rank's shard table");
    DeviceGuard dg(plan->device);
    PeWork& w = plan->pe[0];
    px.drop_graphs();
    for (void* p : px.ropened) CB_CUDA(cudaIpcCloseMemHandle(p));
    px.ropened.clear();
    if (px.rstage) CB_CUDA(cudaFree(px.rstage));
    px.stage_store = local;
    // row buffers of a peer-exchange plan: its src / owner-set capacities are
    // the world-times worst case (c4, 2 ranks: 45M / 90M rows = 11.5 / 23 GB
    // of fp16 rows per plan) against ~0.1M rows seen; the buffers are capped
    // at kPxRowsLimit rows and a step that needs more is flagged (CB_OVERFLOW)
    plan->rows_limit = kPxRowsLimit;
    px.rstage_rows = std::max<uint64_t>(std::min(w.cap_final, kPxRowsLimit), 1);
    CB_CUDA(cudaMalloc(&px.rstage, px.rstage_rows * local->row_bytes));
    if (!px.d_rstage) CB_CUDA(cudaMalloc(&px.d_rstage, kMaxParts * sizeof(void*)));
    px.rstage_of.assign(kMaxParts, nullptr);
    px.rstage_of[px.rank] = static_cast<const unsigned char*>(px.rstage);
    h2d_sync(px.d_rstage, px.rstage_of.data(), kMaxParts * sizeof(void*));
    cudaIpcMemHandle_t h;
    CB_CUDA(cudaIpcGetMemHandle(&h, px.rstage));
    std::memcpy(handle_out, &h, sizeof(h));
  });
}

int cb_px_connect_staging(cb_plan* plan, uint32_t q, const void* handle) {
  return guard([&] {
    require(plan != nullptr && handle != nullptr, "null argument");
    PxState& px = px_of(plan);
    require(px.rstage != nullptr, "call cb_px_setup_staging first");
    require(q < px.world && q != px.rank, "peer rank out of range (or self)");
    DeviceGuard dg(plan->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    CB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    px.ropened.push_back(p);
    px.rstage_of[q] = static_cast<const unsigned char*>(p);
    h2d_sync(px.d_rstage, px.rstage_of.data(), kMaxParts * sizeof(void*));
  });
}

int cb_px_set_cache(cb_plan* plan, cb_cache* cache) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    PxState& px = px_of(plan);
    if (cache) {
      require(px.stage_store != nullptr, "call cb_px_setup_staging first");
      require(cache->lru->row_bytes() == px.stage_store->row_bytes,
              "cache row size does not match the feature table");
      require(cache->lru->n_keys() >= plan->g->g.n, "cache key space smaller than the graph");
    }
    px.cache = cache;
  });
}

int cb_px_set_clock_cache(cb_plan* plan, cb_ccache* cache) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    PxState& px = px_of(plan);
    if (cache) {
      require(px.stage_store != nullptr, "call cb_px_setup_staging first");
      require(cache->cc->row_bytes() == px.stage_store->row_bytes,
              "cache row size does not match the feature table");
      DeviceGuard dg(plan->device);
      cache->cc->reserve(px.rstage_rows);
    }
    px.drop_graphs();  // captured steps baked the uncached staging in
    px.ccache = cache;
  });
}

int cb_px_set_requester_cache(cb_plan* plan, cb_cache* cache) {
  return guard([&] {
    require(plan != nullptr, "null plan");
    PxState& px = px_of(plan);
    if (cache) {
      require(px.stage_store != nullptr, "call cb_px_setup_staging first");
      require(cache->lru->row_bytes() == px.stage_store->row_bytes,
              "cache row size does not match the feature table");
      require(cache->lru->n_keys() >= plan->g->g.n, "cache key space smaller than the graph");
      require(cache != px.cache, "the requester cache must differ from the owner cache");
    }
    px.rcache = cache;
  });
}

int cb_px_requester_stats(const cb_plan* plan, uint64_t* remote, uint64_t* hits,
                          uint64_t* misses) {
  return guard([&] {
    require(plan != nullptr && plan->px != nullptr, "peer exchange not set up");
    const PxState& px = *plan->px;
    if (remote) *remote = px.r_last[0];
    if (hits) *hits = px.r_last[1];
    if (misses) *misses = px.r_last[2];
  });
}

int cb_px_gather_cached(cb_plan* plan, uint64_t order_key, uint64_t* owned, uint64_t* hits,
                        uint64_t* misses) {
  NvtxRange nvtx_("cb.px_gather_cached");
  return guard([&] {
    require(plan != nullptr, "null plan");
    require(plan->have_batch, "no sampled batch in this plan");
    PxState& px = px_of(plan);
    require(px.cache != nullptr, "no cache set (cb_px_set_cache)");
    require_staging(px);
    DeviceGuard dg(plan->device);
    check_overflow(plan);
    const int L = plan->L;
    PeWork& w = plan->pe[0];
    prepare_rows(plan, px.stage_store, false);
    const uint64_t n_own = host_meta(plan, 0, L).n_dst;
    require(n_own <= px.rstage_rows, "owner set larger than the staging buffer");
    DeviceLru& lru = *px.cache->lru;
    const uint64_t h0 = lru.hits(), m0 = lru.misses();
    CacheGatherSrc src;
    src.table = px.stage_store->table;
    src.row_map = px.stage_store->row_map;
    src.rows_out = px.rstage;
    lru.access_ids(w.owner_final, n_own, order_key, nullptr, 0, src, plan->stream);
    // every owner's rows are staged before any requester reads them; the
    // next step's staging comes after that step's barriers, which no rank
    // reaches before finishing this pull
    launch_px_barrier(px.bar, plan->stream);
    const uint64_t rb = px.stage_store->row_bytes;
    PxCaps caps;
    caps.overflow = w.sync.overflow;
    if (!px.rcache) {
      launch_px_gather_staged(px.d_rstage, w.loc_part[L - 1], w.loc_row[L - 1], rb,
                              &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, caps,
                              plan->stream);
    } else {
      // requester side: own rows from the own staging buffer; rows owned by
      // other ranks through this rank's LRU in access_order(R, order_key ^
      // requester tag) -- hits from its HBM rows, misses pulled from the
      // owners' staging buffers over peer memory, then placed requester-aligned
      if (px.r_cap < w.cap_rows || px.r_row_bytes != rb) {
        for (void* p : {static_cast<void*>(px.r_ids), static_cast<void*>(px.r_pos),
                        static_cast<void*>(px.r_miss), px.r_rows})
          if (p) CB_CUDA(cudaFree(p));
        px.r_cap = std::max<uint64_t>(w.cap_rows, 1);
        px.r_row_bytes = rb;
        CB_CUDA(cudaMalloc(&px.r_ids, px.r_cap * 4));
        CB_CUDA(cudaMalloc(&px.r_pos, px.r_cap * 4));
        CB_CUDA(cudaMalloc(&px.r_miss, px.r_cap * sizeof(void*)));
        CB_CUDA(cudaMalloc(&px.r_rows, px.r_cap * rb));
        if (!px.r_n) CB_CUDA(cudaMalloc(&px.r_n, 8));
      }
      launch_px_split_remote(w.L[L - 1].src, &plan->meta_at(0, L - 1)->n_src, w.cap_rows,
                             w.loc_part[L - 1], w.loc_row[L - 1], px.rank, px.d_rstage, rb,
                             px.r_ids, px.r_pos, px.r_miss, px.r_n, plan->stream);
      launch_px_gather_staged_local(px.d_rstage, w.loc_part[L - 1], w.loc_row[L - 1], rb,
                                    &plan->meta_at(0, L - 1)->n_src, w.cap_rows, w.rows, px.rank,
                                    caps, plan->stream);
      unsigned long long nr = 0;
      CB_CUDA(cudaMemcpyAsync(&nr, px.r_n, 8, cudaMemcpyDeviceToHost, plan->stream));
      CB_CUDA(cudaStreamSynchronize(plan->stream));
      DeviceLru& rl = *px.rcache->lru;
      const uint64_t rh0 = rl.hits(), rm0 = rl.misses();
      CacheGatherSrc rs;
      rs.miss_ptr = px.r_miss;
      rs.rows_out = px.r_rows;
      rl.access_ids(px.r_ids, nr, requester_key(order_key), nullptr, 0, rs, plan->stream);
      launch_px_scatter_rows(px.r_rows, px.r_pos, nr, rb, w.rows, plan->stream);
      px.r_last[0] = nr;
      px.r_last[1] = rl.hits() - rh0;
      px.r_last[2] = rl.misses() - rm0;
    }
    plan->have_rows = true;
    if (owned) *owned = n_own;
    if (hits) *hits = lru.hits() - h0;
    if (misses) *misses = lru.misses() - m0;
  });
}

}  // extern "C"
