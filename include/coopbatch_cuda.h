/*
 * coopbatch_cuda.h — the C-ABI of libcoopbatch_b200.so, the B200-native
 * drop-in for the reference's cooperative sample + dedup + feature-gather
 * path (arxiv 2310.12403 "coopbatch", /root/reference/proj).
 *
 * Plain C: opaque handles, host pointers + sizes, int status codes. No torch
 * or CUDA types cross this boundary (streams are passed as void*).
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference/proj):
 *   cb_graph_create_from_csr  <- coopbatch::Graph / build_csr result
 *                                (include/coopbatch/graph.hpp:21-53,
 *                                 src/graph.cpp:17-48)
 *   cb_graph_generate_rmat    <- generate_powerlaw (graph.hpp:57-63,
 *                                src/graph.cpp:111-151); R-MAT per DESIGN.md
 *   cb_partition_random       <- partition_random (partition.hpp:21-23,
 *                                src/partition.cpp:10-20)
 *   cb_partition_create       <- PartitionMap (partition.hpp:12-17)
 *   cb_features_synth         <- FeatureStore::synth (coop.hpp:140-150,
 *                                src/coop.cpp:359-376)
 *   cb_plan_create            <- SamplerConfig + num_layers (samplers.hpp:17-23)
 *   cb_sample (mode INDEP)    <- expand / indep_sample (samplers.hpp:167-169,
 *                                coop.hpp:55-58; src/samplers.cpp:340-354,
 *                                src/coop.cpp:108-119)
 *   cb_sample (mode COOP)     <- coop_sample (coop.hpp:49-52,
 *                                src/coop.cpp:68-106 + build_exchange 25-64)
 *   cb_gather                 <- FeatureStore::load_rows + all_to_all_forward
 *                                (coop.hpp:66-68,151; src/coop.cpp:145-159,
 *                                 378-388)
 *   cb_download_block         <- BipartiteBlock fields (samplers.hpp:30-38)
 *   cb_download_exchange      <- ExchangeRecord fields (coop.hpp:25-37)
 *   cb_download_owner_set     <- CoopSampleResult::owner_sets (coop.hpp:39-43)
 *   cb_cache_*                <- LruCache / feature_load_sim (cache.hpp:17-42,
 *                                80-83; src/cache.cpp:8-32, 74-119)
 *   cb_stack_fingerprint,     <- stack_fingerprint / run_dependent_experiment
 *   cb_shuffled_order            order (src/cache.cpp:123-162)
 *   cb_partition_members      <- part_members (partition.hpp:33-36)
 *   cb_gcn_*, cb_train_step   <- GcnModel, gcn_forward/backward, coop_train_step,
 *                                indep_train_step (coop.hpp:105-185)
 *   cb_px_*                   <- coop_sample + build_exchange + all_to_all_forward
 *                                across processes (coop.cpp:25-106, 145-159)
 *   cb_last_error             <- the what() of coopbatch::InputError etc.
 *                                (include/coopbatch/common.hpp:12-31)
 */
#ifndef COOPBATCH_CUDA_H
#define COOPBATCH_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (0 = ok). CB_INPUT maps to coopbatch::InputError. */
enum {
  CB_OK = 0,
  CB_INPUT = 1,
  CB_FORMAT = 2,
  CB_IO = 3,
  CB_CUDA = 4,
  CB_NCCL = 5,
  CB_OVERFLOW = 6,
  CB_INTERNAL = 7,
  CB_UNCERTIFIED = 8 /* smoothed decisions inside the guard band left unresolved */
};

/* SamplerKind order of samplers.hpp:15 */
enum { CB_FULL = 0, CB_NS = 1, CB_LABOR0 = 2, CB_RW = 3 };
enum { CB_MODE_COOP = 0, CB_MODE_INDEP = 1 };
enum { CB_F64 = 0, CB_F32 = 1, CB_F16 = 2 };

/* SeedSchedule (rng.hpp:93-111); kappa = UINT64_MAX is infinity. */
typedef struct cb_sched {
  uint64_t kappa;
  uint64_t z1;
  uint64_t z2;
  uint64_t iteration;
} cb_sched;

/* VariateSource (samplers.hpp:61-126) given directly: z1, z2, cos/sin of the
 * contribution (exact 1/0 at the endpoints), smoothed flag. */
typedef struct cb_variates {
  uint64_t z1;
  uint64_t z2;
  double cos_c;
  double sin_c;
  int smoothed;
} cb_variates;

typedef struct cb_graph cb_graph;
typedef struct cb_partition cb_partition;
typedef struct cb_features cb_features;
typedef struct cb_plan cb_plan;

/* Thread-local message of the last failing call on this thread. */
const char* cb_last_error(void);
const char* cb_version(void);
int cb_device_count(int* out);

/* ---- graph (CSR resident in HBM) ---- */
int cb_graph_create_from_csr(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                             uint64_t m, int device, cb_graph** out);
/* CBCS binary CSR (graph.hpp:78-80; load_csr / save_csr, src/graph.cpp:196-265):
 * CB_IO when the file cannot be opened/written, CB_FORMAT for a bad magic,
 * version or truncation, CB_INPUT when validate_csr fails. Weights in a file
 * are validated and kept (cb_graph_set_weights). */
int cb_graph_load_cbcs(const char* path, int device, cb_graph** out);
/* Edge weights (graph.hpp:25, Graph::weights; one float per edge, > 0, CB_INPUT
 * otherwise; nullptr drops them). Only the RW sampler reads them:
 * pick_neighbor's weighted choice, samplers.cpp:139-165. */
int cb_graph_set_weights(cb_graph* g, const float* weights);
int cb_graph_save_cbcs(const cb_graph* g, const char* path);
int cb_graph_generate_rmat(uint64_t n, uint64_t m, uint64_t seed, int device,
                           cb_graph** out);
int cb_graph_info(const cb_graph* g, uint64_t* n, uint64_t* m, uint64_t* max_degree);
int cb_graph_download(const cb_graph* g, uint64_t* indptr, uint32_t* indices);
void cb_graph_destroy(cb_graph* g);

/* ---- 1D vertex ownership ---- */
int cb_partition_random(const cb_graph* g, uint32_t parts, uint64_t seed, cb_partition** out);
int cb_partition_create(const cb_graph* g, const uint32_t* owner, uint32_t parts,
                        cb_partition** out);
int cb_partition_download(const cb_partition* pm, uint32_t* owner);
/* cross_edge_ratio (partition.hpp:29-31, src/partition.cpp:79-89): edges whose
 * endpoints have different owners, and their fraction of all edges. */
int cb_cross_edge_ratio(const cb_graph* g, const cb_partition* pm, uint64_t* cross,
                        double* ratio);
/* part_members (partition.hpp:33-36, src/partition.cpp:99-105): the vertices of
 * all parts concatenated part-major, ascending within a part (members[n]);
 * shard_off[parts+1] = start of each part. This order is the feature shard
 * layout (row of v = its index here). Either pointer may be NULL. */
int cb_partition_members(const cb_partition* pm, uint32_t* members, uint64_t* shard_off);
void cb_partition_destroy(cb_partition* pm);

/* ---- feature tables (row-sharded by owner when pm != NULL) ---- */
int cb_features_synth(const cb_graph* g, const cb_partition* pm, uint32_t dim, int dtype,
                      uint64_t seed, cb_features** out);
int cb_features_info(const cb_features* f, uint32_t* dim, int* dtype, uint64_t* row_bytes);
void cb_features_destroy(cb_features* f);

/* ---- sampling plan ---- */
/* fanouts[l] applies at block l (seeds outward); pm may be NULL for P = 1. */
int cb_plan_create(const cb_graph* g, const cb_partition* pm, int num_layers, int kind,
                   const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out);
/* A plan of `parts` independent parts without a partition (indep mode only):
 * the trial batches of work_curve / indep_sample at equal global batch. */
int cb_plan_create_parts(const cb_graph* g, uint32_t parts, int num_layers, int kind,
                         const uint32_t* fanouts, uint64_t max_seeds_per_part, cb_plan** out);
void cb_plan_destroy(cb_plan* plan);
int cb_plan_num_parts(const cb_plan* plan, uint32_t* parts);
/* The CUDA stream every kernel of this plan runs on (cudaStream_t). */
void* cb_plan_stream(const cb_plan* plan);

/* One batch. seeds_flat holds the P per-part seed lists back to back,
 * seeds_off[P+1] their offsets (host memory). Enqueues everything on the plan
 * stream; cb_sample_sync additionally waits and retries with larger
 * buffers if a capacity bound overflowed. */
int cb_sample(cb_plan* plan, int mode, const uint32_t* seeds_flat, const uint64_t* seeds_off,
              const cb_sched* sched);
int cb_sample_sync(cb_plan* plan, int mode, const uint32_t* seeds_flat,
                   const uint64_t* seeds_off, const cb_sched* sched);
/* Block l of the plan hashes as layer l + base: sample_block(g, seeds, cfg,
 * src, layer) (samplers.hpp:158-160) at any layer is a 1-layer plan with
 * base = layer. Drops captured graphs. */
int cb_plan_set_layer_base(cb_plan* plan, int base);
/* sample_block(..., const VariateSource&, layer) (samplers.hpp:158-160): the
 * plan's next batches draw from this source instead of the schedule passed to
 * cb_sample* (whose kappa is then ignored); nullptr
 * returns to schedule-derived variates. */
int cb_plan_set_variate_source(cb_plan* plan, const cb_variates* v);
/* sample_labor0 / labor_block (samplers.cpp:89-104, 305-312) with the
 * caller's variate r(t) instead of the hash stream: table[t] for every vertex
 * t (num_vertices doubles, host or device memory; copied). While a table is
 * set, every LABOR layer of the plan keeps t -> s iff table[t] <= (double)k /
 * (double)d_s, the reference's comparison, with no keep-all shortcut for
 * d_s <= k (a caller variate may exceed 1). NULL restores the schedule's
 * stream. LABOR-0 plans only; drops captured graphs. */
int cb_plan_set_variate_table(cb_plan* plan, const double* table, int on_device);
/* P independent expansions in one batch, part p under its own schedule
 * scheds[p] (indep mode; all schedules plain or all smoothed). This is the
 * trial loop of work_curve (analysis.cpp:78-124: a fresh plain stream
 * hash_bits(seed, {tag, 9}) per trial) with the trials as concurrent parts.
 * Waits, and retries with larger buffers on overflow like cb_sample_sync. */
int cb_sample_multi(cb_plan* plan, const uint32_t* seeds_flat, const uint64_t* seeds_off,
                    const cb_sched* scheds);
/* Same, seeds already in device memory (seeds_off on host). */
int cb_sample_device(cb_plan* plan, int mode, const uint32_t* d_seeds_flat,
                     const uint64_t* seeds_off, const cb_sched* sched);

/* Gather input-feature rows of every part's input vertices (requester
 * aligned, = all_to_all_forward of the owners' load_rows). */
int cb_gather(cb_plan* plan, const cb_features* f);

/* Wait for the plan stream; CB_OVERFLOW if a capacity bound was exceeded. */
int cb_synchronize(cb_plan* plan);

/* sizes[0..5] = n_dst, n_src, n_edges, uncertified, scan_total, n_active */
int cb_layer_sizes(cb_plan* plan, uint32_t part, int layer, uint64_t* sizes);
int cb_download_block(cb_plan* plan, uint32_t part, int layer, uint32_t* dst, uint32_t* src,
                      uint32_t* edges /* 2 per edge */, uint32_t* dst_pos);
/* The whole batch result of one part in one call, for callers that want it in
 * host memory (the reference returns LayerStacks and FeatureMatrix rows by
 * value: samplers.hpp:42-49, coop.hpp:83-91, 151): every layer's dst, src,
 * edges and dst_pos, plus the gathered rows when the batch has them, written
 * by one kernel into pinned (cudaHostAlloc'd / registered) host memory, on the
 * plan stream, without a host round trip. Layout and the truncation header:
 * csrc/result.cu. cb_plan_result_bytes bounds the size from the plan's
 * capacities. */
int cb_plan_result_bytes(const cb_plan* plan, uint32_t part, uint64_t row_bytes,
                         uint64_t* max_bytes);
int cb_plan_result_async(cb_plan* plan, uint32_t part, void* host_pinned, uint64_t cap_bytes);
/* The same layout through a copy engine. cb_plan_result_pack enqueues the
 * packing of the batch's result into a device staging buffer (asynchronous;
 * call it right after the batch). cb_plan_result_copy waits for the batch and
 * its pack (packing first if nothing was packed for this batch), then enqueues
 * ONE D2H copy of the packed bytes on cb_plan_stream (host_pinned should be
 * pinned for asynchrony) and returns; *total_bytes = the result's size (a
 * truncated header only, as the kernel form, when it exceeds cap_bytes). */
int cb_plan_result_pack(cb_plan* plan, uint32_t part);
int cb_plan_result_copy(cb_plan* plan, uint32_t part, void* host_pinned, uint64_t cap_bytes,
                        uint64_t* total_bytes);
int cb_owner_set_size(cb_plan* plan, uint32_t part, uint64_t* n);
int cb_download_owner_set(cb_plan* plan, uint32_t part, uint32_t* ids);
/* send_counts[P*P] (row = sender), owner_row_counts[P]; loc_* hold part p's
 * src_location entries back to back in part order. */
int cb_download_exchange(cb_plan* plan, int layer, uint64_t* send_counts,
                         uint64_t* owner_row_counts, uint32_t* loc_part, uint64_t* loc_row);
/* Gathered rows of `part` (n_src(L-1) x row_bytes). */
int cb_download_rows(cb_plan* plan, uint32_t part, void* out);
/* Device pointer of `part`'s gathered rows (for in-HBM consumers). */
int cb_rows_device(cb_plan* plan, uint32_t part, void** ptr, uint64_t* rows);

/* CUDA-graph form of one batch: capture the launch sequence for fixed
 * per-part seed counts (seeds_off) once, then replay per step with new seeds
 * (host or device pointer) and new variate keys. `sched` fixes whether the
 * smoothed (2 <= kappa < inf) kernels are captured; replays must match.
 * what: 1 = sample, 2 = gather (needs f at capture), 3 = both. */
int cb_plan_capture(cb_plan* plan, int mode, const uint64_t* seeds_off, const cb_features* f,
                    const cb_sched* sched);
int cb_plan_replay(cb_plan* plan, const uint32_t* seeds_flat, int seeds_on_device,
                   const cb_sched* sched, int what);

/* ---- multi-process cooperative step (one rank = one part) ----
 * The library runs each part's kernels; the caller moves ids/rows between
 * ranks (NCCL all-to-allv). This is build_exchange (coop.cpp:25-64) and
 * all_to_all_forward (coop.cpp:145-159) split at the rank boundary.
 * All pointers named d_* are device pointers on the plan's device. */
int cb_plan_create_dist(const cb_graph* g, uint32_t world, int num_layers, int kind,
                        const uint32_t* fanouts, uint64_t max_seeds, cb_plan** out);
/* Sample block `layer` for frontier d_dst[n_dst]; returns |src| (sorted
 * unique sampled ids, device list via cb_plan_layer_src). Synchronous. */
int cb_plan_sample_layer(cb_plan* plan, int layer, const uint32_t* d_dst, uint64_t n_dst,
                         const cb_sched* sched, uint64_t* n_src);
int cb_plan_layer_src(cb_plan* plan, int layer, uint32_t** d_src);
/* Stable partition of d_ids by d_owner[id] (bucket-major, input order inside
 * a bucket); d_perm[k] = input index of d_out[k]; counts[parts] on host. */
int cb_bucket_by_owner(cb_plan* plan, const uint32_t* d_ids, uint64_t n, const uint32_t* d_owner,
                       uint32_t parts, uint32_t* d_out, uint32_t* d_perm, uint64_t* counts);
/* Owner side: sorted unique of the received ids -> d_next (next layer's
 * seeds), and d_rank[i] = row of d_recv[i] in d_next. */
int cb_merge_owned(cb_plan* plan, int layer, const uint32_t* d_recv, uint64_t n_recv,
                   uint32_t* d_next, uint64_t cap_next, uint64_t* n_next, uint32_t* d_rank);
/* d_out[d_perm[k]] = d_in[k] (u32 values / feature rows of row_bytes). */
int cb_scatter_u32(cb_plan* plan, const uint32_t* d_in, const uint32_t* d_perm, uint64_t n,
                   uint32_t* d_out);
int cb_scatter_rows(cb_plan* plan, const void* d_in, const uint32_t* d_perm, uint64_t n,
                    uint64_t row_bytes, void* d_out);
/* The feature rows of one part only (its members in ascending id order). */
int cb_features_synth_shard(const cb_graph* g, const cb_partition* pm, uint32_t part,
                            uint32_t dim, int dtype, uint64_t seed, cb_features** out);
/* d_out[i] = row of vertex d_ids[i] (owned by the table's part). */
int cb_gather_rows(const cb_features* f, const uint32_t* d_ids, uint64_t n, void* d_out,
                   void* stream);

/* Synchronous copy between any host/device pointers (cudaMemcpyDefault). */
int cb_memcpy(void* dst, const void* src, uint64_t bytes, int device);

/* One eager batch (+ gather when f != NULL) with a CUDA event after every
 * launch: ms[i] = device time of launch i, in enqueue order. */
int cb_plan_profile(cb_plan* plan, int mode, const uint32_t* seeds_flat,
                    const uint64_t* seeds_off, const cb_sched* sched, const cb_features* f,
                    float* ms, int max_n, int* n);

/* Replay the captured batch once through its profiling twin (event-record
 * nodes between launches): ms[i] = in-graph device time of launch i. */
int cb_plan_graph_profile(cb_plan* plan, const uint32_t* d_seeds, const cb_sched* sched,
                          float* ms, int max_n, int* n);

/* Debug: globaltimer stamps of the last batch (plan created with CB_TRACE=1). */
int cb_plan_trace(cb_plan* plan, uint64_t* out, uint64_t n);

/* Kernels in one replay of the captured graphs: what = 1 sample, 2 gather,
 * 3 sample + gather (there the last layer's relabel of a 1-part plan is fused
 * into the gather launch, so it is one fewer than 1 + 2), 4 the captured
 * peer-exchange step (cb_px_capture). */
int cb_plan_captured_launches(const cb_plan* plan, int what, uint64_t* n);
/* Number of kernels one cb_sample/cb_gather call enqueues (for reporting). */
int cb_plan_launch_count(const cb_plan* plan, int mode, int with_gather, uint64_t* n);

/* ---- per-GPU feature cache (LruCache, cache.hpp:17-42; cache.cpp:8-32) ----
 * Exact LRU semantics evaluated one id set at a time on the device: the ids
 * of a step (sorted unique, e.g. input_vertices()) are accessed in
 * access_order(ids, order_key) (cache.cpp:74-84), optionally only those with
 * owner == part (feature_load_sim's cooperative filter, cache.cpp:105).
 * row_bytes > 0 gives the cache HBM row storage: with a backing table and
 * d_rows_out, rows of the kept ids are produced in kept (ascending id) order,
 * hits read from the cache, misses from the table (HBM or host tier). */
typedef struct cb_cache cb_cache;
int cb_cache_create(int device, uint64_t n_keys, uint64_t capacity, uint64_t row_bytes,
                    cb_cache** out);
void cb_cache_destroy(cb_cache* c);
/* LruCache::access over an arbitrary host trace: miss[i] = 1 on a miss. */
int cb_cache_access_trace(cb_cache* c, const uint32_t* keys, uint64_t n, uint8_t* miss);
int cb_cache_access_ids(cb_cache* c, const uint32_t* d_ids, uint64_t n, uint64_t order_key,
                        const cb_partition* pm, uint32_t part, const cb_features* backing,
                        void* d_rows_out, uint64_t* kept, void* stream);
/* Host id list (uploaded, then as cb_cache_access_ids without rows). */
int cb_cache_access_host_ids(cb_cache* c, const uint32_t* ids, uint64_t n, uint64_t order_key,
                             const cb_partition* pm, uint32_t part, uint64_t* kept);
/* Same, over the input vertices of part `part` of the plan's last batch.
 * backing != NULL and d_rows_out == NULL: the rows land in the plan's row
 * buffer (cb_download_rows), which needs pm == NULL. */
int cb_cache_access_plan(cb_cache* c, cb_plan* plan, uint32_t part, uint64_t order_key,
                         const cb_partition* pm, uint32_t owner_part,
                         const cb_features* backing, void* d_rows_out, uint64_t* kept);
int cb_cache_stats(const cb_cache* c, uint64_t* hits, uint64_t* misses, uint64_t* size);
int cb_cache_reset_counters(cb_cache* c);
/* LruCache::resident(): resident keys, most recent first. */
int cb_cache_resident(cb_cache* c, uint32_t* out, uint64_t cap_out, uint64_t* n);
int cb_cache_storage(const cb_cache* c, const void** d_rows);

/* ---- fast per-GPU feature cache: set-associative, CLOCK replacement ----
 * The production cache mode: three kernels per batch (lookup,
 * serve, insert), no sort, no host round trip, so it can sit inside a
 * captured step. Its hit rate is its own (not LruCache's: cb_cache_* is the
 * batch-exact LRU for parity); rows served are always the table's rows.
 * cb_ccache_gather_plan: the input rows of part `part` of the plan's last
 * batch into the plan's row buffer (cb_download_rows / cb_rows_device), hits
 * from the cache, misses from `backing` (HBM or host tier), misses inserted. */
typedef struct cb_ccache cb_ccache;
int cb_ccache_create(int device, uint64_t capacity, uint32_t ways, uint64_t row_bytes,
                     cb_ccache** out);
void cb_ccache_destroy(cb_ccache* c);
int cb_ccache_gather_plan(cb_ccache* c, cb_plan* plan, uint32_t part, const cb_features* backing);
/* Running totals: hits, inserted rows, slots (synchronises the device). */
int cb_ccache_stats(cb_ccache* c, uint64_t* hits, uint64_t* inserted, uint64_t* capacity);

/* stack_fingerprint (cache.cpp:123-133) of part `part` of the last batch. */
int cb_stack_fingerprint(cb_plan* plan, uint32_t part, uint64_t* out);
/* run_dependent_experiment's fixed training order (cache.cpp:155-162). */
int cb_shuffled_order(uint64_t n, uint64_t seed, uint32_t* out);
/* Feature storage tier: 1 = pinned host memory mapped into the device
 * (the paper's storage channel), 0 = HBM. */
int cb_features_set_tier(cb_features* f, int host);
/* SamplerConfig's random-walk parameters (samplers.hpp:19-22) of a CB_RW
 * plan: rw_length o >= 1, rw_restart p in [0,1), rw_walks a >= 1, with
 * a*o <= 512 visits per dst on the device. Defaults 3 / 0.5 / 100. */
/* Smoothed variates (2 <= kappa < inf): the device's Phi / Phi^-1 may differ
 * from glibc's by an ulp, so a keep / slot decision whose variate lies within
 * `band` (relative, default 1e-12) of its threshold is recorded. cb_sample_sync
 * evaluates every recorded decision with the reference's own arithmetic on
 * the host (VariateSource::finish, samplers.hpp:96-100; rng.cpp:7-52); if any
 * differs from the device's, the batch is sampled again with the exact values
 * (repeated until no new in-band decision appears), so the result is the
 * reference's by construction. Asynchronous paths (cb_sample, replays, cb_px_*)
 * cannot resolve: with `strict` (default 1) their cb_synchronize / downloads
 * return CB_UNCERTIFIED when a recorded decision is left. `perturb` != 0 is a
 * test hook that flips every unresolved in-band device decision. */
int cb_plan_set_guard(cb_plan* plan, double band, int perturb, int strict);
/* Of the last cb_sample_sync: decisions resolved on the host, and re-samplings. */
int cb_plan_resolve_stats(const cb_plan* plan, uint64_t* resolved, uint64_t* reruns);
int cb_plan_set_rw(cb_plan* plan, uint32_t rw_length, double rw_restart, uint32_t rw_walks);
/* Asynchronous D2H (on cb_plan_stream) of the batch's per-part, per-layer
 * counts (n_dst, scan_total, n_active, n_edges, n_src, uncertified, 2 pad;
 * u64 each, P x (L+1) records) into host_dst (pinned for true asynchrony).
 * host_dst == NULL: only *bytes is set. */
int cb_plan_meta_async(cb_plan* plan, void* host_dst, uint64_t* bytes);
/* Kernels of this library enqueued eagerly by this process so far (CUDA
 * graph replays excluded; for reporting launch counts). */
int cb_kernel_launches(uint64_t* n);
/* Device pointer + count of the input vertices of part `part`. */
int cb_plan_input_ids(cb_plan* plan, uint32_t part, const uint32_t** d_ids, uint64_t* n);

/* ---- multi-process peer exchange (one part per rank, CUDA IPC) ----
 * coop_sample (coop.cpp:68-106) with build_exchange (coop.cpp:25-64) done in
 * peer memory: requesters OR their src ids straight into the owners'
 * exchange bitmaps over NVLink, owners extract their sorted sets in place,
 * requesters read their ranks back from the owners' bitmaps; input rows are
 * pulled from the owners' shards (all_to_all_forward, coop.cpp:145-159).
 * No counts cross ranks and nothing syncs with the host: between
 * cb_px_layer -> cb_px_owner -> cb_px_locate of a layer goes a cross-rank
 * barrier ordered on cb_plan_stream -- cb_px_barrier (a device barrier on
 * flags in the IPC region), an NCCL all-reduce on that stream, or a host
 * barrier after a stream sync. Handles are 64 bytes. */
int cb_px_setup(cb_plan* plan, const cb_partition* pm, uint32_t rank, void* handle_out);
int cb_px_connect(cb_plan* plan, uint32_t peer, const void* handle);
int cb_px_layer(cb_plan* plan, int layer, const uint32_t* seeds, uint64_t n_seeds,
                const cb_sched* sched);
int cb_px_owner(cb_plan* plan, int layer);
int cb_px_locate(cb_plan* plan, int layer);
/* Waits for pending work; CB_OVERFLOW on a capacity overflow, CB_CUDA when a
 * device barrier timed out (CB_PX_BARRIER_TIMEOUT_MS, default 20 s). */
int cb_px_finish(cb_plan* plan);
/* Device barrier across the ranks, ordered on cb_plan_stream: a one-warp
 * kernel stores this rank's arrival (release, system scope) into every peer's
 * flag array and waits for every peer's (acquire). Every rank must issue the
 * same number of barriers. */
int cb_px_barrier(cb_plan* plan);
/* The whole cooperative step (coop_sample, coop.cpp:92-102; then the row pull
 * of cb_px_gather when local != NULL) captured as CUDA graphs (2 or 4, replayed
 * in turn): per layer l, sample + route into exchange slot c % 4 (c = the
 * run's layer count), ONE device barrier, the owner extracts slot c % 4 and
 * the requester locates layer l - 1; one more barrier and the last locate end
 * the step -- L + 1 barriers instead of 2L. Barriers are a signal kernel plus
 * stream memory waits (cuStreamWaitValue32; CB_PX_BARRIER=spin: the spin
 * kernel of cb_px_barrier). Fixed seed count n_seeds; the schedule fixes only
 * whether variates are smoothed. Every rank must have run one eager step
 * before (kernel attributes), be quiescent (no step in flight on any rank),
 * and capture the same step. Eager steps after a replay need a new plan. */
int cb_px_capture(cb_plan* plan, uint64_t n_seeds, const cb_sched* sched,
                  const cb_features* local);
/* One captured step: seeds (host or device) + the schedule's variates are
 * copied on cb_plan_stream, then the graph is launched. No host sync. */
int cb_px_replay(cb_plan* plan, const uint32_t* seeds, int seeds_on_device,
                 const cb_sched* sched);
int cb_px_sizes(cb_plan* plan, int layer, uint64_t* n_src, uint64_t* n_owned);
/* This rank's send_counts row, src_location, and its owned set after layer l. */
int cb_px_download(cb_plan* plan, int layer, uint64_t* send_row, uint32_t* loc_part,
                   uint32_t* loc_row, uint32_t* owned);
int cb_features_export(const cb_features* f, void* handle_out, uint64_t* shard_r0);
int cb_px_connect_features(cb_plan* plan, uint32_t peer, const void* handle, uint64_t shard_r0,
                           const cb_features* local);
/* Input rows of this rank's last layer into the plan's row buffer
 * (cb_download_rows / cb_rows_device), requester-aligned. */
int cb_px_gather(cb_plan* plan, const cb_features* local);
/* Owner staging (all_to_all_forward, coop.cpp:145-159, as the reference does
 * it): with a staging buffer set up and connected on every rank, cb_px_gather
 * and the captured step's row fetch become: owner q loads the rows of its set
 * S^L_q from its shard into its staging buffer (exported through CUDA IPC), a
 * device barrier, then each requester pulls row loc_row[j] of rank
 * loc_part[j]'s buffer. cb_px_set_cache adds the per-GPU cache at the owner
 * (feature_load_sim, cache.cpp:88-119, with S^L_q as part q's accesses):
 * cb_px_gather_cached runs S^L_q through the LRU in access_order(S^L_q,
 * order_key), hits from the cache's HBM rows, misses from the shard (HBM or
 * the host tier, cb_features_set_tier); every rank calls it once per step;
 * *owned / *hits / *misses are this owner's. It synchronises with the host
 * (the owner-set size). */
int cb_px_setup_staging(cb_plan* plan, const cb_features* local, void* handle_out);
int cb_px_connect_staging(cb_plan* plan, uint32_t peer, const void* handle);
int cb_px_set_cache(cb_plan* plan, cb_cache* cache);
/* Requester-side cache for cb_px_gather_cached: the requested rows owned by
 * other ranks go through `cache` (a second LRU, keys = vertex ids) in
 * access_order(R, hstep(order_key, "REQUE")): hits come from its HBM rows,
 * only misses cross NVLink (pulled from the owners' staging buffers). NULL
 * detaches it. cb_px_requester_stats: the last step's remote rows, hits and
 * misses (misses x row bytes = the peer bytes of the step). */
int cb_px_set_requester_cache(cb_plan* plan, cb_cache* cache);
/* The CLOCK cache (cb_ccache_*) in front of this owner's staging: cb_px_gather
 * and the captured step's row fetch serve S^L_q from it (misses from the
 * shard) -- no host round trip, so the cached fetch is part of the graph.
 * Drops captured graphs (re-capture); NULL detaches it. */
int cb_px_set_clock_cache(cb_plan* plan, cb_ccache* cache);
int cb_px_requester_stats(const cb_plan* plan, uint64_t* remote, uint64_t* hits,
                          uint64_t* misses);
int cb_px_gather_cached(cb_plan* plan, uint64_t order_key, uint64_t* owned, uint64_t* hits,
                        uint64_t* misses);

/* ---- GCN training step (coop.hpp:105-185; coop.cpp:161-357, 394-610) ----
 * GcnModel on the device: weights[l] (rows x cols, f64 row-major) is used at
 * block l; hidden layers use tanh, block 0 the identity (logits). */
typedef struct cb_model cb_model;
/* GcnModel::init (coop.cpp:334-357) */
int cb_gcn_model_init(int device, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                      int num_layers, uint64_t seed, cb_model** out);
/* Read (upload = 0) or write (upload = 1) the weights of one layer. */
/* GcnModel with explicit layer shapes and host weights (coop.hpp:126-135);
 * weights row-major, layer after layer. */
int cb_gcn_model_create(int device, int num_layers, const uint32_t* rows, const uint32_t* cols,
                        int tanh_hidden, const double* weights, cb_model** out);
int cb_gcn_model_weights(cb_model* m, int layer, double* host, int upload, uint64_t* rows,
                         uint64_t* cols);
void cb_gcn_model_destroy(cb_model* m);
/* coop_train_step (mode COOP, P > 1) / indep_train_step over the plan's last
 * batch with an f64 FeatureStore (labels = hash(seed,{10,v}) mod classes):
 * mean loss over all seeds and the part-summed weight gradients, layer 0
 * first, each rows x cols (grad_w may be NULL). */
int cb_train_step(cb_plan* plan, const cb_features* store, uint32_t classes, cb_model* model,
                  double* loss, double* grad_w);

/* ---- host-buffer ops for the C++ drop-in (paper_2310_12403_b200/dropin) ----
 * The reference's signatures take and return host vectors; these run the
 * device kernels of the path on uploaded operands and copy the result back.
 * An exchange record is given as P requester lists concatenated: loc_off[P+1],
 * src_location parts / rows (coop.hpp:25-37), owner_row_counts[P]. */
/* all_to_all_forward (coop.hpp:66-68, coop.cpp:145-159) */
int cb_op_forward_rows(int device, uint32_t P, const uint64_t* loc_off, const uint32_t* loc_part,
                       const uint64_t* loc_row, const uint64_t* owner_row_counts, uint32_t dim,
                       const double* owner_flat, double* out_flat);
/* all_to_all_reverse (sum = 0, last writer in (part, index) order) and
 * all_to_all_reverse_sum (sum = 1, summed in (part, index) order)
 * (coop.hpp:70-80, coop.cpp:161-194) */
int cb_op_reverse_rows(int device, uint32_t P, const uint64_t* loc_off, const uint32_t* loc_part,
                       const uint64_t* loc_row, const uint64_t* owner_row_counts, uint32_t dim,
                       const double* requester_flat, int sum, double* owner_out_flat);
/* gcn_forward (out) and, with grad_out, gcn_backward (grad_h_in, grad_w) of one
 * block (coop.hpp:106-124, coop.cpp:196-331); edges (src_idx, dst_idx) pairs. */
int cb_op_gcn_block(int device, uint64_t n_src, uint64_t n_dst, uint64_t n_edges,
                    const uint32_t* edges, const uint32_t* dst_pos, const double* h_in,
                    uint32_t in_dim, const double* w, uint32_t out_dim, int tanh_act,
                    const double* grad_out, double* out, double* grad_h_in, double* grad_w);
/* A feature table from host rows (FeatureStore::values) and its labels. */
int cb_features_from_host(int device, uint64_t n_rows, uint32_t dim, int dtype, const void* rows,
                          cb_features** out);
int cb_features_set_labels(cb_features* f, const uint32_t* labels);
/* A feature table over the caller's host rows, read in place by the device
 * (pinned + mapped until cb_features_destroy; the caller keeps the memory
 * alive and unmodified meanwhile). */
int cb_features_wrap_host(int device, uint64_t n_rows, uint32_t dim, int dtype, const void* rows,
                          cb_features** out);
/* FeatureStore::load_rows (coop.hpp:151, coop.cpp:378-388): host ids -> host
 * rows, gathered on the device. CB_INPUT for an id >= n_rows. */
int cb_op_load_rows(const cb_features* f, const uint32_t* ids, uint64_t n, void* out);
/* FeatureStore::synth (coop.cpp:359-376) on the device, into host arrays. */
int cb_synth_host(int device, uint64_t n, uint32_t dim, uint32_t classes, uint64_t seed,
                  double* values, uint32_t* labels);

#ifdef __cplusplus
}
#endif
#endif
