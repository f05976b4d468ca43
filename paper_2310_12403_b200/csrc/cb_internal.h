// Host-side internals of libcoopbatch_b200: device handles, per-PE workspace
// and the kernel-launch entry points each .cu exposes to the orchestrator
// (capi.cu). Nothing here crosses the C-ABI (include/coopbatch_cuda.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <atomic>
#include <utility>
#include <vector>

#include "cb_device.cuh"

namespace cb {

// Error taxonomy of the C-ABI (mirrors common.hpp:12-31 + device failures).
enum Status : int {
  kOk = 0,
  kInput = 1,     // coopbatch::InputError
  kFormat = 2,    // coopbatch::FormatError
  kIo = 3,        // coopbatch::IoError
  kCuda = 4,
  kNccl = 5,
  kOverflow = 6,  // capacity-bounded buffer overflowed on device (retryable)
  kInternal = 7,
  kUncertified = 8,  // smoothed decisions inside the guard band left unresolved
};

struct Error : std::runtime_error {
  Status code;
  Error(Status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CB_CUDA(x) ::cb::cuda_check((x), #x)
#define CB_LAUNCH(what) ::cb::cuda_check(cudaGetLastError(), what)

// Host-to-device upload that is complete on return. A plain cudaMemcpy from
// pageable memory runs on the legacy stream and may return while the DMA from
// its staging buffer is still in flight; the library's kernels run on
// non-blocking streams that do not wait for the legacy stream.
inline void h2d_sync(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  cuda_check(cudaStreamSynchronize(0), "cudaStreamSynchronize(legacy)");
}

// Scoped device allocation, freed on every exit path (exceptions included).
class DevBuf {
 public:
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc"); }
  ~DevBuf() {
    if (p_) cudaFree(p_);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
};

inline void require(bool ok, const char* msg) {
  if (!ok) throw Error(kInput, msg);
}
// Callers in per-element loops test first and build the message only on
// failure (a std::string per element cost ~70 ns/seed on the host).
inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(kInput, msg);
}

// Kernel launch with programmatic stream serialisation (PDL), so the next
// kernel's launch and prologue overlap this one's tail; every kernel launched
// this way starts with cbdev::pdl_begin(). CB_PDL=0 disables it.
bool pdl_enabled();
// Kernels this process enqueued eagerly (graph replays not included).
extern std::atomic<unsigned long long> g_kernel_launches;
template <typename... KArgs, typename... Args>
void launch_ks(void (*kernel)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t st,
               Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, unsigned block, cudaStream_t st,
              Args&&... args) {
  launch_ks(kernel, grid, block, 0, st, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- graph ----
struct DeviceGraph {
  int device = 0;
  uint64_t n = 0, m = 0;
  uint64_t* indptr = nullptr;   // [n+1]
  uint32_t* indices = nullptr;  // [m]
  float* weights = nullptr;     // [m] or nullptr (graph.hpp:25; RW only)
  uint64_t max_degree = 0;
};

// ------------------------------------------------------- per-layer meta ----
// Device-resident counts produced by the kernels of one layer of one PE.
struct LayerMeta {
  unsigned long long n_dst;
  unsigned long long scan_total;   // scan-space size (sum of per-dst work)
  unsigned long long n_active;     // dsts with non-empty scan work
  unsigned long long n_edges;
  unsigned long long n_src;
  unsigned long long uncertified;  // smoothed decisions inside the guard band
  unsigned long long pad[2];
};

struct LayerBufs {
  uint32_t* dst = nullptr;          // D_l        (cap_dst)
  struct ActRec* act = nullptr;     // records of active dsts (cap_dst+1)
  uint32_t* tile_first = nullptr;   // scan tile -> first record (max_tiles+1)
  uint2* tile_list = nullptr;       // (tile, record) of single-record tiles from the
                                    // front, tiles with record boundaries from the back
  uint64_t* out_prefix = nullptr;   // NS output prefix (cap_dst+1)
  uint32_t* slots = nullptr;        // NS reservoir slots (cap_edges)
  uint2* edges = nullptr;           // (src_idx, dst_idx) (cap_edges)
  uint32_t* src = nullptr;          // S~_{l+1} sorted unique (cap_src)
  uint32_t* dst_pos = nullptr;      // (cap_dst)
  uint64_t cap_dst = 0, cap_edges = 0, cap_src = 0;
  bool dst_aliases_prev_src = false;
};

// Device scratch shared by every kernel of a PE's batch.
struct Sync {
  unsigned* epoch = nullptr;                  // [1] batch epoch (device)
  unsigned* tickets = nullptr;                // [2*kMaxTickets]: ticket, exit ctr
  unsigned long long* status_a = nullptr;     // [max_tiles]
  unsigned long long* status_b = nullptr;     // [max_tiles]
  unsigned long long* status_c = nullptr;     // [max_tiles]
  unsigned* overflow = nullptr;               // [1]
  uint32_t* keep_words = nullptr;             // [max_tiles*kLaborTile/32]
  uint2* stage = nullptr;                     // [max_tiles*kLaborTile] kept edges by position
  double* vtab = nullptr;                     // smoothed LABOR r_t table [n] (nullptr: none)
  uint64_t max_tiles = 0;
  static constexpr int kMaxTickets = 256;
  // tickets [kListTicket + 2l, +1]: layer l's single-record / mixed tile counts
  static constexpr int kListTicket = 192;
  // ticket [kPureTicket + l]: layer l's labor_mark phase-A work counter
  static constexpr int kPureTicket = 128;
};

// Bitmap dedup structure over the vertex id space.
// Two levels: bits (1 per vertex) and summ (1 per data word, set by the
// setter that turns a word non-zero), so extraction of large sparse bitmaps
// visits only non-empty words.
struct Bitmap {
  uint32_t* bits = nullptr;     // [words_padded]
  uint32_t* wprefix = nullptr;  // [words_padded] rank of first bit of word
  uint32_t* summ = nullptr;     // [words_padded / 32]
  uint64_t words = 0, words_padded = 0;
};

// Packed record of one active dst (scan work > 0), written by the frontier
// kernel so the scan-space kernels need one 32-byte load per dst.
//   LABOR/FULL: a = row base (indices[a + x] is the neighbour at position x),
//               b = integer keep threshold floor((k/d)*2^53) (plain), the
//                   double bits of k/d (smoothed), or ~0 = keep all
//   NS        : a = output offset of the dst's k slots, b = hash prefix
//               {kStreamNs, layer, s} under z1
struct ActRec {
  unsigned long long pre;  // scan-space prefix
  unsigned long long a;
  unsigned long long b;
  uint32_t di;             // index into D
  uint32_t d;              // degree
};

// Debug tracing (CB_TRACE=1): per kernel, per CTA (<= kTraceCtas) up to 8
// %globaltimer stamps at fixed points.
constexpr int kTraceCtas = 64;
constexpr int kTraceKernel = kTraceCtas * 8;
constexpr int kTraceSlots = 32 * kTraceKernel;

struct FrontierArgs {
  unsigned long long* trace;
  const uint32_t* D;
  LayerMeta* meta;
  unsigned long long n_dst_param;  // ~0 = read meta->n_dst
  const uint64_t* indptr;
  int kind;
  uint32_t k;
  int layer;
  const cbdev::Variates* var;
  uint32_t* set_bits;
  uint32_t* set_summ;
  ActRec* act;
  uint32_t* tile_first;
  uint64_t* out_prefix;
  uint32_t* slots;
  uint64_t cap_edges;
  uint64_t cap_tiles;  // scan tiles the plan holds (tile_first has cap_tiles + 1)
  uint2* tile_list;    // (LABOR/FULL, may be null) tile lists for labor_mark
  unsigned* list_ctr;  // [2]: single-record tiles, mixed tiles (zeroed per batch)
  uint64_t list_cap;
  unsigned* ticket;
  unsigned long long *st_a, *st_b, *st_c;
  const unsigned* epoch;
  int slot;
  unsigned* overflow;
};

struct LaborArgs {
  unsigned long long* trace;
  LayerMeta* meta;
  const ActRec* act;
  const uint32_t* tile_first;
  const uint32_t* D;
  const uint32_t* indices;
  int kind;
  uint32_t k;
  int layer;
  const cbdev::Variates* var;
  uint32_t* bits;
  uint32_t* summ;
  uint2* edges;
  uint32_t* slots;
  const uint2* tile_list;    // the frontier's tile lists (null: every tile in phase B)
  const unsigned* list_ctr;
  unsigned* pure_ticket;  // phase A's dynamic split of the single-record tiles
  uint64_t list_cap;
  uint32_t* keep_words;  // 1 bit per scan position (labor_mark -> labor_emit)
  uint2* stage;          // (t, dst index) of each kept scan position
  double* vtab;          // smoothed r_t per vertex (nullptr: evaluate per position)
  uint64_t n_vert;
  uint64_t cap_edges;
  unsigned* ticket;
  unsigned long long* status;
  const unsigned* epoch;
  int slot;
  unsigned* overflow;
};

// Random walks with restart (samplers.cpp:202-285 rw_block), one warp per dst.
struct RwArgs {
  const uint32_t* D;
  LayerMeta* meta;
  const uint64_t* indptr;
  const uint32_t* indices;
  const float* weights;  // nullptr = unweighted
  int layer;
  uint32_t k;            // fanout: top-k visited vertices per dst
  uint32_t walks, length;
  double restart;        // p
  const cbdev::Variates* var;
  uint32_t* bits;
  uint32_t* summ;
  uint32_t* slots;       // [cap_dst * k] ranked picks per dst
  uint64_t* cnt;         // [cap_dst] picks per dst
  uint2* edges;
  uint64_t cap_edges;
  unsigned long long* status;
  const unsigned* epoch;
  int slot;
  unsigned* ticket;
  unsigned* overflow;
};
constexpr uint32_t kRwMaxVisits = 512;  // rw_walks * rw_length per dst on the device

struct ExtractArgs {
  unsigned long long* trace;  // debug stamps (CB_TRACE), nullptr = off
  const uint32_t* bits;
  const uint32_t* summ;
  uint32_t* wprefix;
  uint32_t* zero_bits;  // optional: bitmap zeroed word-for-word on the way
  uint32_t* zero_summ;
  uint64_t words_padded;
  uint32_t* out;
  uint64_t cap_out;
  unsigned long long* count_out;
  unsigned long long* count_out2;
  unsigned* ticket;
  unsigned long long* status;
  const unsigned* epoch;
  int slot;
  unsigned* overflow;
};

struct RelabelArgs {  // edges == nullptr disables
  const uint32_t* bits;
  const uint32_t* wprefix;
  const LayerMeta* meta;
  uint2* edges;
  uint64_t cap_edges;
  const uint32_t* D;
  uint32_t* dst_pos;
};

constexpr int kExtractTileWords = 2048;  // bitmap padding granule (max tile)
constexpr uint64_t kExtractBigWords = 256 * 1024;  // summary-mode threshold
#ifndef CB_MARK_NT
#define CB_MARK_NT 128
#endif
#ifndef CB_MARK_IPT
#define CB_MARK_IPT 8
#endif
constexpr int kMarkNT = CB_MARK_NT;                // labor_mark block size
constexpr int kLaborTile = kMarkNT * CB_MARK_IPT;  // scan positions per mark tile
constexpr uint64_t kVtabMaxVerts = 1ULL << 26;  // smoothed variate table cap (512 MiB)
#ifndef CB_FRONTIER_IPT
#define CB_FRONTIER_IPT 1
#endif
constexpr int kFrontierIPT = CB_FRONTIER_IPT;  // destinations per frontier thread
constexpr int kFrontierTile = 256 * kFrontierIPT;
// Scan positions one layer may hold before the overflow retry doubles it
// (stage 8 B + keep bit per position: ~1.1 GB per part).
constexpr uint64_t kScanBudget = 1ULL << 27;

// ----------------------------------------------------- kernel launchers ----
// sample.cu
void launch_batch_begin(const Sync& s, uint32_t* clear_bits, uint32_t* clear_summ,
                        const uint32_t* clear_list,
                        const unsigned long long* clear_count, uint64_t clear_cap,
                        uint64_t nwords, cudaStream_t st);
void launch_frontier(const FrontierArgs& a, const RelabelArgs& r, uint64_t cap_dst,
                     uint64_t relabel_work, cudaStream_t st);
void launch_labor(const LaborArgs& a, uint64_t max_tiles, bool smooth, cudaStream_t st);
void launch_ns(const LaborArgs& a, const uint32_t* D, const uint64_t* out_prefix,
               const uint64_t* indptr, const uint32_t* indices, uint64_t cap_dst, bool smooth,
               cudaStream_t st);
void launch_extract(const ExtractArgs& a, cudaStream_t st);
void launch_rw(const RwArgs& a, uint64_t cap_dst, bool smooth, cudaStream_t st);
void launch_labor_post(const LaborArgs& a, uint64_t max_tiles, const ExtractArgs& e,
                       cudaStream_t st);
void launch_relabel(const RelabelArgs& r, uint64_t work, cudaStream_t st);
void launch_clear(Bitmap& bm, const uint32_t* list, const unsigned long long* count,
                  cudaStream_t st);
void launch_rank(const Bitmap& bm, const uint32_t* ids, const unsigned long long* count,
                 uint32_t* rank_out, cudaStream_t st);

int grid_for(uint64_t work_items, int per_block, int max_per_sm);

}  // namespace cb
