// Host-side internals of libcoopbatch_b200: device handles, per-PE workspace
// and the kernel-launch entry points each .cu exposes to the orchestrator
// (capi.cu). Nothing here crosses the C-ABI (include/coopbatch_cuda.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
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

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(kInput, msg);
}

// ---------------------------------------------------------------- graph ----
struct DeviceGraph {
  int device = 0;
  uint64_t n = 0, m = 0;
  uint64_t* indptr = nullptr;   // [n+1]
  uint32_t* indices = nullptr;  // [m]
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
  uint32_t* act_di = nullptr;       // dst index of each active dst (cap_dst)
  uint64_t* act_pre = nullptr;      // scan prefix of active dsts (cap_dst+1)
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
  unsigned* tickets = nullptr;                // [kMaxTickets]
  unsigned long long* status_a = nullptr;     // [max_tiles]
  unsigned long long* status_b = nullptr;     // [max_tiles]
  unsigned long long* status_c = nullptr;     // [max_tiles]
  unsigned* overflow = nullptr;               // [1]
  uint64_t max_tiles = 0;
  static constexpr int kMaxTickets = 256;
};

// Bitmap dedup structure over the vertex id space.
struct Bitmap {
  uint32_t* bits = nullptr;     // [words_padded]
  uint32_t* wprefix = nullptr;  // [words_padded] rank of first bit of word
  uint64_t words = 0, words_padded = 0;
};

// ----------------------------------------------------- kernel launchers ----
// sample.cu
void launch_batch_begin(const Sync& s, LayerMeta* meta, int num_layers, uint64_t n_seeds,
                        cudaStream_t st);
void launch_frontier(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, int kind,
                     uint32_t fanout, Bitmap& set_bm, const Bitmap* clear_bm,
                     const Sync& s, int ticket_base, int epoch_slot, cudaStream_t st);
void launch_labor(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, int kind,
                  uint32_t fanout, int layer, const cbdev::Variates* var, Bitmap& bm,
                  const Sync& s, int ticket, int epoch_slot, cudaStream_t st);
void launch_ns(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, uint32_t fanout,
               int layer, const cbdev::Variates* var, Bitmap& bm, cudaStream_t st);
void launch_extract(const Bitmap& bm, uint32_t* out, uint64_t cap_out,
                    unsigned long long* count_out, unsigned long long* count_out2,
                    const Sync& s, int ticket, int epoch_slot, cudaStream_t st);
constexpr int kExtractTileWords = 2048;
constexpr int kLaborTile = 1024;
constexpr int kFrontierTile = 1024;
void launch_relabel(const Bitmap& bm, const LayerBufs& b, const LayerMeta* meta,
                    cudaStream_t st);
void launch_clear(Bitmap& bm, const uint32_t* list, const unsigned long long* count,
                  cudaStream_t st);
void launch_rank(const Bitmap& bm, const uint32_t* ids, const unsigned long long* count,
                 uint32_t* rank_out, cudaStream_t st);

int grid_for(uint64_t work_items, int per_block, int max_per_sm);

}  // namespace cb
