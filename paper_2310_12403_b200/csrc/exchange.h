// Launchers for the on-device cooperative rendezvous (exchange.cu).
#pragma once

#include "cb_internal.h"

namespace cb {

constexpr int kMaxParts = 16;

// Per-part device pointers passed by value as kernel parameters.
struct PartPtrs {
  const uint32_t* src[kMaxParts];              // sender's sorted src list
  const unsigned long long* count[kMaxParts];  // its length (device)
  uint32_t* clear_bits[kMaxParts];             // sender's sampling bitmap
  uint32_t* clear_summ[kMaxParts];
  uint32_t* xbits[kMaxParts];                  // owner's exchange bitmap
  uint32_t* xsumm[kMaxParts];
  uint32_t* xprefix[kMaxParts];                // owner's exchange word ranks
  uint32_t* loc_part[kMaxParts];
  uint32_t* loc_row[kMaxParts];
};

// ---- multi-process peer exchange (one part per rank, CUDA IPC peer memory) ----
// Pointers into every rank's exchange region for one layer slot (entry q =
// rank q's bitmap, IPC-mapped; q == self is local memory).
struct PxPeers {
  uint32_t* bits[kMaxParts];
  uint32_t* summ[kMaxParts];  // nullptr: flat bitmaps
  const uint32_t* pre[kMaxParts];
};

// Cross-rank barrier in peer memory: flags[q] = rank q's arrival slots
// (IPC-mapped; entry r of rank q's array is written by rank r). The epoch is a
// device counter, so a captured graph replays it; ranks run the same number
// of barriers. A wait longer than timeout_ns sets *err and gives up (no hang).
constexpr int kBarRows = 64;  // flag rows per rank: row 0 epoch barrier, 1.. captured
struct PxBarrier {
  uint32_t* flags[kMaxParts];  // rank q's flag block [kBarRows][kMaxParts]
  uint32_t* ctr;
  uint32_t* err;
  uint32_t rank, world;
  unsigned long long timeout_ns;
};
void launch_px_barrier(const PxBarrier& b, cudaStream_t st);
// Arrival only: store `value` into row `row`, entry rank, of every peer's
// flag block (release, system scope). The waits are stream memory ops.
void launch_px_signal(const PxBarrier& b, uint32_t row, uint32_t value, cudaStream_t st);
// Loads the barrier kernels' module outside any stream capture (lazy loading).
void px_preload();

// Requester side of build_exchange (coop.cpp:35-51): OR every src id into its
// owner's exchange bitmap over peer memory; send_row[q] += ids sent to q.
void launch_px_route(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                     const uint32_t* owner, const PxPeers& peers, unsigned long long* send_row,
                     cudaStream_t st);
// src_location (coop.cpp:53-62): (owner, rank of v in the owner's sorted set)
// read from the owner's exchange bitmap and word ranks over peer memory.
void launch_px_locate(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                      const uint32_t* owner, const PxPeers& peers, uint32_t* loc_part,
                      uint32_t* loc_row, cudaStream_t st);
// all_to_all_forward (coop.cpp:145-159) as one-sided reads: row of input
// vertex v from its owner's shard, bases[q] = rank q's shard (virtual base
// indexed by the global shard-major row) -> out[j] requester-aligned.
void launch_px_gather(const unsigned char* const* d_bases, const uint32_t* owner,
                      const uint32_t* row_map, uint64_t row_bytes, const uint32_t* ids,
                      const unsigned long long* count, uint64_t cap, void* out,
                      cudaStream_t st);

// Capacity checks of a staged pull: *count (this pull) > cap or *count2 (the
// owner's staged rows) > cap2 sets *overflow (nullptr: no check).
struct PxCaps {
  const unsigned long long* count2 = nullptr;
  uint64_t cap2 = 0;
  unsigned* overflow = nullptr;
};
// all_to_all_forward from the owners' staged rows: out[j] = row loc_row[j] of
// rank loc_part[j]'s staging buffer (bases[q], IPC-mapped).
void launch_px_gather_staged(const unsigned char* const* d_bases, const uint32_t* loc_part,
                             const uint32_t* loc_row, uint64_t row_bytes,
                             const unsigned long long* count, uint64_t cap, void* out,
                             const PxCaps& caps, cudaStream_t st);

// Requester-side cache support: the requested rows owned by OTHER ranks,
// compacted (any order): ids[k], their positions pos[k] in the request list
// and the address of their row in the owner's staging buffer (miss_ptr[k]);
// *n_remote counts them. skip_rank >= 0 in the staged pull leaves those
// positions alone (they come from the requester cache instead).
void launch_px_split_remote(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                            const uint32_t* loc_part, const uint32_t* loc_row, uint32_t rank,
                            const unsigned char* const* d_bases, uint64_t row_bytes,
                            uint32_t* ids, uint32_t* pos, const void** miss_ptr,
                            unsigned long long* n_remote, cudaStream_t st);
void launch_px_scatter_rows(const void* rows, const uint32_t* pos, uint64_t n, uint64_t row_bytes,
                            void* out, cudaStream_t st);
void launch_px_gather_staged_local(const unsigned char* const* d_bases, const uint32_t* loc_part,
                                   const uint32_t* loc_row, uint64_t row_bytes,
                                   const unsigned long long* count, uint64_t cap, void* out,
                                   uint32_t rank, const PxCaps& caps, cudaStream_t st);

void launch_route(const PartPtrs& pp, const uint32_t* owner, uint32_t P,
                  unsigned long long* send_counts, uint64_t max_src, cudaStream_t st);
void launch_locate(const PartPtrs& pp, const uint32_t* owner, uint32_t P, uint64_t max_src,
                   cudaStream_t st);

}  // namespace cb
