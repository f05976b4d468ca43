// Launchers of the multi-process cooperative primitives (dist.cu).
#pragma once

#include "cb_internal.h"

namespace cb {

constexpr uint32_t kDistMaxParts = 64;
constexpr uint32_t kBucketTile = 4096;

// Stable partition of `ids` (n) by owner[id]: out is bucket-major, each
// bucket in input order; perm[k] = input index of out[k]; counts_host[q] =
// bucket sizes. Synchronises the stream (the counts feed the host-side
// all-to-allv split sizes).
void bucket_by_owner(const uint32_t* ids, uint64_t n, const uint32_t* owner, uint32_t P,
                     uint32_t* out, uint32_t* perm, uint64_t* counts_host, cudaStream_t st);
void scatter_u32(const uint32_t* in, const uint32_t* perm, uint64_t n, uint32_t* out,
                 cudaStream_t st);
void scatter_rows(const void* in, const uint32_t* perm, uint64_t n, uint64_t row_bytes,
                  void* out, cudaStream_t st);
void mark_ids(const uint32_t* ids, uint64_t n, uint32_t* bits, uint32_t* summ,
              cudaStream_t st);

}  // namespace cb
