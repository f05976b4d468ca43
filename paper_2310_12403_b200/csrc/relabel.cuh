// Relabel of a sampled block (BlockBuilder::finish, samplers.cpp:17-60): edge
// src ids -> their rank in the layer's sorted unique src list, and
// dst_pos_in_src, both by a popcount over the dedup bitmap. Shared by the
// relabel kernel (sample.cu) and the fused relabel + gather launch (gather.cu).
#pragma once

#include <cstdint>

#include "cb_internal.h"

namespace cb {
namespace rbody {

__device__ __forceinline__ uint32_t bm_rank(const uint32_t* bits, const uint32_t* wprefix,
                                            uint32_t v) {
  const uint32_t w = v >> 5;
  return wprefix[w] + __popc(bits[w] & ((1u << (v & 31u)) - 1u));
}

__device__ __forceinline__ void relabel_range(const RelabelArgs& r, uint64_t tid,
                                              uint64_t stride) {
  const uint64_t ne = min(static_cast<uint64_t>(r.meta->n_edges), r.cap_edges);
  const uint64_t nd = r.meta->n_dst;
  for (uint64_t e = tid; e < ne; e += stride) {
    uint2 x = r.edges[e];
    x.x = bm_rank(r.bits, r.wprefix, x.x);
    r.edges[e] = x;
  }
  for (uint64_t i = tid; i < nd; i += stride) r.dst_pos[i] = bm_rank(r.bits, r.wprefix, r.D[i]);
}

}  // namespace rbody
}  // namespace cb
