// Cooperative rendezvous between the parts that live on one device
// (build_exchange, coop.cpp:25-64): route every sampled source id to its
// owner, deduplicate at the owner into the next layer's sorted seed list, and
// record send_counts[p][q] and src_location[p][j] = (q, rank at owner).
//
// route  : (blockIdx.y = sender p) id v -> owner q; OR v into q's exchange
//          bitmap; per-block owner histogram -> send_counts[p][*]; clears
//          p's sampling bitmap word (its relabel is done).
// extract: (sample.cu) owner bitmap -> sorted owner set = next dst list.
// locate : (blockIdx.y = p) loc_part[j] = q, loc_row[j] = rank of v at q.
#include "cb_internal.h"
#include "exchange.h"

namespace cb {
using namespace cbdev;

namespace {

__global__ void route_kernel(PartPtrs pp, const uint32_t* __restrict__ owner, uint32_t P,
                             unsigned long long* send_counts) {
  pdl_begin();
  __shared__ unsigned long long hist[kMaxParts];
  const uint32_t p = blockIdx.y;
  for (uint32_t q = threadIdx.x; q < P; q += blockDim.x) hist[q] = 0;
  __syncthreads();
  const uint64_t n = *pp.count[p];
  const uint32_t* src = pp.src[p];
  uint32_t* clear = pp.clear_bits[p];
  uint32_t* clear_s = pp.clear_summ[p];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += stride) {
    const uint32_t v = src[j];
    const uint32_t q = owner[v];
    atomicOr(&pp.xbits[q][v >> 5], 1u << (v & 31u));
    if (pp.xsumm[q]) atomicOr(&pp.xsumm[q][v >> 10], 1u << ((v >> 5) & 31u));
    atomicAdd(&hist[q], 1ULL);
    if (clear) {
      clear[v >> 5] = 0u;
      if (clear_s) clear_s[v >> 10] = 0u;
    }
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < P; q += blockDim.x)
    if (hist[q]) atomicAdd(&send_counts[p * P + q], hist[q]);
}

__global__ void locate_kernel(PartPtrs pp, const uint32_t* __restrict__ owner) {
  pdl_begin();
  const uint32_t p = blockIdx.y;
  const uint64_t n = *pp.count[p];
  const uint32_t* src = pp.src[p];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += stride) {
    const uint32_t v = src[j];
    const uint32_t q = owner[v];
    const uint32_t w = v >> 5;
    pp.loc_part[p][j] = q;
    pp.loc_row[p][j] = pp.xprefix[q][w] + __popc(pp.xbits[q][w] & ((1u << (v & 31u)) - 1u));
  }
}

}  // namespace

void launch_route(const PartPtrs& pp, const uint32_t* owner, uint32_t P,
                  unsigned long long* send_counts, uint64_t max_src, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(grid_for(max_src, 256, 8) / P + 1), P);
  launch_k(route_kernel, grid, 256, st, pp, owner, P, send_counts);
  CB_LAUNCH("route");
}

void launch_locate(const PartPtrs& pp, const uint32_t* owner, uint32_t P, uint64_t max_src,
                   cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(grid_for(max_src, 256, 8) / P + 1), P);
  launch_k(locate_kernel, grid, 256, st, pp, owner);
  CB_LAUNCH("locate");
}

}  // namespace cb
