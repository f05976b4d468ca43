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

// ---- peer exchange kernels ----
__global__ void px_route_kernel(const uint32_t* __restrict__ src,
                                const unsigned long long* __restrict__ count, uint64_t cap,
                                const uint32_t* __restrict__ owner, PxPeers peers,
                                unsigned long long* send_row) {
  pdl_begin();
  __shared__ unsigned long long hist[kMaxParts];
  for (uint32_t q = threadIdx.x; q < kMaxParts; q += blockDim.x) hist[q] = 0;
  __syncthreads();
  const uint64_t n = min(static_cast<uint64_t>(*count), cap);
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = src[j];
    const uint32_t q = owner[v];
    atomicOr(&peers.bits[q][v >> 5], 1u << (v & 31u));
    if (peers.summ[q]) atomicOr(&peers.summ[q][v >> 10], 1u << ((v >> 5) & 31u));
    atomicAdd(&hist[q], 1ULL);
  }
  // the owner reads these bits after a cross-rank barrier: one system-scope
  // fence per CTA, cumulative over the CTA's REDs ordered before it by the
  // barrier (a fence per thread cost ~20 us per launch at c4)
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  for (uint32_t q = threadIdx.x; q < kMaxParts; q += blockDim.x)
    if (hist[q]) atomicAdd(&send_row[q], hist[q]);
}

__global__ void px_locate_kernel(const uint32_t* __restrict__ src,
                                 const unsigned long long* __restrict__ count, uint64_t cap,
                                 const uint32_t* __restrict__ owner, PxPeers peers,
                                 uint32_t* loc_part, uint32_t* loc_row) {
  pdl_begin();
  const uint64_t n = min(static_cast<uint64_t>(*count), cap);
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = src[j];
    const uint32_t q = owner[v];
    const uint32_t w = v >> 5;
    loc_part[j] = q;
    loc_row[j] = peers.pre[q][w] + __popc(peers.bits[q][w] & ((1u << (v & 31u)) - 1u));
  }
}

// One warp: publish this rank's arrival to every peer (release at system
// scope, after the layer's peer-memory writes of the preceding kernels), then
// lane q waits for rank q's arrival in the local flag array (acquire).
__global__ void px_barrier_kernel(PxBarrier b) {
  const uint32_t lane = threadIdx.x;
  uint32_t e = 0;
  if (lane == 0) {
    e = *b.ctr + 1;
    *b.ctr = e;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (lane < b.world)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(b.flags[lane] + b.rank), "r"(e)
                 : "memory");
  if (lane < b.world) {
    const uint32_t* f = b.flags[b.rank] + lane;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (static_cast<int32_t>(v - e) >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > b.timeout_ns) {
        atomicExch(b.err, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

template <typename V>
__global__ void px_gather_staged_kernel(const unsigned char* const* __restrict__ bases,
                                        const uint32_t* __restrict__ loc_part,
                                        const uint32_t* __restrict__ loc_row, uint32_t vpr,
                                        uint64_t row_bytes,
                                        const unsigned long long* __restrict__ count,
                                        uint64_t cap, V* __restrict__ out, uint32_t only_rank,
                                        const unsigned long long* __restrict__ count2,
                                        uint64_t cap2, unsigned* overflow) {
  pdl_begin();
  // rows beyond a capped buffer (this pull's, or the owner's staging count2)
  // are never silently dropped: the step is flagged
  if (overflow && blockIdx.x == 0 && threadIdx.x == 0 &&
      (*count > cap || (count2 && *count2 > cap2)))
    atomicExch(overflow, 1u);
  const uint64_t n = min(static_cast<uint64_t>(*count), cap);
  const uint64_t total = n * vpr;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  constexpr int U = 4;
  for (uint64_t x0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x0 < total;
       x0 += stride * U) {
    V buf[U];
    const V* srcp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t x = x0 + u * stride;
      srcp[u] = nullptr;
      if (x < total) {
        const uint64_t r = x / vpr, c = x - r * vpr;
        const uint32_t q = __ldg(loc_part + r);
        if (only_rank == ~0u || q == only_rank)
          srcp[u] = reinterpret_cast<const V*>(bases[q] +
                                               static_cast<uint64_t>(__ldg(loc_row + r)) *
                                                   row_bytes) + c;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (srcp[u]) buf[u] = *srcp[u];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (srcp[u]) __stcs(out + x0 + u * stride, buf[u]);
  }
}

__global__ void px_signal_kernel(PxBarrier b, uint32_t row, uint32_t value) {
  pdl_begin();
  const uint32_t q = threadIdx.x;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (q < b.world && q != b.rank)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(b.flags[q] + row * kMaxParts +
                                                           b.rank),
                 "r"(value)
                 : "memory");
}

template <typename V>
__global__ void px_gather_kernel(const unsigned char* const* __restrict__ bases,
                                 const uint32_t* __restrict__ owner,
                                 const uint32_t* __restrict__ row_map, uint32_t vpr,
                                 uint64_t row_bytes, const uint32_t* __restrict__ ids,
                                 const unsigned long long* __restrict__ count, uint64_t cap,
                                 V* __restrict__ out) {
  pdl_begin();
  const uint64_t n = min(static_cast<uint64_t>(*count), cap);
  const uint64_t total = n * vpr;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  constexpr int U = 4;
  for (uint64_t x0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x0 < total;
       x0 += stride * U) {
    V buf[U];
    const V* srcp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t x = x0 + u * stride;
      srcp[u] = nullptr;
      if (x < total) {
        const uint64_t r = x / vpr, c = x - r * vpr;
        const uint32_t v = __ldg(ids + r);
        srcp[u] = reinterpret_cast<const V*>(bases[__ldg(owner + v)] +
                                             static_cast<uint64_t>(__ldg(row_map + v)) *
                                                 row_bytes) + c;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (srcp[u]) buf[u] = *srcp[u];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (srcp[u]) __stcs(out + x0 + u * stride, buf[u]);
  }
}

}  // namespace

void launch_px_route(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                     const uint32_t* owner, const PxPeers& peers, unsigned long long* send_row,
                     cudaStream_t st) {
  launch_k(px_route_kernel, grid_for(cap, 256, 8), 256, st, src, count, cap, owner, peers,
           send_row);
  CB_LAUNCH("px_route");
}

void launch_px_locate(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                      const uint32_t* owner, const PxPeers& peers, uint32_t* loc_part,
                      uint32_t* loc_row, cudaStream_t st) {
  launch_k(px_locate_kernel, grid_for(cap, 256, 8), 256, st, src, count, cap, owner, peers,
           loc_part, loc_row);
  CB_LAUNCH("px_locate");
}

void launch_px_barrier(const PxBarrier& b, cudaStream_t st) {
  launch_k(px_barrier_kernel, 1, 32, st, b);
  CB_LAUNCH("px_barrier");
}

void launch_px_signal(const PxBarrier& b, uint32_t row, uint32_t value, cudaStream_t st) {
  launch_k(px_signal_kernel, 1, 32, st, b, row, value);
  CB_LAUNCH("px_signal");
}

void px_preload() {
  cudaFuncAttributes fa;
  cuda_check(cudaFuncGetAttributes(&fa, px_signal_kernel), "cudaFuncGetAttributes");
  cuda_check(cudaFuncGetAttributes(&fa, px_barrier_kernel), "cudaFuncGetAttributes");
}

void launch_px_gather(const unsigned char* const* d_bases, const uint32_t* owner,
                      const uint32_t* row_map, uint64_t row_bytes, const uint32_t* ids,
                      const unsigned long long* count, uint64_t cap, void* out,
                      cudaStream_t st) {
  int vb = 16;
  while (row_bytes % vb) vb >>= 1;
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vb);
  const unsigned grid = kNumSMs * 8;
  switch (vb) {
    case 16:
      launch_k(px_gather_kernel<uint4>, grid, 256, st, d_bases, owner, row_map, vpr, row_bytes,
               ids, count, cap, static_cast<uint4*>(out));
      break;
    case 8:
      launch_k(px_gather_kernel<uint2>, grid, 256, st, d_bases, owner, row_map, vpr, row_bytes,
               ids, count, cap, static_cast<uint2*>(out));
      break;
    case 4:
      launch_k(px_gather_kernel<uint32_t>, grid, 256, st, d_bases, owner, row_map, vpr,
               row_bytes, ids, count, cap, static_cast<uint32_t*>(out));
      break;
    default:
      launch_k(px_gather_kernel<unsigned short>, grid, 256, st, d_bases, owner, row_map, vpr,
               row_bytes, ids, count, cap, static_cast<unsigned short*>(out));
  }
  CB_LAUNCH("px_gather");
}

namespace {
void staged(const unsigned char* const* d_bases, const uint32_t* loc_part, const uint32_t* loc_row,
            uint64_t row_bytes, const unsigned long long* count, uint64_t cap, void* out,
            uint32_t only_rank, const PxCaps& caps, cudaStream_t st) {
  int vb = 16;
  while (row_bytes % vb) vb >>= 1;
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vb);
  const unsigned grid = kNumSMs * 8;
  switch (vb) {
    case 16:
      launch_k(px_gather_staged_kernel<uint4>, grid, 256, st, d_bases, loc_part, loc_row, vpr,
               row_bytes, count, cap, static_cast<uint4*>(out), only_rank, caps.count2, caps.cap2, caps.overflow);
      break;
    case 8:
      launch_k(px_gather_staged_kernel<uint2>, grid, 256, st, d_bases, loc_part, loc_row, vpr,
               row_bytes, count, cap, static_cast<uint2*>(out), only_rank, caps.count2, caps.cap2, caps.overflow);
      break;
    case 4:
      launch_k(px_gather_staged_kernel<uint32_t>, grid, 256, st, d_bases, loc_part, loc_row,
               vpr, row_bytes, count, cap, static_cast<uint32_t*>(out), only_rank, caps.count2, caps.cap2, caps.overflow);
      break;
    default:
      launch_k(px_gather_staged_kernel<unsigned short>, grid, 256, st, d_bases, loc_part,
               loc_row, vpr, row_bytes, count, cap, static_cast<unsigned short*>(out),
               only_rank, caps.count2, caps.cap2, caps.overflow);
  }
  CB_LAUNCH("px_gather_staged");
}

__global__ void px_split_remote_kernel(const uint32_t* __restrict__ src,
                                       const unsigned long long* __restrict__ count, uint64_t cap,
                                       const uint32_t* __restrict__ loc_part,
                                       const uint32_t* __restrict__ loc_row, uint32_t rank,
                                       const unsigned char* const* __restrict__ bases,
                                       uint64_t row_bytes, uint32_t* ids, uint32_t* pos,
                                       const void** miss_ptr, unsigned long long* n_remote) {
  pdl_begin();
  const uint64_t n = min(static_cast<uint64_t>(*count), cap);
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t q = loc_part[j];
    const bool remote = q != rank;
    const unsigned m = __ballot_sync(__activemask(), remote);
    if (!m) continue;
    unsigned long long base = 0;
    const unsigned leader = __ffs(m) - 1;
    if (lane_id() == leader) base = atomicAdd(n_remote, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(__activemask(), base, leader);
    if (remote) {
      const uint64_t k = base + __popc(m & ((1u << lane_id()) - 1u));
      ids[k] = src[j];
      pos[k] = static_cast<uint32_t>(j);
      miss_ptr[k] = bases[q] + static_cast<uint64_t>(loc_row[j]) * row_bytes;
    }
  }
}

template <typename V>
__global__ void px_scatter_rows_kernel(const V* __restrict__ rows, const uint32_t* __restrict__ pos,
                                       uint64_t n, uint32_t vpr, V* __restrict__ out) {
  pdl_begin();
  const uint64_t total = n * vpr;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = x / vpr, c = x - k * vpr;
    out[static_cast<uint64_t>(pos[k]) * vpr + c] = rows[x];
  }
}
}  // namespace

void launch_px_gather_staged(const unsigned char* const* d_bases, const uint32_t* loc_part,
                             const uint32_t* loc_row, uint64_t row_bytes,
                             const unsigned long long* count, uint64_t cap, void* out,
                             const PxCaps& caps, cudaStream_t st) {
  staged(d_bases, loc_part, loc_row, row_bytes, count, cap, out, ~0u, caps, st);
}

void launch_px_gather_staged_local(const unsigned char* const* d_bases, const uint32_t* loc_part,
                                   const uint32_t* loc_row, uint64_t row_bytes,
                                   const unsigned long long* count, uint64_t cap, void* out,
                                   uint32_t rank, const PxCaps& caps, cudaStream_t st) {
  staged(d_bases, loc_part, loc_row, row_bytes, count, cap, out, rank, caps, st);
}

void launch_px_split_remote(const uint32_t* src, const unsigned long long* count, uint64_t cap,
                            const uint32_t* loc_part, const uint32_t* loc_row, uint32_t rank,
                            const unsigned char* const* d_bases, uint64_t row_bytes,
                            uint32_t* ids, uint32_t* pos, const void** miss_ptr,
                            unsigned long long* n_remote, cudaStream_t st) {
  cuda_check(cudaMemsetAsync(n_remote, 0, 8, st), "cudaMemsetAsync");
  launch_k(px_split_remote_kernel, grid_for(cap, 256, 8), 256, st, src, count, cap, loc_part,
           loc_row, rank, d_bases, row_bytes, ids, pos, miss_ptr, n_remote);
  CB_LAUNCH("px_split_remote");
}

void launch_px_scatter_rows(const void* rows, const uint32_t* pos, uint64_t n, uint64_t row_bytes,
                            void* out, cudaStream_t st) {
  if (n == 0) return;
  int vb = 16;
  while (row_bytes % vb) vb >>= 1;
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vb);
  const unsigned grid = grid_for(n * vpr, 256, 8);
  switch (vb) {
    case 16:
      launch_k(px_scatter_rows_kernel<uint4>, grid, 256, st, static_cast<const uint4*>(rows), pos,
               n, vpr, static_cast<uint4*>(out));
      break;
    case 8:
      launch_k(px_scatter_rows_kernel<uint2>, grid, 256, st, static_cast<const uint2*>(rows), pos,
               n, vpr, static_cast<uint2*>(out));
      break;
    case 4:
      launch_k(px_scatter_rows_kernel<uint32_t>, grid, 256, st,
               static_cast<const uint32_t*>(rows), pos, n, vpr, static_cast<uint32_t*>(out));
      break;
    default:
      launch_k(px_scatter_rows_kernel<unsigned short>, grid, 256, st,
               static_cast<const unsigned short*>(rows), pos, n, vpr,
               static_cast<unsigned short*>(out));
  }
  CB_LAUNCH("px_scatter_rows");
}

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
