// Device primitives of the multi-process cooperative step (one rank = one
// part, ids and rows move between ranks with NCCL all-to-allv driven by the
// host; coop.cpp:25-64 build_exchange and coop.cpp:145-159
// all_to_all_forward split at the rank boundary):
//   bucket  : stable partition of a sorted id list by owner (each bucket stays
//             sorted), with the position map perm[k] = source index;
//   scatter : out[perm[k]] = in[k] for u32 values and for feature rows;
//   mark    : OR a received id list into a bitmap (owner-side dedup).
#include "cb_internal.h"
#include "dist.h"

namespace cb {
using namespace cbdev;

namespace {

constexpr int kBT = 256;

__global__ void bucket_count_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                    const uint32_t* __restrict__ owner, uint32_t P,
                                    uint32_t* tile_counts) {
  __shared__ uint32_t cnt[kDistMaxParts];
  for (uint32_t q = threadIdx.x; q < P; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBucketTile;
  for (uint32_t i = threadIdx.x; i < kBucketTile; i += blockDim.x) {
    const uint64_t k = t0 + i;
    if (k < n) atomicAdd(&cnt[owner[ids[k]]], 1u);
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < P; q += blockDim.x)
    tile_counts[static_cast<uint64_t>(blockIdx.x) * P + q] = cnt[q];
}

// tile_off[tile*P + q] = output index of the tile's first id owned by q.
__global__ void bucket_scatter_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                      const uint32_t* __restrict__ owner, uint32_t P,
                                      const uint64_t* __restrict__ tile_off, uint32_t* out,
                                      uint32_t* perm) {
  __shared__ uint64_t run[kDistMaxParts];
  __shared__ uint32_t wcnt[kBT / 32][kDistMaxParts];
  for (uint32_t q = threadIdx.x; q < P; q += blockDim.x)
    run[q] = tile_off[static_cast<uint64_t>(blockIdx.x) * P + q];
  const uint32_t w = threadIdx.x >> 5;
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kBucketTile;
  for (uint32_t c0 = 0; c0 < kBucketTile; c0 += kBT) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < (kBT / 32) * P; i += blockDim.x)
      wcnt[i / P][i % P] = 0;
    __syncthreads();
    const uint64_t k = t0 + c0 + threadIdx.x;
    const bool valid = k < n;
    const uint32_t v = valid ? ids[k] : 0u;
    const uint32_t q = valid ? owner[v] : 0xffffffffu;
    const unsigned same = __match_any_sync(0xffffffffu, q);
    const uint32_t rank = __popc(same & lanemask_lt());
    if (valid && rank == 0) wcnt[w][q] = __popc(same);
    __syncthreads();
    if (valid) {
      uint64_t before = run[q] + rank;
      for (uint32_t ww = 0; ww < w; ++ww) before += wcnt[ww][q];
      out[before] = v;
      perm[before] = static_cast<uint32_t>(k);
    }
    __syncthreads();
    for (uint32_t qq = threadIdx.x; qq < P; qq += blockDim.x) {
      uint64_t add = 0;
      for (uint32_t ww = 0; ww < kBT / 32; ++ww) add += wcnt[ww][qq];
      run[qq] += add;
    }
  }
}

__global__ void scatter_u32_kernel(const uint32_t* __restrict__ in,
                                   const uint32_t* __restrict__ perm, uint64_t n,
                                   uint32_t* out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += stride)
    out[perm[k]] = in[k];
}

template <typename V>
__global__ void scatter_rows_kernel(const V* __restrict__ in, const uint32_t* __restrict__ perm,
                                    uint64_t n, uint32_t vpr, V* out) {
  const uint64_t total = n * vpr;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += stride) {
    const uint64_t r = x / vpr, c = x - r * vpr;
    out[static_cast<uint64_t>(perm[r]) * vpr + c] = in[x];
  }
}

__global__ void mark_kernel(const uint32_t* __restrict__ ids, uint64_t n, uint32_t* bits,
                            uint32_t* summ) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += stride) {
    const uint32_t v = ids[k];
    atomicOr(&bits[v >> 5], 1u << (v & 31u));
    if (summ) atomicOr(&summ[v >> 10], 1u << ((v >> 5) & 31u));
  }
}

}  // namespace

void bucket_by_owner(const uint32_t* ids, uint64_t n, const uint32_t* owner, uint32_t P,
                     uint32_t* out, uint32_t* perm, uint64_t* counts_host,
                     cudaStream_t st) {
  require(P >= 1 && P <= kDistMaxParts, "bucket_by_owner: 1 <= parts <= 64");
  for (uint32_t q = 0; q < P; ++q) counts_host[q] = 0;
  if (n == 0) return;
  const uint64_t ntiles = (n + kBucketTile - 1) / kBucketTile;
  uint32_t* d_counts = nullptr;
  uint64_t* d_off = nullptr;
  CB_CUDA(cudaMallocAsync(&d_counts, ntiles * P * 4, st));
  CB_CUDA(cudaMallocAsync(&d_off, ntiles * P * 8, st));
  bucket_count_kernel<<<static_cast<unsigned>(ntiles), kBT, 0, st>>>(ids, n, owner, P,
                                                                     d_counts);
  CB_LAUNCH("bucket_count");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  std::vector<uint32_t> h(ntiles * P);
  CB_CUDA(cudaMemcpyAsync(h.data(), d_counts, ntiles * P * 4, cudaMemcpyDeviceToHost, st));
  CB_CUDA(cudaStreamSynchronize(st));
  // bucket-major offsets: bucket q starts after all ids of buckets < q
  std::vector<uint64_t> off(ntiles * P);
  for (uint32_t q = 0; q < P; ++q)
    for (uint64_t t = 0; t < ntiles; ++t) counts_host[q] += h[t * P + q];
  uint64_t base = 0;
  for (uint32_t q = 0; q < P; ++q) {
    uint64_t run = base;
    for (uint64_t t = 0; t < ntiles; ++t) {
      off[t * P + q] = run;
      run += h[t * P + q];
    }
    base = run;
  }
  CB_CUDA(cudaMemcpyAsync(d_off, off.data(), ntiles * P * 8, cudaMemcpyHostToDevice, st));
  bucket_scatter_kernel<<<static_cast<unsigned>(ntiles), kBT, 0, st>>>(ids, n, owner, P, d_off,
                                                                       out, perm);
  CB_LAUNCH("bucket_scatter");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  CB_CUDA(cudaFreeAsync(d_counts, st));
  CB_CUDA(cudaFreeAsync(d_off, st));
  CB_CUDA(cudaStreamSynchronize(st));
}

void scatter_u32(const uint32_t* in, const uint32_t* perm, uint64_t n, uint32_t* out,
                 cudaStream_t st) {
  if (!n) return;
  scatter_u32_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(in, perm, n, out);
  CB_LAUNCH("scatter_u32");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void scatter_rows(const void* in, const uint32_t* perm, uint64_t n, uint64_t row_bytes,
                  void* out, cudaStream_t st) {
  if (!n) return;
  int vb = 16;
  while (row_bytes % vb) vb >>= 1;
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vb);
  const int grid = grid_for(n * vpr, 256, 8);
  switch (vb) {
    case 16:
      scatter_rows_kernel<uint4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(in), perm, n,
                                                       vpr, static_cast<uint4*>(out));
      break;
    case 8:
      scatter_rows_kernel<uint2><<<grid, 256, 0, st>>>(static_cast<const uint2*>(in), perm, n,
                                                       vpr, static_cast<uint2*>(out));
      break;
    case 4:
      scatter_rows_kernel<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(in),
                                                          perm, n, vpr,
                                                          static_cast<uint32_t*>(out));
      break;
    default:
      scatter_rows_kernel<unsigned short><<<grid, 256, 0, st>>>(
          static_cast<const unsigned short*>(in), perm, n, vpr,
          static_cast<unsigned short*>(out));
  }
  CB_LAUNCH("scatter_rows");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void mark_ids(const uint32_t* ids, uint64_t n, uint32_t* bits, uint32_t* summ,
              cudaStream_t st) {
  if (!n) return;
  mark_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(ids, n, bits, summ);
  CB_LAUNCH("mark");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace cb
