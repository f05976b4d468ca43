// Input-feature path: synthetic row-sharded embedding tables
// (FeatureStore::synth, coop.cpp:359-376) and the row gather of the final
// layer's vertices (FeatureStore::load_rows, coop.cpp:378-388), fused with the
// requester-side placement of all_to_all_forward (coop.cpp:145-159) when the
// owner table is reachable from the gathering device.
//
// The gather is HBM-bound: per row, row_bytes read at a random 16 B-aligned
// address and row_bytes written sequentially. Loads use the non-coherent,
// L1-no-allocate path, stores are streaming (evict-first) so the output does
// not displace the graph/bitmaps in L2; 4 independent 16 B loads in flight
// per thread.
#include <cuda_fp16.h>

#include <algorithm>

#include "cb_internal.h"
#include "gather.h"
#include "gather_body.cuh"
#include "relabel.cuh"

namespace cb {
using namespace cbdev;

namespace {

// 8 CTAs of 256 per SM (32 registers). 16-byte rows keep 3 vectors in
// flight per thread: UNROLL 4 spilled 56 B to the stack under the 32-register
// bound (gather 14.8 -> 14.0 us at c2, 14.7 -> 13.6 us at c4; tools/ab.sh).
constexpr int kGatherCtasPerSM = 8;
#ifndef CB_GATHER_GRID_PER_SM
#define CB_GATHER_GRID_PER_SM 8
#endif
constexpr int kGatherGridPerSM = CB_GATHER_GRID_PER_SM;  // CTAs launched per SM
#ifndef CB_FUSED_GRID_PER_SM
#define CB_FUSED_GRID_PER_SM 4
#endif
// relabel + gather launch of the in-flight graph: half the gather's CTAs, so
// it leaves SM room to the other batches (63.1 -> 61.8 us/step; the
// standalone roofline gather keeps 8 per SM)
constexpr int kFusedGridPerSM = CB_FUSED_GRID_PER_SM;
template <typename V>
constexpr int gather_unroll() { return sizeof(V) == 16 ? 3 : 4; }

template <typename V, int UNROLL>
__global__ void __launch_bounds__(256, kGatherCtasPerSM) gather_kernel(
    const V* __restrict__ table, const uint32_t* __restrict__ ids,
    const unsigned long long* __restrict__ count, uint64_t cap_rows,
    const uint32_t* __restrict__ row_map, uint32_t vpr, V* __restrict__ out) {
  pdl_begin();
  gbody::gather_body<V, UNROLL>(table, ids, count, cap_rows, row_map, vpr, out, blockIdx.x,
                                gridDim.x);
}

// The last layer's relabel and the feature gather in one launch (they are
// independent: the gather reads the src list, the relabel rewrites edges and
// dst_pos): CTAs [0, n_rel) relabel, the rest gather. Used by the captured
// sample + gather graph, one launch fewer per batch.
template <typename V, int UNROLL>
__global__ void __launch_bounds__(256, kGatherCtasPerSM) relabel_gather_kernel(
    RelabelArgs r, unsigned n_rel, const V* __restrict__ table,
    const uint32_t* __restrict__ ids, const unsigned long long* __restrict__ count,
    uint64_t cap_rows, const uint32_t* __restrict__ row_map, uint32_t vpr, V* __restrict__ out) {
  pdl_begin();
  if (blockIdx.x < n_rel) {
    rbody::relabel_range(r, blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
                         static_cast<uint64_t>(n_rel) * blockDim.x);
    return;
  }
  gbody::gather_body<V, UNROLL>(table, ids, count, cap_rows, row_map, vpr, out,
                                blockIdx.x - n_rel, gridDim.x - n_rel);
}

// value[v, j] = 2*U(hash(seed,{9,v,j})) - 1 (exact in f64), one rounding to
// the table dtype (cvt.rn.f32.f64 / cvt.rn.f16.f64).
__global__ void synth_kernel(uint64_t seed, uint32_t dim, int dtype, uint64_t n_rows,
                             const uint32_t* __restrict__ row_vertex, uint64_t v_base,
                             void* out) {
  const uint64_t pfx = hstep(hinit(seed), 9ULL);
  const uint64_t total = n_rows * dim;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += stride) {
    const uint64_t r = x / dim;
    const uint32_t j = static_cast<uint32_t>(x - r * dim);
    const uint64_t v = row_vertex ? row_vertex[r] : v_base + r;
    const double val = __dsub_rn(__dmul_rn(2.0, ufb(hstep(hstep(pfx, v), j))), 1.0);
    if (dtype == 0) static_cast<double*>(out)[x] = val;
    else if (dtype == 1) static_cast<float*>(out)[x] = __double2float_rn(val);
    else static_cast<__half*>(out)[x] = __double2half(val);
  }
}

}  // namespace

void launch_gather(const void* table, int vec_bytes, uint64_t row_bytes, const uint32_t* ids,
                   const unsigned long long* count, uint64_t cap_rows, const uint32_t* row_map,
                   void* out, cudaStream_t st) {
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vec_bytes);
  const int grid = kNumSMs * kGatherGridPerSM;
  switch (vec_bytes) {
    case 16:
      launch_k(gather_kernel<uint4, gather_unroll<uint4>()>, grid, 256, st, static_cast<const uint4*>(table), ids,
                                                   count, cap_rows, row_map, vpr,
                                                   static_cast<uint4*>(out));
      break;
    case 8:
      launch_k(gather_kernel<uint2, gather_unroll<uint2>()>, grid, 256, st, static_cast<const uint2*>(table), ids,
                                                   count, cap_rows, row_map, vpr,
                                                   static_cast<uint2*>(out));
      break;
    case 4:
      launch_k(gather_kernel<uint32_t, gather_unroll<uint32_t>()>, grid, 256, st, static_cast<const uint32_t*>(table),
                                                       ids, count, cap_rows, row_map, vpr,
                                                       static_cast<uint32_t*>(out));
      break;
    default:
      launch_k(gather_kernel<unsigned short, gather_unroll<unsigned short>()>, grid, 256, st, 
          static_cast<const unsigned short*>(table), ids, count, cap_rows, row_map, vpr,
          static_cast<unsigned short*>(out));
  }
  CB_LAUNCH("gather");
}

namespace {
__global__ void shard_check_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                   const uint32_t* __restrict__ row_map, uint64_t r0,
                                   uint64_t rows, unsigned* bad) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (static_cast<uint64_t>(row_map[ids[i]]) - r0 >= rows) atomicOr(bad, 1u);
}
}  // namespace

bool shard_holds(const uint32_t* ids, uint64_t n, const uint32_t* row_map, uint64_t r0,
                 uint64_t rows, unsigned* d_flag, cudaStream_t st) {
  CB_CUDA(cudaMemsetAsync(d_flag, 0, 4, st));
  if (n) {
    launch_k(shard_check_kernel, kNumSMs * 4, 256, st, ids, n, row_map, r0, rows, d_flag);
    CB_LAUNCH("shard_check");
  }
  unsigned h = 0;
  CB_CUDA(cudaMemcpyAsync(&h, d_flag, 4, cudaMemcpyDeviceToHost, st));
  CB_CUDA(cudaStreamSynchronize(st));
  return h == 0;
}

void launch_relabel_gather(const RelabelArgs& r, uint64_t relabel_work, const void* table,
                           int vec_bytes, uint64_t row_bytes, const uint32_t* ids,
                           const unsigned long long* count, uint64_t cap_rows,
                           const uint32_t* row_map, void* out, cudaStream_t st) {
  const uint32_t vpr = static_cast<uint32_t>(row_bytes / vec_bytes);
  // up to 2 relabel CTAs per SM, the gather takes the rest of the grid
  const unsigned n_rel = static_cast<unsigned>(
      std::min<uint64_t>(std::max<uint64_t>((relabel_work + 1023) / 1024, 1), kNumSMs * 2));
  const int grid = kNumSMs * kFusedGridPerSM;
  switch (vec_bytes) {
    case 16:
      launch_k(relabel_gather_kernel<uint4, gather_unroll<uint4>()>, grid, 256, st, r, n_rel,
               static_cast<const uint4*>(table), ids, count, cap_rows, row_map, vpr,
               static_cast<uint4*>(out));
      break;
    case 8:
      launch_k(relabel_gather_kernel<uint2, gather_unroll<uint2>()>, grid, 256, st, r, n_rel,
               static_cast<const uint2*>(table), ids, count, cap_rows, row_map, vpr,
               static_cast<uint2*>(out));
      break;
    case 4:
      launch_k(relabel_gather_kernel<uint32_t, gather_unroll<uint32_t>()>, grid, 256, st, r,
               n_rel, static_cast<const uint32_t*>(table), ids, count, cap_rows, row_map, vpr,
               static_cast<uint32_t*>(out));
      break;
    default:
      launch_k(relabel_gather_kernel<unsigned short, gather_unroll<unsigned short>()>, grid, 256,
               st, r, n_rel, static_cast<const unsigned short*>(table), ids, count, cap_rows,
               row_map, vpr, static_cast<unsigned short*>(out));
  }
  CB_LAUNCH("relabel_gather");
}

void launch_synth(uint64_t seed, uint32_t dim, int dtype, uint64_t n_rows,
                  const uint32_t* row_vertex, uint64_t v_base, void* out, cudaStream_t st) {
  synth_kernel<<<kNumSMs * 16, 256, 0, st>>>(seed, dim, dtype, n_rows, row_vertex, v_base, out);
  CB_LAUNCH("synth");
}

int vec_bytes_for(uint64_t row_bytes) {
  for (int v : {16, 8, 4, 2})
    if (row_bytes % v == 0) return v;
  return 2;
}

}  // namespace cb
