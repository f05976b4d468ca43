// Feature-path launchers (gather.cu) and graph construction (graph.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cb_internal.h"

namespace cb {

void launch_gather(const void* table, int vec_bytes, uint64_t row_bytes, const uint32_t* ids,
                   const unsigned long long* count, uint64_t cap_rows, const uint32_t* row_map,
                   void* out, cudaStream_t st);
// the last layer's relabel (sample.cu relabel_kernel) fused with the gather
void launch_relabel_gather(const RelabelArgs& r, uint64_t relabel_work, const void* table,
                           int vec_bytes, uint64_t row_bytes, const uint32_t* ids,
                           const unsigned long long* count, uint64_t cap_rows,
                           const uint32_t* row_map, void* out, cudaStream_t st);
void launch_synth(uint64_t seed, uint32_t dim, int dtype, uint64_t n_rows,
                  const uint32_t* row_vertex, uint64_t v_base, void* out, cudaStream_t st);
int vec_bytes_for(uint64_t row_bytes);
// true iff every id's row lies in the shard [r0, r0 + rows) (synchronises st)
bool shard_holds(const uint32_t* ids, uint64_t n, const uint32_t* row_map, uint64_t r0,
                 uint64_t rows, unsigned* d_flag, cudaStream_t st);

// graph.cu
void graph_generate_rmat(DeviceGraph& g, uint64_t n, uint64_t m, uint64_t seed,
                         cudaStream_t st);
void graph_max_degree(DeviceGraph& g, cudaStream_t st);
uint64_t cross_edges(const DeviceGraph& g, const uint32_t* owner, cudaStream_t st);
void partition_random_device(uint64_t n, uint32_t parts, uint64_t seed, uint32_t* owner,
                             cudaStream_t st);

}  // namespace cb
