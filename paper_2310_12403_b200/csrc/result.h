// Batch result -> pinned host memory in one kernel (result.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cb_internal.h"

namespace cb {

constexpr int kResultMaxLayers = 8;

struct ResultArgs {
  const LayerMeta* meta;  // this part's layers (meta[l])
  int L;
  const void* ptr[kResultMaxLayers][4];  // dst, src, edges, dst_pos per layer
  const void* rows;       // gathered rows or nullptr
  uint64_t row_bytes;
  unsigned char* out;     // device-visible pointer of the pinned host buffer
  uint64_t cap;
};

void launch_result(const ResultArgs& a, cudaStream_t st);

}  // namespace cb
