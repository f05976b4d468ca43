// Device temporaries and small kernels shared by the training step
// (capi_train.cu) and the host-buffer ops of the C++ drop-in (capi_ops.cu).
#pragma once

#include "capi_internal.h"

namespace cb_train_util {

struct TmpArena {
  std::vector<void*> ptrs;
  template <typename T>
  T* get(uint64_t n) {
    void* p = nullptr;
    CB_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T) + 16));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~TmpArena() {
    for (void* p : ptrs) cudaFree(p);
  }
};

struct U32ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// out[0..n] = exclusive prefix of the u32 counts (out[n] = total)
inline void scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* out, TmpArena& A, cudaStream_t st) {
  auto it = thrust::make_transform_iterator(cnt, U32ToU64{});
  size_t bytes = 0;
  CB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, static_cast<int64_t>(n + 1), st));
  void* tmp = A.get<unsigned char>(bytes);
  CB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, it, out, static_cast<int64_t>(n + 1), st));
}

static __global__ void src_hist_kernel(const uint2* __restrict__ edges, uint64_t n, uint32_t* cnt,
                                uint32_t* key, uint32_t* val) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&cnt[edges[e].x], 1u);
    key[e] = edges[e].x;
    val[e] = static_cast<uint32_t>(e);
  }
}

static __global__ void owner_key_kernel(const uint32_t* __restrict__ part, const uint32_t* __restrict__ row,
                                 uint64_t n, const uint64_t* __restrict__ owner_base,
                                 uint64_t g0, uint32_t* cnt, uint64_t* key, uint64_t* val) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = owner_base[part[j]] + row[j];
    atomicAdd(&cnt[k], 1u);
    key[g0 + j] = k;
    val[g0 + j] = g0 + j;
  }
}

inline int grid_of_n(uint64_t n) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)));
}

}  // namespace cb_train_util
