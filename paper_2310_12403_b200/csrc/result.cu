// Batch result straight into pinned host memory: every layer's block (dst,
// src, edges, dst_pos — the reference's BipartiteBlock fields, samplers.hpp:
// 30-38) and the gathered input rows (load_rows / all_to_all_forward output,
// coop.cpp:145-159, 378-388), written by one kernel over PCIe. The kernel
// reads the batch's counts from device memory, so no host round trip sizes
// the copies (a cudaMemcpyAsync would need them on the host first).
//
// Layout (little-endian), every section 16-byte aligned:
//   u64 header[5 + 3L] = {magic 'CBRS1', L, row_bytes, total_bytes, truncated,
//                          (n_dst, n_src, n_edges) per layer}
//   per layer: u32 dst[n_dst], u32 src[n_src], u32x2 edges[n_edges],
//              u32 dst_pos[n_dst]
//   rows[n_src(L-1) * row_bytes] (when the batch has gathered rows)
// When total_bytes exceeds the buffer only the header is written, with
// truncated = 1 and total_bytes = the size needed.
#include "result.h"

#include "cb_device.cuh"

namespace cb {
namespace {

constexpr uint64_t kMagic = 0x3153524243ULL;  // "CBRS1"

__device__ __forceinline__ uint64_t pad16(uint64_t b) { return (b + 15) & ~15ULL; }

struct Seg {
  const unsigned char* src;
  uint64_t bytes, off;
};

__device__ void segments(const ResultArgs& a, Seg* seg, int& ns, uint64_t& total) {
  uint64_t off = pad16(8ULL * (5 + 3 * a.L));
  ns = 0;
  for (int l = 0; l < a.L; ++l) {
    const LayerMeta& m = a.meta[l];
    const uint64_t b[4] = {m.n_dst * 4, m.n_src * 4, m.n_edges * 8, m.n_dst * 4};
    for (int f = 0; f < 4; ++f) {
      seg[ns++] = {static_cast<const unsigned char*>(a.ptr[l][f]), b[f], off};
      off += pad16(b[f]);
    }
  }
  if (a.rows) {
    const uint64_t b = a.meta[a.L - 1].n_src * a.row_bytes;
    seg[ns++] = {static_cast<const unsigned char*>(a.rows), b, off};
    off += pad16(b);
  }
  total = off;
}

__global__ void __launch_bounds__(256) result_kernel(ResultArgs a) {
  cbdev::pdl_begin();
  Seg seg[4 * kResultMaxLayers + 1];
  int ns;
  uint64_t total;
  segments(a, seg, ns, total);
  const bool fits = total <= a.cap;
  if (blockIdx.x == 0 && threadIdx.x < 5 + 3 * a.L) {
    const uint32_t i = threadIdx.x;
    uint64_t v;
    if (i == 0) v = kMagic;
    else if (i == 1) v = a.L;
    else if (i == 2) v = a.rows ? a.row_bytes : 0;
    else if (i == 3) v = total;
    else if (i == 4) v = fits ? 0 : 1;
    else {
      const LayerMeta& m = a.meta[(i - 5) / 3];
      const uint32_t f = (i - 5) % 3;
      v = f == 0 ? m.n_dst : (f == 1 ? m.n_src : m.n_edges);
    }
    reinterpret_cast<volatile uint64_t*>(a.out)[i] = v;
  }
  if (!fits) return;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (int s = 0; s < ns; ++s) {
    const unsigned char* src = seg[s].src;
    unsigned char* dst = a.out + seg[s].off;
    const uint64_t bytes = seg[s].bytes;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const uint64_t nv = bytes / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (uint64_t u = tid; u < nv; u += nth) d4[u] = __ldg(s4 + u);
      for (uint64_t b = nv * 16 + tid; b < bytes; b += nth) dst[b] = src[b];
    } else {  // 4-byte aligned id lists (a part's seeds inside the seed buffer)
      const uint64_t nw = bytes / 4;
      const uint32_t* s1 = reinterpret_cast<const uint32_t*>(src);
      uint32_t* d1 = reinterpret_cast<uint32_t*>(dst);
      for (uint64_t u = tid; u < nw; u += nth) d1[u] = __ldg(s1 + u);
      for (uint64_t b = nw * 4 + tid; b < bytes; b += nth) dst[b] = src[b];
    }
  }
}

}  // namespace

void launch_result(const ResultArgs& a, cudaStream_t st) {
  launch_k(result_kernel, cbdev::kNumSMs * 2, 256, st, a);
  CB_LAUNCH("result");
}

}  // namespace cb
