// Row gather body of the gather kernel (gather.cu): out[j] = table[row(ids[j])], flattened
// (row, vector) index space, 16/8/4/2-byte vectors, non-coherent
// L1-no-allocate loads, streaming stores, UNROLL loads in flight per thread.
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace cb {
namespace gbody {

template <typename V>
__device__ __forceinline__ V ld_stream(const V* p);
template <>
__device__ __forceinline__ uint4 ld_stream<uint4>(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint2 ld_stream<uint2>(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ld_stream<uint32_t>(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ld_stream<unsigned short>(const unsigned short* p) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

template <typename V>
__device__ __forceinline__ void st_stream(V* p, V v) {
  __stcs(p, v);
}
template <>
__device__ __forceinline__ void st_stream<unsigned short>(unsigned short* p, unsigned short v) {
  asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v));
}

// out[j] = table[row(ids[j])], j < count. Flattened (row, vector) index space
// so every lane moves a full vector even when row_bytes/16 is not a multiple
// of 32. row(v) = row_map ? row_map[v] : v. Index math is 32-bit whenever the
// flattened space fits (division by vpr = multiply-high + correction), and
// each thread issues all its id loads before any table load so the UNROLL
// table reads are in flight together.
template <typename V, int UNROLL>
__device__ __forceinline__ void gather_body(const V* __restrict__ table,
                                            const uint32_t* __restrict__ ids,
                                            const unsigned long long* __restrict__ count,
                                            uint64_t cap_rows, const uint32_t* __restrict__ row_map,
                                            uint32_t vpr, V* __restrict__ out, unsigned role,
                                            unsigned ncta) {
  const uint64_t stride = static_cast<uint64_t>(ncta) * blockDim.x;
  if (cap_rows * vpr + stride * UNROLL < (1ULL << 32)) {
    // the row count (written by the previous kernel) is loaded together with
    // the first ids, which are read speculatively within the capacity
    const unsigned long long cnt = count ? __ldg(count) : cap_rows;
    const uint32_t s32 = static_cast<uint32_t>(stride);
    const uint32_t magic = 0xffffffffu / vpr;
    const uint32_t last = static_cast<uint32_t>(cap_rows ? cap_rows - 1 : 0);
    uint32_t tot32 = 0xffffffffu;
    for (uint32_t idx = role * blockDim.x + threadIdx.x;; idx += s32 * UNROLL) {
      uint32_t r[UNROLL], c[UNROLL];
      V buf[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint32_t x = idx + u * s32;
        uint32_t q = __umulhi(x, magic);
        uint32_t rem = x - q * vpr;
        while (rem >= vpr) {
          ++q;
          rem -= vpr;
        }
        r[u] = min(q, last);
        c[u] = rem;
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) r[u] = __ldg(ids + r[u]);
      if (tot32 == 0xffffffffu)
        tot32 = static_cast<uint32_t>(min(static_cast<uint64_t>(cnt), cap_rows) * vpr);
      if (idx >= tot32) break;
      if (row_map) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          if (idx + u * s32 < tot32) r[u] = __ldg(row_map + r[u]);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (idx + u * s32 < tot32)
          buf[u] = ld_stream(table + static_cast<uint64_t>(r[u]) * vpr + c[u]);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint32_t x = idx + u * s32;
        if (x < tot32) st_stream(out + x, buf[u]);
      }
    }
    return;
  }
  const uint64_t n = count ? min(static_cast<uint64_t>(*count), cap_rows) : cap_rows;
  const uint64_t total = n * vpr;
  uint64_t idx = role * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (; idx < total; idx += stride * UNROLL) {
    V buf[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t x = idx + u * stride;
      if (x < total) {
        const uint64_t r = x / vpr;
        const uint64_t c = x - r * vpr;
        const uint32_t v = __ldg(ids + r);
        const uint64_t row = row_map ? __ldg(row_map + v) : v;
        buf[u] = ld_stream(table + row * vpr + c);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t x = idx + u * stride;
      if (x < total) st_stream(out + x, buf[u]);
    }
  }
}


}  // namespace gbody
}  // namespace cb
