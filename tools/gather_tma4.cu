// Row gather via the sm_100 TMA tile::gather4 mode vs the product's 16-byte
// vector gather (not part of the product). Shapes of the
// two headline feature tables: c4 (94.5K random rows x 256 B out of 111M fp16
// rows) and c2 (55K rows x 400 B out of 2.45M fp32 rows). L2 flushed before
// every launch, CUDA-event timed.
//   gather4: one elected lane per warp issues cp.async.bulk.tensor.2d
//   .tile::gather4 (4 table rows -> 4 consecutive rows in shared memory,
//   mbarrier completion), S stages per warp; the 4 rows leave either by one
//   bulk store (TMA, shared -> global) or by the warp's vector stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gt4 tools/gather_tma4.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e) {                                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                           \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// the product's gather (gather_body.cuh): flattened (row, vector) index, U loads in flight
template <int U>
__global__ void __launch_bounds__(256, 8) g_vec(const uint4* __restrict__ t,
                                                const unsigned* __restrict__ ids, unsigned n,
                                                unsigned vpr, unsigned magic, uint4* __restrict__ out) {
  const unsigned total = n * vpr, stride = gridDim.x * blockDim.x;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride * U) {
    unsigned r[U], c[U], v[U];
    uint4 b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned x = i + u * stride;
      unsigned q = __umulhi(x, magic);
      unsigned rem = x - q * vpr;
      if (rem >= vpr) { ++q; rem -= vpr; }
      r[u] = x < total ? q : 0u;
      c[u] = rem;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(ids + r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < total) b[u] = ldnc(t + 1ull * v[u] * vpr + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned x = i + u * stride;
      if (x < total) __stcs(out + x, b[u]);
    }
  }
}

constexpr int kWarps = 4;
template <int S, bool TMA_STORE>
__global__ void __launch_bounds__(kWarps * 32) g_tma4(const __grid_constant__ CUtensorMap tm,
                                                      const unsigned* __restrict__ ids,
                                                      unsigned n, unsigned row_bytes,
                                                      unsigned char* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarps][S];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned grp = 4 * row_bytes;               // bytes of one gather4
  const unsigned gstride = (grp + 127) & ~127u;     // TMA destinations are 128 B aligned
  unsigned char* ring = smem + w * S * gstride;
  const unsigned ngroups = (n + 3) / 4;
  const unsigned gw = blockIdx.x * kWarps + w, W = gridDim.x * kWarps;
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](unsigned g, int s) {
    if (lane == 0) {
      int r[4];
      for (int k = 0; k < 4; ++k) r[k] = 4 * g + k < n ? static_cast<int>(ids[4 * g + k]) : 0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[w][s])),
                   "r"(grp)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(ring + s * gstride)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(sa(&bar[w][s])), "r"(0), "r"(r[0]), "r"(r[1]),
          "r"(r[2]), "r"(r[3])
          : "memory");
    }
  };
  unsigned phase = 0;
  int s_issue = 0;
  unsigned next = gw;
  for (int q = 0; q < S && next < ngroups; ++q, next += W) {
    issue(next, s_issue);
    s_issue = (s_issue + 1) % S;
  }
  int s = 0;
  for (unsigned g = gw; g < ngroups; g += W) {
    for (unsigned spin = 0;; ++spin) {  // bounded: a bad tensor map must not hang the GPU
      uint32_t ok;
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(sa(&bar[w][s])), "r"((phase >> s) & 1u)
          : "memory");
      if (ok || spin > (1u << 22)) break;
    }
    phase ^= 1u << s;
    const unsigned rows = min(4u, n - 4 * g);
    unsigned char* dst = out + 4ull * g * row_bytes;
    if (TMA_STORE) {
      if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(sa(ring + s * gstride)), "r"(rows * row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(ring + s * gstride);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (unsigned v = lane; v < rows * row_bytes / 16; v += 32) __stcs(d4 + v, src[v]);
    }
    __syncwarp();
    if (next < ngroups) {
      issue(next, s);
      next += W;
    }
    s = (s + 1) % S;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int run_shape(const char* name, unsigned long long nrows, unsigned row_bytes, unsigned n) {
  printf("== %s: %u rows x %u B out of %llu\n", name, n, row_bytes, nrows);
  unsigned char *table, *out, *out2;
  unsigned* ids;
  CK(cudaMalloc(&table, nrows * row_bytes));
  CK(cudaMalloc(&out, 1ull * n * row_bytes + 4096));
  CK(cudaMalloc(&out2, 1ull * n * row_bytes + 4096));
  CK(cudaMalloc(&ids, n * 4ull));
  std::vector<unsigned> h(n);
  unsigned long long x = 12345;
  for (unsigned i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = static_cast<unsigned>(x % nrows);
  }
  std::sort(h.begin(), h.end());
  CK(cudaMemcpy(ids, h.data(), n * 4ull, cudaMemcpyHostToDevice));
  // row r = bytes (r * 7 + c) & 0xff: checkable
  {
    std::vector<unsigned char> row(row_bytes);
    CK(cudaMemset(table, 0, nrows * row_bytes));
    for (unsigned i = 0; i < n; i += 97) {
      for (unsigned c = 0; c < row_bytes; ++c) row[c] = static_cast<unsigned char>(h[i] * 7 + c);
      CK(cudaMemcpy(table + 1ull * h[i] * row_bytes, row.data(), row_bytes,
                    cudaMemcpyHostToDevice));
    }
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  const cuuint64_t dims[2] = {row_bytes / 2, nrows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {row_bytes / 2, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = reinterpret_cast<EncodeFn>(fn)(
      &tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, table, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed: %d\n", static_cast<int>(cr));
    return 1;
  }
  void* flush;
  CK(cudaMalloc(&flush, 512u << 20));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 2.0 * n * row_bytes + n * 4.0;
  auto run = [&](const char* nm, auto launch, unsigned char* o) {
    float sum = 0, best = 1e9f;
    for (int r = 0; r < 25; ++r) {
      cudaMemsetAsync(flush, r, 512u << 20, st);
      cudaEventRecord(a, st);
      launch();
      cudaEventRecord(b, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 5) { sum += ms; best = std::min(best, ms); }
    }
    cudaError_t e = cudaGetLastError();
    // check a few rows
    std::vector<unsigned char> got(row_bytes);
    int bad = 0;
    for (unsigned i = 0; i < n && !e; i += 97) {
      cudaMemcpy(got.data(), o + 1ull * i * row_bytes, row_bytes, cudaMemcpyDeviceToHost);
      for (unsigned c = 0; c < row_bytes; ++c)
        if (got[c] != static_cast<unsigned char>(h[i] * 7 + c)) { ++bad; break; }
    }
    printf("%-32s avg %7.2f us best %7.2f us %6.0f GB/s %s%s\n", nm, sum / 20 * 1e3, best * 1e3,
           bytes / (sum / 20 * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "",
           bad ? " WRONG ROWS" : " rows ok");
  };
  const unsigned vpr = row_bytes / 16;
  const unsigned magic = static_cast<unsigned>((1ull << 32) / vpr);
  run("vector gather U=3 (product)",
      [&] { g_vec<3><<<148 * 8, 256, 0, st>>>(reinterpret_cast<const uint4*>(table), ids, n, vpr,
                                              magic, reinterpret_cast<uint4*>(out)); }, out);
  auto tma = [&](const char* nm, auto kern, int S, int ctas) {
    const size_t sm = static_cast<size_t>(kWarps) * S * ((4 * row_bytes + 127) & ~127u);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    char buf[96];
    snprintf(buf, sizeof buf, "%s S=%d ctas/SM=%d", nm, S, ctas);
    cudaMemset(out2, 0, 1ull * n * row_bytes);
    run(buf, [&] { kern<<<148 * ctas, kWarps * 32, sm, st>>>(tm, ids, n, row_bytes, out2); }, out2);
  };
  tma("gather4 + bulk store", g_tma4<2, true>, 2, 8);
  tma("gather4 + bulk store", g_tma4<3, true>, 3, 8);
  tma("gather4 + bulk store", g_tma4<4, true>, 4, 8);
  tma("gather4 + bulk store", g_tma4<4, true>, 4, 12);
  tma("gather4 + bulk store", g_tma4<8, true>, 8, 4);
  tma("gather4 + warp stores", g_tma4<4, false>, 4, 8);
  tma("gather4 + warp stores", g_tma4<8, false>, 8, 6);
  tma("gather4 + warp stores", g_tma4<8, false>, 8, 4);
  cudaFree(table); cudaFree(out); cudaFree(out2); cudaFree(ids); cudaFree(flush);
  return 0;
}

int main() {
  if (run_shape("c4 (fp16 x 128)", 111059956ull, 256, 94500)) return 1;
  if (run_shape("c2 (fp32 x 100)", 2449029ull, 400, 54874)) return 1;
  return 0;
}
