// Calibration of B200 latency primitives used to pick the sampling-kernel
// structure (not part of the product): kernel-to-kernel gap inside a CUDA
// graph, dependent global-load chains (L2-cold / warm), same-address atomics,
// and a software grid barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void empty_k() {}

__global__ void chain_k(const unsigned* __restrict__ next, int depth, unsigned* out) {
  unsigned i = blockIdx.x * 977u;
  for (int d = 0; d < depth; ++d) i = next[i];
  if (threadIdx.x == 0 && i == 0xffffffffu) *out = i;
}

__global__ void atomic_k(unsigned* ctr, int depth, unsigned* out) {
  unsigned acc = 0;
  if (threadIdx.x == 0)
    for (int d = 0; d < depth; ++d) acc += atomicAdd(ctr, 1u + acc % 2);
  if (threadIdx.x == 0 && acc == 0xffffffffu) *out = acc;
}

__device__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    const unsigned target = gen * nblocks;
    atomicAdd(bar, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}

__global__ void barrier_k(unsigned* bar, int n) {
  unsigned gen = 0;
  for (int i = 0; i < n; ++i) grid_barrier(bar, gridDim.x, gen);
}

int main() {
  const size_t N = 64u << 20;  // 256 MB index array (beyond L2)
  unsigned *next, *out, *ctr, *bar;
  CK(cudaMalloc(&next, N * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&ctr, 4));
  CK(cudaMalloc(&bar, 4));
  std::vector<unsigned> h(N);
  unsigned long long x = 88172645463325252ULL;
  for (size_t i = 0; i < N; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = static_cast<unsigned>(x % N);
  }
  CK(cudaMemcpy(next, h.data(), N * 4, cudaMemcpyHostToDevice));
  void* flush;
  CK(cudaMalloc(&flush, 512u << 20));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time_graph = [&](auto enqueue, int reps, bool cold) -> float {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    enqueue();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    float best = 1e9f;
    for (int r = 0; r < reps; ++r) {
      if (cold) cudaMemsetAsync(flush, r, 512u << 20, st);
      cudaEventRecord(a, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return best * 1000.f;
  };
  printf("empty kernel x20 in one graph:      %.2f us per kernel\n",
         time_graph([&] { for (int i = 0; i < 20; ++i) empty_k<<<1, 32, 0, st>>>(); }, 20, false) / 20);
  printf("empty kernel (1184 CTAs) x20:       %.2f us per kernel\n",
         time_graph([&] { for (int i = 0; i < 20; ++i) empty_k<<<1184, 256, 0, st>>>(); }, 20, false) / 20);
  for (int depth : {1, 4, 16}) {
    printf("dependent load chain depth %2d, cold: %.2f us (kernel)\n", depth,
           time_graph([&] { chain_k<<<1, 32, 0, st>>>(next, depth, out); }, 10, true));
    printf("dependent load chain depth %2d, warm: %.2f us (kernel)\n", depth,
           time_graph([&] { chain_k<<<1, 32, 0, st>>>(next, depth, out); }, 10, false));
  }
  printf("atomicAdd chain depth 16 (1 CTA):   %.2f us\n",
         time_graph([&] { atomic_k<<<1, 32, 0, st>>>(ctr, 16, out); }, 10, false));
  printf("atomicAdd once from 1184 CTAs:      %.2f us\n",
         time_graph([&] { atomic_k<<<1184, 32, 0, st>>>(ctr, 1, out); }, 10, false));
  CK(cudaMemset(bar, 0, 4));
  printf("grid barrier x16 (296 CTAs):        %.2f us per barrier\n",
         time_graph([&] { cudaMemsetAsync(bar, 0, 4, st); barrier_k<<<296, 256, 0, st>>>(bar, 16); }, 10, false) / 16);
  printf("grid barrier x16 (148 CTAs):        %.2f us per barrier\n",
         time_graph([&] { cudaMemsetAsync(bar, 0, 4, st); barrier_k<<<148, 256, 0, st>>>(bar, 16); }, 10, false) / 16);
  return 0;
}
