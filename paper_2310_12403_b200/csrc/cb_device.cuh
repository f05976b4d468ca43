// Device-side building blocks shared by every kernel of the coopbatch B200
// path: the reference's counter-based hash (rng.hpp:17-48), its FP64 normal
// CDF / quantile (rng.cpp:7-52), warp/block scans, and a decoupled look-back
// tile prefix so every compaction in the path is single-pass and keeps the
// reference's element order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cbdev {

constexpr uint64_t kSalt = 0x736f6d6570736575ULL;  // rng.hpp:24
constexpr uint64_t kKappaInf = ~0ULL;               // rng.hpp:70-71
constexpr int kNumSMs = 148;

// rng.hpp:17-22 — SplitMix64 finalizer. Integer-only: bit-identical on device.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// 64-bit x * C (mod 2^64) as one 32x32->64 multiply plus two multiply-adds
// into the high word (the compiler's form needs a fourth add).
__device__ __forceinline__ uint64_t mul64c(uint64_t x, uint64_t c) {
  const uint32_t xl = static_cast<uint32_t>(x), xh = static_cast<uint32_t>(x >> 32);
  const uint32_t cl = static_cast<uint32_t>(c), ch = static_cast<uint32_t>(c >> 32);
  uint32_t lo, hi;
  asm("{\n\t.reg .u32 ph;\n\t"
      "mul.lo.u32 %0, %2, %4;\n\t"
      "mul.hi.u32 ph, %2, %4;\n\t"
      "mad.lo.u32 ph, %3, %4, ph;\n\t"
      "mad.lo.u32 %1, %2, %5, ph;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(xl), "r"(xh), "r"(cl), "r"(ch));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}
// mix64 on the device with the cheaper multiplies (bit-identical)
__device__ __forceinline__ uint64_t mix64_dev(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = mul64c(x ^ (x >> 30), 0xbf58476d1ce4e5b9ULL);
  x = mul64c(x ^ (x >> 27), 0x94d049bb133111ebULL);
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t hinit(uint64_t seed) { return mix64(seed ^ kSalt); }
__host__ __device__ __forceinline__ uint64_t hstep(uint64_t h, uint64_t id) { return mix64(h ^ id); }
// rng.hpp:42-44; (bits>>11) < 2^53 converts exactly, the 2^-53 scale is exact.
__host__ __device__ __forceinline__ double ufb(uint64_t bits) {
  return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

// ---- FP64 phi / inverse_phi (rng.cpp:7-52) ---------------------------------
// Same constants and evaluation order as the reference; explicit _rn
// intrinsics keep nvcc from contracting into FMA (the reference's x86-64
// build has no FMA). libdevice erfc/log/log1p/exp may differ from glibc by
// an ulp; labor/ns kernels count decisions within kGuard of the threshold
// ("uncertified") and report them (DESIGN.md §Smoothed variates).
__device__ __forceinline__ double dphi(double x) {
  return __dmul_rn(0.5, erfc(__dmul_rn(-x, 0.7071067811865475244)));
}

__device__ __forceinline__ double horner6(const double* c, double q) {
  double v = c[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) v = __dadd_rn(__dmul_rn(v, q), c[i]);
  return v;
}

__device__ inline double dinverse_phi(double p) {
  const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                      -2.759285104469687e+02, 1.383577518672690e+02,
                      -3.066479806614716e+01, 2.506628277459239e+00};
  const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                      -1.556989798598866e+02, 6.680131188771972e+01,
                      -1.328068155288572e+01, 1.0};
  const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                      -2.400758277161838e+00, -2.549732539343734e+00,
                      4.374664141464968e+00,  2.938163982698783e+00};
  const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                      2.445134137142996e+00, 3.754408661907416e+00, 1.0};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = sqrt(__dmul_rn(-2.0, log(p)));
    double den = d[0];
#pragma unroll
    for (int i = 1; i < 5; ++i) den = __dadd_rn(__dmul_rn(den, q), d[i]);
    x = __ddiv_rn(horner6(c, q), den);
  } else if (p <= __dsub_rn(1.0, plow)) {
    const double q = __dsub_rn(p, 0.5);
    const double r = __dmul_rn(q, q);
    const double num = __dmul_rn(horner6(a, r), q);
    double den = b[0];
#pragma unroll
    for (int i = 1; i < 6; ++i) den = __dadd_rn(__dmul_rn(den, r), b[i]);
    x = __ddiv_rn(num, den);
  } else {
    const double q = sqrt(__dmul_rn(-2.0, log1p(-p)));
    double den = d[0];
#pragma unroll
    for (int i = 1; i < 5; ++i) den = __dadd_rn(__dmul_rn(den, q), d[i]);
    x = __ddiv_rn(-horner6(c, q), den);
  }
  const double e = __dsub_rn(dphi(x), p);
  const double u = __dmul_rn(__dmul_rn(e, sqrt(__dmul_rn(2.0, 3.14159265358979323846))),
                             exp(__dmul_rn(__dmul_rn(0.5, x), x)));
  x = __dsub_rn(x, __ddiv_rn(u, __dadd_rn(1.0, __dmul_rn(__dmul_rn(0.5, x), u))));
  return x;
}

// rng.hpp:54-56
__device__ __forceinline__ double dnormal_from_bits(uint64_t bits) {
  return dinverse_phi(__dmul_rn(__dadd_rn(static_cast<double>(bits >> 11), 0.5), 0x1.0p-53));
}

// Smoothed decisions inside the guard band, resolved on the host with the
// reference's own arithmetic (glibc erfc/log/exp, no FMA; host_variates in
// capi.cu). Keys: LABOR (kResolveLabor | part << 48 | layer << 32 | t, 0),
// NS (part << 48 | layer << 32 | s, i); `val` is the host's exact variate,
// sorted by key.
// Decisions not in the table are appended to `pend` for the host.
constexpr uint64_t kResolveLabor = 1ULL << 63;
struct ResolvePend {
  uint64_t k1, k2;
  double dev;  // the value the device decided with
  double aux;  // LABOR: the threshold k/d; NS: the device's r = floor(u * (i + 1))
};
struct Resolve {
  const uint64_t* k1;
  const uint64_t* k2;
  const double* val;
  uint32_t n;
  uint32_t cap_pend;
  ResolvePend* pend;
  unsigned long long* n_pend;
  int perturb;  // test hook: flip every unresolved in-band device decision
  int pad;
};

// Per-batch variate parameters (samplers.hpp:53-126 VariateSource), resident
// in device memory so a captured batch replays with new keys.
struct Variates {
  uint64_t z1, z2;
  double cos_c, sin_c;
  int smoothed;
  int part;            // index of the part these variates belong to
  double guard;        // relative guard band of smoothed decisions
  const Resolve* rs;   // host-resolved decisions (nullptr: count only)
};

__device__ inline bool resolve_lookup(const Resolve* rs, uint64_t k1, uint64_t k2, double& out) {
  if (rs == nullptr) return false;
  uint32_t lo = 0, hi = rs->n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t a = rs->k1[mid], b = rs->k2[mid];
    if (a < k1 || (a == k1 && b < k2)) lo = mid + 1;
    else hi = mid;
  }
  if (lo < rs->n && rs->k1[lo] == k1 && rs->k2[lo] == k2) {
    out = rs->val[lo];
    return true;
  }
  return false;
}

__device__ inline void resolve_record(const Resolve* rs, uint64_t k1, uint64_t k2, double dev,
                                      double aux) {
  if (rs == nullptr) return;
  const unsigned long long i = atomicAdd(rs->n_pend, 1ULL);
  if (i < rs->cap_pend) rs->pend[i] = ResolvePend{k1, k2, dev, aux};
}

// samplers.hpp:96-100 finish() for the smoothed stream. Out of line: it is
// FP64-transcendental heavy and only runs for 2 <= kappa < inf.
static __device__ __noinline__ double smooth_finish(const Variates& v, uint64_t b1, uint64_t b2) {
  const double n = __dadd_rn(__dmul_rn(v.cos_c, dnormal_from_bits(b1)),
                             __dmul_rn(v.sin_c, dnormal_from_bits(b2)));
  return dphi(n);
}

// Default guard band for smoothed decisions (relative); see DESIGN.md.
constexpr double kGuard = 1e-12;

// ---- memory-order helpers ---------------------------------------------------
// Look-back status words carry their own payload (the aggregate / prefix), and
// consumers read nothing else a producer wrote, so relaxed gpu-scope
// accesses suffice: no fence waits on the producer's outstanding bitmap REDs.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The publish is an atomic exchange, not a relaxed store: a st.relaxed.gpu
// could sit in the SM's store path for several microseconds (measured: the
// extract look-back of a 152-tile layer waited 5-8 us for its predecessor's
// flag), while the atomic is performed at L2 immediately.
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  atomicExch(p, v);
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialisation may start while its predecessor drains; it waits here for the
// predecessor's completion (and memory) before touching its outputs. No
// explicit launch_dependents: a CTA's exit counts as its trigger, so the
// successor's CTAs are scheduled as this grid's last CTAs retire instead of
// occupying SM slots for its whole run. No-ops for ordinary launches.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef CB_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace[63*8 + 7] = the latest end of any CTA of the kernel (thread 0 of each)
__device__ __forceinline__ void tlast(unsigned long long* trace) {
  if (trace && threadIdx.x == 0) atomicMax(trace + 63 * 8 + 7, gtimer());
}
// trace[cta*8 + k] = time stamp k of this CTA (first writer per slot wins)
__device__ __forceinline__ void tstamp(unsigned long long* trace, unsigned cta, int k) {
  if (trace && cta < 64 && threadIdx.x == 0) trace[cta * 8 + k] = gtimer();
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- warp / block scans -----------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= static_cast<unsigned>(o)) v += n;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive block scan; `total` receives the block sum. `smem` needs
// NWARPS+1 entries. Ends with a __syncthreads-free read of smem, so callers
// must __syncthreads() before reusing smem.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T& total) {
  constexpr int NW = NT / 32;
  const unsigned w = threadIdx.x >> 5;
  const T inc = warp_inclusive_scan(v);
  if (lane_id() == 31) smem[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = (lane_id() < static_cast<unsigned>(NW)) ? smem[lane_id()] : T(0);
    const T si = warp_inclusive_scan(s);
    if (lane_id() < static_cast<unsigned>(NW)) smem[lane_id()] = si - s;
    if (lane_id() == NW - 1) smem[NW] = si;
  }
  __syncthreads();
  total = smem[NW];
  return smem[w] + inc - v;
}

// ---- decoupled look-back tile prefix ----------------------------------------
// Status word: [epoch:24 | flag:2 | value:38]. Epoch-tagging means status
// arrays never need clearing between batches: batch_begin bumps the epoch.
constexpr int kValBits = 38;
constexpr unsigned long long kValMask = (1ULL << kValBits) - 1;
constexpr unsigned long long kFlagAgg = 1ULL << kValBits;
constexpr unsigned long long kFlagPre = 2ULL << kValBits;
constexpr int kEpochShift = kValBits + 2;

__device__ __forceinline__ unsigned long long mkstat(unsigned epoch, unsigned long long flag,
                                                     unsigned long long val) {
  return (static_cast<unsigned long long>(epoch & 0xffffffu) << kEpochShift) | flag |
         (val & kValMask);
}

// All threads of the block call this with the same `agg`; returns the
// exclusive prefix of the tile in tile order. Warp 0 looks back over W*32
// predecessors per step (lane l reads tiles base - l*W - j), so the
// inclusive-prefix front advances W*32 tiles per L2 round trip.
// tile_prefix_async: the same look-back run by warp `warp` only, result in
// *s_bcast, no barrier (several independent scans of one tile can look back
// concurrently in different warps; the caller syncs once).
template <int W = 4>
__device__ inline void tile_prefix_async(unsigned long long* status, unsigned tile,
                                         unsigned long long agg, unsigned epoch,
                                         unsigned long long* s_bcast, unsigned warp) {
  if ((threadIdx.x >> 5) == warp) {
    const unsigned long long want = static_cast<unsigned long long>(epoch & 0xffffffu);
    if (tile == 0) {
      if (lane_id() == 0) {
        st_release(&status[0], mkstat(epoch, kFlagPre, agg));
        *s_bcast = 0;
      }
    } else {
      if (lane_id() == 0) st_release(&status[tile], mkstat(epoch, kFlagAgg, agg));
      unsigned long long excl = 0;
      long long base = static_cast<long long>(tile) - 1;
      const int me = static_cast<int>(lane_id());
      while (true) {
        unsigned long long s[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const long long idx = base - static_cast<long long>(me) * W - j;
          s[j] = (idx < 0) ? mkstat(epoch, kFlagPre, 0) : ld_acquire(&status[idx]);
        }
        int first;      // lane holding the nearest inclusive prefix (32 = none)
        int fj = W;     // its entry
        while (true) {
          unsigned inval = 0;
          fj = W;
#pragma unroll
          for (int j = W - 1; j >= 0; --j) {
            const bool ok = (s[j] >> kEpochShift) == want && ((s[j] >> kValBits) & 3u) != 0;
            if (!ok) inval |= 1u << j;
            else if (((s[j] >> kValBits) & 3u) == 2u) fj = j;
          }
          // an entry only matters if it is nearer than the nearest prefix
          const unsigned pmask = __ballot_sync(0xffffffffu, fj < W);
          first = pmask ? (__ffs(pmask) - 1) : 32;
          unsigned need = 0;
          if (me < first) need = inval;
          else if (me == first) need = inval & ((1u << fj) - 1u);
          if (!__any_sync(0xffffffffu, need != 0)) break;
          // no sleep: the re-poll is itself an L2 round trip
#pragma unroll
          for (int j = 0; j < W; ++j)
            if ((need >> j) & 1u) {
              const long long idx = base - static_cast<long long>(me) * W - j;
              s[j] = ld_acquire(&status[idx]);
            }
        }
        unsigned long long c = 0;
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (me < first || (me == first && j <= fj)) c += s[j] & kValMask;
        excl += warp_sum(c);
        if (first < 32) break;
        base -= 32 * W;
      }
      if (lane_id() == 0) {
        st_release(&status[tile], mkstat(epoch, kFlagPre, excl + agg));
        *s_bcast = excl;
      }
    }
  }
}

template <int W = 4>
__device__ inline unsigned long long tile_prefix(unsigned long long* status, unsigned tile,
                                                 unsigned long long agg, unsigned epoch,
                                                 unsigned long long* s_bcast) {
  tile_prefix_async<W>(status, tile, agg, epoch, s_bcast, 0);
  __syncthreads();
  return *s_bcast;
}

// Tile cursor for ordered (look-back) kernels: the first tile of each CTA is
// its role index (the first wave is co-resident: grids are capped at the
// kernel's resident capacity, as in CUB's blockIdx-ordered scans); later
// tiles come from a ticket counter offset by the CTA count, so a CTA waits
// only on tiles held by running CTAs. No atomic at all when one wave covers
// every tile.
__device__ __forceinline__ unsigned next_tile_after(unsigned* ticket, unsigned* s_tile,
                                                    unsigned ncta, unsigned long long ntiles) {
  if (ncta >= ntiles) return 0xffffffffu;
  __syncthreads();
  if (threadIdx.x == 0) *s_tile = atomicAdd(ticket, 1u) + ncta;
  __syncthreads();
  return *s_tile;
}

// Ticket in ticket order (deadlock-free look-back with persistent CTAs).
__device__ __forceinline__ unsigned next_tile(unsigned* ticket, unsigned* s_tile) {
  __syncthreads();
  if (threadIdx.x == 0) *s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  return *s_tile;
}

// Upper-bound search: largest i in [lo, hi) with a[i] <= x (a nondecreasing).
template <typename T>
__device__ __forceinline__ int seg_search(const T* a, int lo, int hi, T x) {
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

}  // namespace cbdev
