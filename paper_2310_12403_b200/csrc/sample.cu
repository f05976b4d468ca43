// Frontier expansion kernels: one layer of LABOR-0 / NS / FULL sampling
// (samplers.cpp:62-136, 289-296) plus the bitmap dedup/relabel that replaces
// BlockBuilder::finish (samplers.cpp:28-54).
//
// Per layer (indep / P = 1 order):
//   frontier(l) : [relabel of layer l-1 fused in] degree scan of D_l with
//                 three look-back scans -> packed records of the active dsts
//                 (ActRec: scan prefix, row base, threshold / NS hash prefix),
//                 a scan-tile -> first-record map, NS output prefix and slot
//                 init; marks D_l in the layer bitmap
//   labor(l)    : scan-space tiles over every neighbour position; keep rule;
//                 order-preserving compaction (ballot + decoupled look-back),
//                 so edges land grouped by dst, CSR order inside a dst — the
//                 reference order; kept ids OR-ed into the bitmap
//   ns(l)       : reservoir via per-slot atomicMax, then slot-order emission
//   extract(l)  : bitmap popcount scan -> sorted unique src list + word ranks;
//                 zeroes the other (previous-layer) bitmap on the way
//   relabel     : edge (t, di) -> (rank(t), di); dst_pos = rank(D) (fused into
//                 the next frontier; standalone only after the last layer)
// No host synchronisation: all counts live in device LayerMeta; every kernel
// is a persistent ticketed loop bounded by those counts.
#include <mutex>
#include <unordered_map>

#include "cb_internal.h"
#include "gather_body.cuh"
#include "relabel.cuh"

namespace cb {
using namespace cbdev;

namespace {

constexpr int kNT = 256;
constexpr uint32_t kTileExact = 0x80000000u;
// labor_mark residency: 8 CTAs/SM at 64 registers and ~21 KB of shared
// memory each (one TMA id stage per warp, 128 staged records): one CTA's
// staging barrier overlaps another's hashing, and the small footprint leaves
// room for the other in-flight batches' kernels. A/B on one box (c4, 8
// batches in flight): 4 CTAs x 3 stages 161.6 us/step, 6 x 2 146-149,
// 8 x 1 134; the mark alone 103.6 / 93-97 / 91 us.
#ifndef CB_MARK_CTAS
#define CB_MARK_CTAS 8
#endif
constexpr int kMarkCtasPerSM = CB_MARK_CTAS;
#ifndef CB_MARK_MINB
#define CB_MARK_MINB CB_MARK_CTAS
#endif
constexpr int kMarkMinBlocks = CB_MARK_MINB;  // register bound: 64K / (128 * this)

__device__ __forceinline__ unsigned inv_epoch(const unsigned* ep, int slot) {
  return ((*ep & 0x3ffffu) << 6) | static_cast<unsigned>(slot);
}

// summ == nullptr for bitmaps small enough to be extracted flat; otherwise
// the summary bit of the word is OR-ed too (both fire-and-forget REDs).
__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t* summ, uint32_t v) {
  atomicOr(&bits[v >> 5], 1u << (v & 31u));
  if (summ) atomicOr(&summ[v >> 10], 1u << ((v >> 5) & 31u));
}

using rbody::bm_rank;

// Tickets are zeroed by batch_begin_kernel at the start of every batch /
// per-layer op (stream order), so kernels need no exit bookkeeping.

using rbody::relabel_range;

// ------------------------------------------------------------ batch begin --
// Clears the previous batch's last bitmap (its final id list), bumps the
// look-back epoch, resets the overflow flag. One launch per batch.
__device__ __forceinline__ void batch_begin_body(unsigned* epoch, unsigned* overflow,
                                                 unsigned* tickets, int n_tickets,
                                                 uint32_t* clear_bits, uint32_t* clear_summ,
                                                 const uint32_t* __restrict__ clear_list,
                                                 const unsigned long long* clear_count,
                                                 uint64_t cap, uint64_t nwords, unsigned role,
                                                 unsigned ncta) {
  if (role == 0) {
    if (threadIdx.x == 0) {
      *epoch = *epoch + 1;
      *overflow = 0;
    }
    for (int i = threadIdx.x; i < n_tickets; i += blockDim.x) tickets[i] = 0u;
  }
  if (!clear_bits) return;
  const uint64_t n = min(static_cast<uint64_t>(*clear_count), cap);
  const uint64_t stride = static_cast<uint64_t>(ncta) * blockDim.x;
  for (uint64_t i = role * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const uint32_t w = clear_list[i] >> 5;
    if (w < nwords) {
      clear_bits[w] = 0u;
      if (clear_summ) clear_summ[w >> 5] = 0u;
    }
  }
}

__global__ void batch_begin_kernel(unsigned* epoch, unsigned* overflow, unsigned* tickets,
                                   int n_tickets, uint32_t* clear_bits, uint32_t* clear_summ,
                                   const uint32_t* __restrict__ clear_list,
                                   const unsigned long long* clear_count, uint64_t cap,
                                   uint64_t nwords) {
  pdl_begin();
  batch_begin_body(epoch, overflow, tickets, n_tickets, clear_bits, clear_summ, clear_list,
                   clear_count, cap, nwords, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------- frontier --
// kind: 0 FULL, 1 NS, 2 LABOR0 (samplers.hpp:15). Per dst: scan work q
// (LABOR/FULL: d; NS: reservoir positions max(d-k,0)), active flag q>0 and,
// for NS, the output count min(d,k).
template <int IPT>
__device__ __forceinline__ void frontier_body(const FrontierArgs& a, const RelabelArgs& r,
                                              unsigned role, unsigned ncta) {
  __shared__ unsigned long long s_scan[3][kNT / 32 + 1];
  __shared__ unsigned long long s_bc[3];
  __shared__ unsigned s_tile;
  tstamp(a.trace, role, 0);
  if (r.edges) {  // relabel of the previous layer (independent work)
    relabel_range(r, role * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
                  static_cast<uint64_t>(ncta) * blockDim.x);
  }
  tstamp(a.trace, role, 1);
  LayerMeta* meta = a.meta;
  if (a.n_dst_param != ~0ULL && role == 0 && threadIdx.x == 0)
    meta->n_dst = a.n_dst_param;
  const uint64_t n = (a.n_dst_param != ~0ULL) ? a.n_dst_param : meta->n_dst;
  constexpr int TILE = kNT * IPT;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const bool is_ns = (a.kind == 1);
  const bool full = (a.kind == 0);
  const Variates v = *a.var;
  const bool smooth = v.smoothed != 0;
  const uint64_t z1p = hstep(hstep(hinit(v.z1), 1ULL), static_cast<uint64_t>(a.layer));
  const uint32_t k = a.k;
  for (unsigned tile = role; tile < ntiles;
       tile = next_tile_after(a.ticket, &s_tile, ncta, ntiles)) {
    const uint64_t i0 = static_cast<uint64_t>(tile) * TILE + threadIdx.x * IPT;
    unsigned long long q[IPT], o[IPT];
    uint32_t vv[IPT];
    uint64_t rs[IPT], re[IPT];
    unsigned long long qs = 0, as = 0, os = 0;
    // batched loads: all ids, then all indptr pairs, then the bitmap REDs (the
    // atomics may alias, so interleaving them would serialise the loads)
#pragma unroll
    for (int j = 0; j < IPT; ++j) vv[j] = (i0 + j < n) ? __ldg(a.D + i0 + j) : 0u;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      rs[j] = (i0 + j < n) ? __ldg(a.indptr + vv[j]) : 0;
      re[j] = (i0 + j < n) ? __ldg(a.indptr + vv[j] + 1) : 0;
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t i = i0 + j;
      q[j] = o[j] = 0;
      if (i < n) {
        const uint64_t d = re[j] - rs[j];
        set_bit(a.set_bits, a.set_summ, vv[j]);
        if (is_ns) {
          q[j] = d > k ? d - k : 0;
          o[j] = d < k ? d : k;
        } else {
          q[j] = d;
        }
      }
      qs += q[j];
      as += (q[j] > 0);
      os += o[j];
    }
    if (tile == role) tstamp(a.trace, role, 2);
    unsigned long long tq, ta, to = 0;
    unsigned long long eq = block_exclusive_scan<kNT>(qs, s_scan[0], tq);
    unsigned long long ea = block_exclusive_scan<kNT>(as, s_scan[1], ta);
    unsigned long long eo = 0;
    if (is_ns) eo = block_exclusive_scan<kNT>(os, s_scan[2], to);
    // the (two or three) look-backs run concurrently in warps 0, 1, 2
    tile_prefix_async<4>(a.st_a, tile, tq, inv_epoch(a.epoch, a.slot), &s_bc[0], 0);
    tile_prefix_async<4>(a.st_b, tile, ta, inv_epoch(a.epoch, a.slot + 1), &s_bc[1], 1);
    if (is_ns)
      tile_prefix_async<4>(a.st_c, tile, to, inv_epoch(a.epoch, a.slot + 2), &s_bc[2], 2);
    __syncthreads();
    const unsigned long long bq = s_bc[0], ba = s_bc[1];
    const unsigned long long bo = is_ns ? s_bc[2] : 0ULL;
    if (tile == role) tstamp(a.trace, role, 3);
    eq += bq;
    ea += ba;
    eo += bo;
    // Tiles started inside each record get tile_first; with lists, the
    // single-record ones (pure) go to the front of labor_mark's tile list
    // and the record's last started tile, when it holds a record boundary
    // (mixed), to the back. A hub starts hundreds of tiles: the whole warp
    // writes each record's tiles, one record after another.
    const bool lists = a.tile_list != nullptr;
    // list slots for all IPT records of a thread: one warp scan and one
    // atomic per list per warp (not per record), so the loop below does not
    // wait on an atomic round trip per j
    uint32_t bp = 0, bm = 0;
    if (lists) {
      uint32_t tnp = 0, tmix = 0;
      uint64_t e2 = eq;
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        if (i0 + j < n && q[j] > 0) {
          const uint64_t f = (e2 + kLaborTile - 1) / kLaborTile;
          const uint64_t l = min(static_cast<uint64_t>((e2 + q[j] - 1) / kLaborTile), a.cap_tiles);
          const uint64_t p = min(l + 1, static_cast<uint64_t>((e2 + q[j]) / kLaborTile));
          if (f <= l) {
            tnp += p > f ? static_cast<uint32_t>(p - f) : 0u;
            tmix += (l + 1 > p) ? 1u : 0u;
          }
        }
        e2 += q[j];
      }
      const uint32_t ip = warp_inclusive_scan(tnp), im2 = warp_inclusive_scan(tmix);
      uint32_t base_p = 0, base_m = 0;
      if (lane_id() == 31) {
        if (ip) base_p = atomicAdd(&a.list_ctr[0], ip);
        if (im2) base_m = atomicAdd(&a.list_ctr[1], im2);
      }
      bp = __shfl_sync(0xffffffffu, base_p, 31) + ip - tnp;
      bm = __shfl_sync(0xffffffffu, base_m, 31) + im2 - tmix;
    }
    if (tile == role) tstamp(a.trace, role, 5);  // list slots known
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t i = i0 + j;
      uint64_t tf = 1, tl = 0, pe = 0;  // started tiles [tf, tl]; pure below pe
      uint32_t rec_idx = 0;
      bool exact = false;
      if (i < n) {
        if (q[j] > 0) {
          ActRec rec;
          rec.pre = eq;
          rec.di = static_cast<uint32_t>(i);
          const uint64_t d = is_ns ? q[j] + k : q[j];
          rec.d = static_cast<uint32_t>(d);
          if (is_ns) {
            rec.a = eo;                  // output offset of the slots
            rec.b = hstep(z1p, vv[j]);   // prefix({kStreamNs, layer, s}) under z1
            if (eo + k <= a.cap_edges)   // hub: slots start as the identity
              for (uint32_t r2 = 0; r2 < k; ++r2) a.slots[eo + r2] = r2;
          } else {
            rec.a = rs[j] - eq;          // indices[rec.a + x] = neighbour at x
            // (a caller variate table may hold values > 1: no keep-all shortcut)
            if (full || (d <= k && v.smoothed != 2)) {
              rec.b = ~0ULL;
            } else {
              const double thr = __ddiv_rn(static_cast<double>(k), static_cast<double>(d));
              rec.b = smooth ? static_cast<unsigned long long>(__double_as_longlong(thr))
                             : __double2ull_rz(__dmul_rn(thr, 0x1.0p53));
            }
          }
          a.act[ea] = rec;
          // scan tiles whose first position falls inside this record
          // (clamped to the scan capacity: an overflowing layer is flagged
          // below and sampled empty, then retried with a larger plan)
          tf = (eq + kLaborTile - 1) / kLaborTile;
          tl = min(static_cast<uint64_t>((eq + q[j] - 1) / kLaborTile), a.cap_tiles);
          // bit 31: the record starts exactly at the tile start (so the
          // previous tile ends with record ea-1: no load to find it)
          exact = eq == tf * kLaborTile;
          // tiles t with (t + 1) * kLaborTile <= end lie inside this record
          pe = min(tl + 1, static_cast<uint64_t>((eq + q[j]) / kLaborTile));
          rec_idx = static_cast<uint32_t>(ea);
          ++ea;
        }
        if (is_ns) a.out_prefix[i] = eo;
      }
      eq += q[j];
      eo += o[j];
      // this record's list slots: pure tiles from bp, its mixed tile at bm
      const bool any = tf <= tl;
      const uint32_t np = (lists && any && pe > tf) ? static_cast<uint32_t>(pe - tf) : 0u;
      const bool mixed = lists && any && tl + 1 > pe;
      if (mixed && bm < a.list_cap)
        a.tile_list[a.list_cap - 1 - bm] = make_uint2(static_cast<uint32_t>(tl), rec_idx);
      // a record that starts a few tiles writes them itself; hubs (many
      // tiles) are written by the whole warp
      const bool coop = any && tl >= tf + 4;
      if (any && !coop) {
        for (uint64_t t = tf; t <= tl; ++t) {
          a.tile_first[t] = rec_idx | ((t == tf && exact) ? kTileExact : 0u);
          if (lists && t < pe && bp + (t - tf) < a.list_cap)
            a.tile_list[bp + (t - tf)] = make_uint2(static_cast<uint32_t>(t), rec_idx);
        }
      }
      unsigned todo = __ballot_sync(0xffffffffu, coop);
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint64_t f = __shfl_sync(0xffffffffu, tf, src);
        const uint64_t l2 = __shfl_sync(0xffffffffu, tl, src);
        const uint64_t p2 = __shfl_sync(0xffffffffu, pe, src);
        const uint32_t r2 = __shfl_sync(0xffffffffu, rec_idx, src);
        const bool ex = __shfl_sync(0xffffffffu, exact, src);
        const uint32_t b2 = __shfl_sync(0xffffffffu, bp, src);
        for (uint64_t t = f + lane_id(); t <= l2; t += 32) {
          a.tile_first[t] = r2 | ((t == f && ex) ? kTileExact : 0u);
          if (lists && t < p2 && b2 + (t - f) < a.list_cap)
            a.tile_list[b2 + (t - f)] = make_uint2(static_cast<uint32_t>(t), r2);
        }
      }
      bp += np;
      bm += mixed ? 1u : 0u;
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      uint64_t tot = bq + tq, nact = ba + ta;
      if ((tot + kLaborTile - 1) / kLaborTile > a.cap_tiles) {  // scan space overflow
        atomicExch(a.overflow, 1u);
        tot = nact = 0;
      }
      ActRec sent{};
      sent.pre = tot;
      a.act[nact] = sent;
      a.tile_first[(tot + kLaborTile - 1) / kLaborTile] = static_cast<uint32_t>(nact) | kTileExact;
      meta->scan_total = tot;
      meta->n_active = nact;
      meta->uncertified = 0;
      if (is_ns) {
        a.out_prefix[n] = bo + to;
        meta->n_edges = bo + to;
        if (bo + to > a.cap_edges) atomicExch(a.overflow, 1u);
      }
    }
  }
  tstamp(a.trace, role, 4);
  tlast(a.trace);
  if (n == 0 && role == 0 && threadIdx.x == 0) {
    ActRec sent{};
    a.act[0] = sent;
    a.tile_first[0] = kTileExact;
    meta->scan_total = 0;
    meta->n_active = 0;
    meta->uncertified = 0;
    meta->n_edges = 0;
    if (is_ns) a.out_prefix[0] = 0;
  }
}

// CTAs [0, n_front) run the frontier; the rest relabel layer l-1 (independent
// work on its own CTAs, so the frontier's load chain starts at once).
template <int IPT>
__global__ void __launch_bounds__(kNT) frontier_kernel(FrontierArgs a, RelabelArgs r,
                                                       unsigned n_front) {
  pdl_begin();
  if (blockIdx.x >= n_front) {
    relabel_range(r, (blockIdx.x - n_front) * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
                  static_cast<uint64_t>(gridDim.x - n_front) * blockDim.x);
    return;
  }
  frontier_body<IPT>(a, RelabelArgs{}, blockIdx.x, n_front);
}

// Largest record index in [lo, hi] whose scan prefix is <= x.
__device__ __forceinline__ uint32_t rec_search(const ActRec* __restrict__ act, uint32_t lo,
                                               uint32_t hi, uint64_t x) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(&act[mid].pre) <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Record range [a0, a1] overlapping scan tile [x0, x1).
// tile_first[t] = first record overlapping scan tile t, bit 31 set when that
// record starts exactly at the tile start (frontier_body).
__device__ __forceinline__ void tile_decode(uint32_t tf0, uint32_t tf1, uint32_t& a0,
                                            uint32_t& a1) {
  a0 = tf0 & ~kTileExact;
  a1 = (tf1 & ~kTileExact) - ((tf1 & kTileExact) ? 1u : 0u);
}
__device__ __forceinline__ void tile_records(const ActRec*, const uint32_t* tile_first, uint64_t,
                                             uint64_t tile, uint64_t, uint32_t& a0,
                                             uint32_t& a1) {
  tile_decode(__ldg(&tile_first[tile]), __ldg(&tile_first[tile + 1]), a0, a1);
}

// ------------------------------------------------------------- LABOR/FULL --
// keep(t -> s) iff U(hash(z1,{2,layer,t})) <= k/d_s  (samplers.cpp:117-134);
// plain stream compared in integers: (h>>11) <= floor((k/d)*2^53), exact.
//
// Two phases so the hashing never waits on an ordered scan:
//   labor_mark : every scan position independently (grid-stride tiles); lane
//                l of a warp owns position xw+l, so the warp ballot IS the
//                keep word of 32 consecutive positions; kept ids are OR-ed
//                into the layer bitmap (order-free)
//   labor_emit : ordered popcount compaction of the keep words (decoupled
//                look-back over 64K-position tiles) -> edges in scan order =
//                grouped by dst, CSR order inside a dst (the reference order)
// Keep decision for neighbour t under threshold th (frontier ActRec.b). Plain
// stream: th = ~0 (keep all) needs no special case since (h>>11) < 2^53.
// The layer's smoothed variate table r_t = finish(hash(z1,{2,l,t}),
// hash(z2,{2,l,t})) for every vertex, built when the scan space is at least
// twice the vertex count (each r_t then serves >= 2 positions on average).
__device__ __forceinline__ bool vtab_used(const LaborArgs& a, uint64_t scan_total) {
  return a.vtab != nullptr && scan_total >= 2 * a.n_vert;
}

__global__ void __launch_bounds__(kNT) vtab_kernel(LaborArgs a) {
  pdl_begin();
  if (!vtab_used(a, a.meta->scan_total)) return;
  const Variates v = *a.var;
  const uint64_t p1 = hstep(hstep(hinit(v.z1), 2ULL), static_cast<uint64_t>(a.layer));
  const uint64_t p2 = hstep(hstep(hinit(v.z2), 2ULL), static_cast<uint64_t>(a.layer));
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < a.n_vert;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a.vtab[t] = smooth_finish(v, hstep(p1, t), hstep(p2, t));
}

// Smoothed stream: r_t from the layer's variate table when one was built
// (samplers.cpp:114-129 memoises r_t per t the same way), else evaluated.
// Plain stream: (mix64(p1 ^ t) >> 11) <= th  <=>  mix64(p1 ^ t) <= T with
// T = th * 2^11 + 2^11 - 1 (th < 2^53; th >= 2^53 keeps every position), so
// the per-position test is one 64-bit compare without the shift.
__device__ __forceinline__ uint64_t plain_bound(uint64_t th) {
  return th >= (1ULL << 53) ? ~0ULL : ((th << 11) | 0x7ffULL);
}

// A smoothed decision inside the guard band takes the host-resolved r_t when
// the resolve table has it; otherwise it is counted as uncertified and
// recorded for the host (Variates::rs, DESIGN.md §Smoothed variates).
__device__ __noinline__ bool labor_in_band(const Variates& v, int layer, uint32_t t, double rr,
                                           double thr, unsigned long long& uncert) {
  const uint64_t k1 = kResolveLabor | (static_cast<uint64_t>(v.part) << 48) |
                      (static_cast<uint64_t>(layer) << 32) | t;
  double ex;
  if (resolve_lookup(v.rs, k1, 0, ex)) return ex <= thr;
  ++uncert;
  bool keep = rr <= thr;
  if (v.rs && v.rs->perturb) keep = !keep;  // test hook: a wrong device decision
  resolve_record(v.rs, k1, 0, keep ? thr : 2.0 * thr + 1.0, thr);
  return keep;
}

template <bool SMOOTH>
__device__ __forceinline__ bool keep_rule(const Variates& v, uint64_t p1, uint64_t p2,
                                          uint32_t t, uint64_t th, unsigned long long& uncert,
                                          const double* vtab, int layer) {
  if (!SMOOTH) return (mix64_dev(p1 ^ t) >> 11) <= th;
  if (th == ~0ULL) return true;
  const double thr = __longlong_as_double(static_cast<long long>(th));
  const double rr = vtab ? __ldg(vtab + t) : smooth_finish(v, hstep(p1, t), hstep(p2, t));
  // (a caller's variate table, smoothed == 2, is exact by definition)
  if (v.smoothed != 2 && fabs(rr - thr) <= v.guard * thr)
    return labor_in_band(v, layer, t, rr, thr, uncert);
  return rr <= thr;
}

// phase-B spans (mark_span, plain stream) with phase A's high-word
// prefilter: bit 0 spans inside one record, bit 1 spans across records.
// Off: A/B at c4, last-layer mark 81.7 (off) / 83.9 (1) / 92.5 (3) us --
// mixed tiles are mostly low-degree records whose positions pass the
// prefilter and then pay the exact hash as well.
#ifndef CB_SPAN_PREFILTER
#define CB_SPAN_PREFILTER 0
#endif
constexpr int kSpanPrefilter = CB_SPAN_PREFILTER;
#ifndef CB_COMPACT_SPAN
#define CB_COMPACT_SPAN 0
#endif
// CTA-mode phase B (small layers) with rolled keep loops (latency A/B)
constexpr bool kCompactSpan = CB_COMPACT_SPAN != 0;

// High word of y = z * c2, the last SplitMix64 multiply of mix64(p1 ^ t)
// (z after the second xor-shift): keep_plain's prefilter input.
__device__ __forceinline__ uint32_t mix64_yhi(uint64_t p1, uint32_t t) {
  uint64_t x = (p1 ^ t) + 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = x ^ (x >> 27);
  const uint32_t zlo = static_cast<uint32_t>(x), zhi = static_cast<uint32_t>(x >> 32);
  return __umulhi(zlo, 0x133111ebu) + zlo * 0x94d049bbu + zhi * 0x133111ebu;
}

// Carry-split form of mix64_yhi for a layer prefix p1 and a 32-bit id t.
// x = (p1 ^ t) + C0: t only touches the low word, so the high word is
// H + cy (cy = the carry out of the low add). After x ^= x >> 30 the high
// word's contribution to the first product's high half, (hi ^ hi >> 30) *
// 0x1ce4e5b9, is one of two per-layer constants K[cy]: one select instead of
// a shift, an xor and a multiply. Bit-exact with mix64_yhi.
struct YhiConst {
  uint32_t p1lo, Q0, Q1, K0, K1;
};
__host__ __device__ __forceinline__ YhiConst yhi_const(uint64_t p1) {
  YhiConst k;
  k.p1lo = static_cast<uint32_t>(p1);
  const uint32_t h0 = static_cast<uint32_t>(p1 >> 32) + 0x9e3779b9u, h1 = h0 + 1u;
  k.Q0 = h0 << 2;  // the high word's bits in the low word of x >> 30
  k.Q1 = h1 << 2;
  k.K0 = (h0 ^ (h0 >> 30)) * 0x1ce4e5b9u;
  k.K1 = (h1 ^ (h1 >> 30)) * 0x1ce4e5b9u;
  return k;
}
// K0 / K1 pass through an opaque move: otherwise the compiler sinks their
// multiply past the select (select(a, b) * c), one IMAD more per position.
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  uint32_t r;
  asm("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t mix64_yhi_cs(const YhiConst& k, uint32_t t) {
  uint32_t lo, cy;
  asm("add.cc.u32 %0, %2, 0x7f4a7c15;\n\taddc.u32 %1, 0, 0;"
      : "=r"(lo), "=r"(cy)
      : "r"(k.p1lo ^ t));
  const bool c = cy != 0;
  const uint32_t xl = lo ^ (lo >> 30) ^ (c ? k.Q1 : k.Q0);  // disjoint bits: | == ^
  const uint32_t hk = c ? k.K1 : k.K0;
  const uint32_t zl0 = xl * 0x1ce4e5b9u;
  const uint32_t zh0 = __umulhi(xl, 0x1ce4e5b9u) + xl * 0xbf58476du + hk;
  const uint32_t zlo = zl0 ^ __funnelshift_r(zl0, zh0, 27);
  const uint32_t zhi = zh0 ^ (zh0 >> 27);
  return __umulhi(zlo, 0x133111ebu) + zlo * 0x94d049bbu + zhi * 0x133111ebu;
}

// acc = 2 * acc + (yhi <= b2): the prefilter pass bit shifted in through
// the carry of b2 - yhi (one subtract with carry-out, one add with carry-in)
__device__ __forceinline__ uint32_t shift_in_pass(uint32_t acc, uint32_t b2, uint32_t yhi) {
  uint32_t r;
  asm("{\n .reg .u32 t;\n sub.cc.u32 t, %1, %2;\n addc.u32 %0, %3, %3;\n}"
      : "=r"(r)
      : "r"(b2), "r"(yhi), "r"(acc));
  return r;
}

// Plain-stream keep test with a high-word prefilter. out = y ^ (y >> 31) for
// y = z * c2 (the last SplitMix64 round), so out's top 31 bits are y's: when
// (y_hi >> 1) > (T_hi >> 1) the position is rejected without the final
// xor-shift and the 64-bit compare. Only survivors (about T / 2^64 of the
// positions: k/d of a hub's) finish the hash. Exact: same result as
// mix64(p1 ^ t) <= T.
__device__ __forceinline__ bool keep_plain(uint64_t p1, uint32_t t, uint64_t T) {
  uint64_t x = (p1 ^ t) + 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = x ^ (x >> 27);
  const uint32_t zlo = static_cast<uint32_t>(x), zhi = static_cast<uint32_t>(x >> 32);
  const uint32_t yhi = __umulhi(zlo, 0x133111ebu) + zlo * 0x94d049bbu + zhi * 0x133111ebu;
  if ((yhi >> 1) > static_cast<uint32_t>(T >> 33)) return false;
  const uint64_t y = x * 0x94d049bb133111ebULL;
  return (y ^ (y >> 31)) <= T;
}

// Per-warp body of labor_mark: IPT words of 32 consecutive positions starting
// at tile-relative offset r0. Records come either from smem (STAGED) or
// straight from the global record array (tiles spanning > kRecs records).
// Lane j keeps word j's ballot; one coalesced store at the end. Every kept
// position also leaves its finished edge (t, dst index) in the stage array,
// so the ordered emission is one load per edge.
// MODE 0: records read from global memory; 1: the tile's records staged in
// shared memory (s_act[0] = record a0, nd of them); 2: a window of nd records
// starting at `cur` in shared memory (s_act[0] = record a0 + cur), global
// memory past it.
template <int IPT, bool SMOOTH, int MODE, bool COMPACT = false>
__device__ __forceinline__ void mark_span(const LaborArgs& a, const Variates& v, uint64_t p1,
                                          uint64_t p2, uint64_t x0, uint32_t r0, uint32_t rend,
                                          uint32_t a0, uint32_t a1, uint32_t cur,
                                          const ActRec* s_act, uint32_t nd,
                                          unsigned long long& uncert, const double* vtab,
                                          const YhiConst& yk) {
  static_assert(IPT <= 32, "one word per lane");
  const uint32_t lane = lane_id();
  constexpr bool STAGED = MODE == 1;
  const uint32_t cw = cur;  // MODE 2: window base
  // record c in shared memory (MODE 1, or inside the MODE-2 window)
  auto in_smem = [&](uint32_t c) -> bool { return STAGED || (MODE == 2 && c - cw < nd); };
  auto sm = [&](uint32_t c) -> const ActRec& { return s_act[MODE == 2 ? c - cw : c]; };
  auto nxt_of = [&](uint32_t c) -> uint32_t {  // tile-relative start of record c+1
    if (STAGED)
      return (c + 1 < nd) ? static_cast<uint32_t>(min(static_cast<uint64_t>(s_act[c + 1].pre) - x0,
                                                      static_cast<uint64_t>(0xffffffffu)))
                          : 0xffffffffu;
    if (a0 + c + 1 > a1) return 0xffffffffu;
    const uint64_t pr = in_smem(c + 1) ? sm(c + 1).pre : __ldg(&a.act[a0 + c + 1].pre);
    return static_cast<uint32_t>(min(pr - x0, static_cast<uint64_t>(0xffffffffu)));
  };
  auto row_of = [&](uint32_t c) -> const uint32_t* {
    return a.indices + ((in_smem(c) ? sm(c).a : __ldg(&a.act[a0 + c].a)) + x0);
  };
  auto th_of = [&](uint32_t c) -> uint64_t {
    return in_smem(c) ? sm(c).b : __ldg(&a.act[a0 + c].b);
  };
  auto di_of = [&](uint32_t c) -> uint32_t {
    return in_smem(c) ? sm(c).di : __ldg(&a.act[a0 + c].di);
  };
  uint2* stage = a.stage + x0 + r0;
  uint32_t my_word = 0;
  const uint32_t nxt0 = nxt_of(cur);
  if (nxt0 >= r0 + 32 * IPT && r0 + 32 * IPT <= rend) {
    // fast path: the whole span lies inside record `cur`
    const uint32_t* row = row_of(cur) + r0 + lane;
    const uint64_t th = th_of(cur);
    const uint64_t T = plain_bound(th);
    const uint32_t di = di_of(cur);
    uint2* const st_lane = stage + lane;  // kept position j -> st_lane[32 j]
    uint32_t tv[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) tv[j] = __ldg(row + j * 32);
    if constexpr (!SMOOTH && (kSpanPrefilter & 1)) {
      // phase A's test: high-word prefilter, the exact hash for survivors
      // only (re-read: row is L1-hot), ballots only when the warp kept any
      const uint32_t b2 = static_cast<uint32_t>(T >> 32) | 1u;
      uint32_t cand = 0;
#pragma unroll
      for (int j = 0; j < IPT; ++j) cand = shift_in_pass(cand, b2, mix64_yhi_cs(yk, tv[j]));
      uint32_t km = __brev(cand) >> (32 - IPT);
      for (uint32_t kk = km; kk;) {
        const int j = __ffs(kk) - 1;
        kk &= kk - 1;
        if (!keep_plain(p1, __ldg(row + j * 32), T)) km &= ~(1u << j);
      }
      if (__any_sync(0xffffffffu, km != 0)) {
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
          const unsigned bal = __ballot_sync(0xffffffffu, (km >> j) & 1u);
          if (lane == j) my_word = bal;
        }
        for (uint32_t kk = km; kk;) {
          const int j = __ffs(kk) - 1;
          kk &= kk - 1;
          const uint32_t t = __ldg(row + j * 32);
          set_bit(a.bits, a.summ, t);
          st_lane[j * 32] = make_uint2(t, di);
        }
      }
      if (lane < IPT) a.keep_words[((x0 + r0) >> 5) + lane] = my_word;
      return;
    } else {
#pragma unroll
      auto keep_at = [&](int j) {
        const bool keep = SMOOTH ? keep_rule<SMOOTH>(v, p1, p2, tv[j], th, uncert, vtab, a.layer)
                                 : mix64_dev(p1 ^ tv[j]) <= T;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == j) my_word = bal;
        if (keep) {
          set_bit(a.bits, a.summ, tv[j]);
          st_lane[j * 32] = make_uint2(tv[j], di);
        }
      };
      if constexpr (COMPACT) {
#pragma unroll 1
        for (int j = 0; j < IPT; ++j) keep_at(j);
      } else {
#pragma unroll
        for (int j = 0; j < IPT; ++j) keep_at(j);
      }
    }
  } else {
    uint32_t li[IPT];
    uint32_t tv[IPT];
    uint32_t c = cur;
    uint32_t nxt = nxt0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint32_t r = r0 + j * 32 + lane;
      while (r >= nxt) {  // forward walk, only at record boundaries
        ++c;
        nxt = nxt_of(c);
      }
      li[j] = c;
      tv[j] = (r < rend) ? __ldg(row_of(c) + r) : 0u;
    }
    uint32_t km = 0;  // prefilter survivors (plain stream, kSpanPrefilter & 2)
    if (!SMOOTH && (kSpanPrefilter & 2)) {
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t b2 = static_cast<uint32_t>(plain_bound(th_of(li[j])) >> 32) | 1u;
        const bool pass = r0 + j * 32 + lane < rend && mix64_yhi_cs(yk, tv[j]) <= b2;
        km |= (pass ? 1u : 0u) << j;
      }
    }
    auto keep_at = [&](int j) {
      const uint32_t r = r0 + j * 32 + lane;
      const bool keep =
          (r < rend) &&
          (SMOOTH ? keep_rule<SMOOTH>(v, p1, p2, tv[j], th_of(li[j]), uncert, vtab, a.layer)
           : (kSpanPrefilter & 2) ? ((km >> j) & 1u) && keep_plain(p1, tv[j], plain_bound(th_of(li[j])))
                                  : mix64_dev(p1 ^ tv[j]) <= plain_bound(th_of(li[j])));
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == j) my_word = bal;
      if (keep) {
        set_bit(a.bits, a.summ, tv[j]);
        stage[j * 32 + lane] = make_uint2(tv[j], di_of(li[j]));
      }
    };
    // COMPACT (small layers' CTA-mode tiles): one loop body instead of IPT
    // unrolled copies, so a cold instruction cache fetches less code
    if constexpr (COMPACT) {
#pragma unroll 1
      for (int j = 0; j < IPT; ++j) keep_at(j);
    } else {
#pragma unroll
      for (int j = 0; j < IPT; ++j) keep_at(j);
    }
  }
  if (lane < IPT && r0 + lane * 32 < rend) a.keep_words[((x0 + r0) >> 5) + lane] = my_word;
}

// Record (local index from a0) of scan position x for a warp: 32-ary search
// over the records' starts in global memory (2-3 rounds of 32 parallel loads
// instead of a dependent binary search), then the next 32 records from there
// loaded into the warp's shared-memory window `win` (MODE 2 of mark_span).
// Returns the record; *nw = records in the window.
__device__ __forceinline__ uint32_t rec_window(const ActRec* __restrict__ act, uint32_t a0,
                                               uint32_t a1, uint64_t x, ActRec* win,
                                               uint32_t* nw) {
  const uint32_t lane = lane_id();
  uint32_t lo = 0, hi = a1 - a0;
  while (lo < hi) {
    const uint32_t step = (hi - lo + 32) / 32;
    const uint32_t cand = lo + lane * step;
    const bool le = cand <= hi && __ldg(&act[a0 + cand].pre) <= x;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const uint32_t best = lo + (31 - __clz(m)) * step;
    lo = best;
    hi = min(hi, best + step - 1);
    if (step == 1) break;
  }
  const uint32_t n = min(32u, a1 - a0 - lo + 1);
  __syncwarp();  // every lane is done with the window's previous contents
  if (lane < n) {
    const uint4* src = reinterpret_cast<const uint4*>(act + a0 + lo + lane);
    uint4* dst = reinterpret_cast<uint4*>(win + lane);
    const uint4 u0 = __ldg(src), u1 = __ldg(src + 1);
    dst[0] = u0;
    dst[1] = u1;
  }
  __syncwarp();
  *nw = n;
  return lo;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

// ---- bulk (TMA engine) staging of a single-record tile's neighbour ids ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
// one elected thread: expect `bytes` on bar, then the bulk global->shared copy
#ifndef CB_IDS_EVICT_FIRST
#define CB_IDS_EVICT_FIRST 0
#endif
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
#if CB_IDS_EVICT_FIRST
  // neighbour ids are read once per batch: evict them first so they do not
  // push the kernels' code and the batch metadata out of L2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n MBW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Span of a single-record tile whose ids sit in shared memory: the IPT keep
// decisions first (a bit mask per lane), then the keep words by ballot only
// when the warp kept anything (hub records keep ~k/d of their positions), and
// each kept position's bitmap bit and staged edge.
template <int IPT, bool SMOOTH>
__device__ __forceinline__ void mark_span_smem(const LaborArgs& a, const Variates& v,
                                               uint64_t p1, uint64_t p2, uint64_t x0,
                                               uint32_t r0, const uint32_t* ids,
                                               const ActRec& rec, unsigned long long& uncert,
                                               const double* vtab) {
  const uint32_t lane = lane_id();
  const uint64_t th = rec.b;
  const uint64_t T = plain_bound(th);
  uint32_t tv[IPT];
#pragma unroll
  for (int j = 0; j < IPT; ++j) tv[j] = ids[r0 + lane + 32 * j];
  uint32_t km = 0;
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const bool keep = SMOOTH ? keep_rule<SMOOTH>(v, p1, p2, tv[j], th, uncert, vtab, a.layer)
                             : mix64_dev(p1 ^ tv[j]) <= T;
    km |= (keep ? 1u : 0u) << j;
  }
  uint32_t my_word = 0;
  if (__any_sync(0xffffffffu, km != 0)) {
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const unsigned bal = __ballot_sync(0xffffffffu, (km >> j) & 1u);
      if (lane == j) my_word = bal;
    }
    if (km) {
      uint2* st_lane = a.stage + x0 + r0 + lane;
#pragma unroll
      for (int j = 0; j < IPT; ++j)
        if ((km >> j) & 1u) {
          set_bit(a.bits, a.summ, tv[j]);
          st_lane[j * 32] = make_uint2(tv[j], rec.di);
        }
    }
  }
  if (lane < IPT) a.keep_words[((x0 + r0) >> 5) + lane] = my_word;
}

#ifndef CB_MARK_RECS
#define CB_MARK_RECS (kLaborTile / 8)
#endif
constexpr int kMarkRecs = CB_MARK_RECS;
#ifndef CB_PURE_STAGES
#define CB_PURE_STAGES 1
#endif
// sub-tiles per single-record tile: the ring holds CB_PURE_STAGES stages of
// kLaborTile / CB_PURE_PARTS positions per warp
#ifndef CB_PURE_PARTS
#define CB_PURE_PARTS 1
#endif
constexpr int kPureParts = CB_PURE_PARTS;
// phase A work split: 0 = static (warp gw takes entries gw, gw + W, ...),
// G > 0 = G entries at a time from a ticket
#ifndef CB_PURE_GRAB
#define CB_PURE_GRAB 0
#endif
// phase B (tiles with record boundaries): one warp per tile without CTA
// barriers once there is at least one tile per CB_MIXED_WARP_DIV warps of the
// grid, else CTA-cooperative tiles (staged records, a barrier per tile).
// A/B at c4: 134 -> 129 us/step in warp mode; the small early layers keep the
// shorter CTA path (layer-0 mark 16 vs 34 us).
#ifndef CB_MIXED_WARP_DIV
#define CB_MIXED_WARP_DIV 1
#endif
constexpr int kMixedWarpDiv = CB_MIXED_WARP_DIV;

constexpr int kPureStages = CB_PURE_STAGES;     // id tiles in flight per warp
constexpr uint32_t kPureStride = kLaborTile / kPureParts + 8;  // u32 per stage (+ alignment slack)

// labor_mark's dynamic shared memory: phase B (records, ids, tile list) and
// phase A (per-warp id rings) reuse the same bytes one after the other.
struct MarkSmemB {
  ActRec act[3][kMarkRecs];
  uint32_t ids[2][kLaborTile + 4];
};
struct MarkSmemA {
  uint32_t ring[kMarkNT / 32][kPureStages][kPureStride];
};
constexpr size_t mark_smem_bytes(bool smooth) {
  return smooth ? sizeof(MarkSmemB)
                : (sizeof(MarkSmemA) > sizeof(MarkSmemB) ? sizeof(MarkSmemA) : sizeof(MarkSmemB));
}

// Phase A of labor_mark (plain stream): every full scan tile that lies inside
// ONE record (hub neighbour lists: most positions at c4) is hashed by one warp
// on its own, from a per-warp ring of kPureStages tiles brought into shared
// memory by bulk copies (TMA engine, mbarrier-completed) issued kPureStages
// tiles ahead, with no CTA barrier. Warp gw of W takes candidate tiles
// gw, gw + W, ...; a batch of 32 candidates is classified at once (lane i:
// candidate i, its record read when pure). Lane l owns positions l + 32 j of
// the tile, so the ballot at j is keep word j; warps that kept nothing (the
// common case for a hub: ~k/d of its positions survive) skip the ballots.
template <int NS>
__device__ __forceinline__ void mark_pure(const LaborArgs& a, uint64_t p1, uint64_t n_pure,
                                          unsigned role, unsigned ncta, uint32_t* ring,
                                          uint64_t* bars) {
  constexpr uint32_t TILE = kLaborTile;
  constexpr uint32_t PARTS = kPureParts;   // sub-tiles per tile (ring stages per tile)
  constexpr uint32_t SUB = TILE / PARTS;   // positions per sub-tile
  constexpr uint32_t WPS = SUB / 32;       // keep words per sub-tile
  static_assert(WPS >= 1 && WPS <= 32 && TILE % PARTS == 0, "sub-tile shape");
  constexpr uint32_t WPC = kMarkNT / 32;
  const uint32_t lane = lane_id();
  const uint64_t W = static_cast<uint64_t>(ncta) * WPC;
  const uint64_t gw = static_cast<uint64_t>(role) * WPC + (threadIdx.x >> 5);
  if (gw >= n_pure) return;
  YhiConst yk = yhi_const(p1);
  yk.K0 = opaque(yk.K0);
  yk.K1 = opaque(yk.K1);
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;  // parity bit per stage
  unsigned long long dbg_tiles = 0, dbg_surv = 0;  // trace diagnostics
#if CB_PURE_GRAB > 0
  // dynamic split (build option): the warp takes CB_PURE_GRAB entries at a
  // time from the layer's phase-A ticket (zeroed by batch_begin). A/B at c4:
  // the last-layer mark alone 91.6 -> 85.4 us (warps of a CTA reach the
  // phase-B barrier together), but 134 -> 145 us/step with 8 batches in
  // flight, so the static split stays the default.
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(a.pure_ticket, static_cast<unsigned>(CB_PURE_GRAB));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n_pure) break;
    const uint64_t e = static_cast<uint64_t>(base) + lane;
    const bool have = lane < static_cast<uint32_t>(CB_PURE_GRAB) && e < n_pure;
    uint64_t row = 0, T = 0, x0 = 0;
    uint32_t di = 0;
#else
  for (uint64_t kb = 0; gw + kb * 32 * W < n_pure; ++kb) {
    // lane i: list entry gw + (32 kb + i) W = (tile, record)
    const uint64_t e = gw + (kb * 32 + lane) * W;
    uint64_t row = 0, T = 0, x0 = 0;
    uint32_t di = 0;
    const bool have = e < n_pure;
#endif
    if (have) {
      const uint2 tr = a.tile_list[e];
      x0 = static_cast<uint64_t>(tr.x) * TILE;
      row = __ldg(&a.act[tr.y].a) + x0;
      T = plain_bound(__ldg(&a.act[tr.y].b));
      di = __ldg(&a.act[tr.y].di);
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, have);
    // work items: each listed tile in lane order, as PARTS sub-tiles of SUB
    // positions (WPS keep words) each, one ring stage per sub-tile
    uint32_t im = mask;  // items still to issue: lane __ffs(im) - 1, sub-tile ih
    uint32_t ih = 0;
    // bulk copy of item (lane `src`, sub-tile h) into stage s (lane 0 issues)
    auto issue = [&](uint32_t src, uint32_t h, int s) {
      const uint64_t r = __shfl_sync(0xffffffffu, row, src) + h * SUB;
      if (lane == 0) {
        const uint32_t* first = a.indices + r;
        const uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~static_cast<uintptr_t>(15);
        const uint32_t delta = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(first) - lo) >> 2);
        bulk_g2s(ring + s * kPureStride, reinterpret_cast<const void*>(lo),
                 ((SUB + delta) * 4u + 15u) & ~15u, &bars[s]);
      }
    };
    auto issue_next = [&](int s) {
      issue(__ffs(im) - 1, ih, s);
      if (++ih == PARTS) {
        ih = 0;
        im &= im - 1;
      }
    };
    int s_issue = 0;
    for (int q = 0; q < NS && im; ++q) {
      issue_next(s_issue);
      s_issue = s_issue + 1 == NS ? 0 : s_issue + 1;
    }
    uint32_t cm = mask, ch = 0;
    int s = 0;
    while (cm) {
      const uint32_t src = __ffs(cm) - 1;
      const uint32_t h = ch;
      if (++ch == PARTS) {
        ch = 0;
        cm &= cm - 1;
      }
      const uint64_t r = __shfl_sync(0xffffffffu, row, src) + h * SUB;
      const uint64_t Tq = __shfl_sync(0xffffffffu, T, src);
      const uint64_t xq = __shfl_sync(0xffffffffu, x0, src) + h * SUB;
      const uint32_t dq = __shfl_sync(0xffffffffu, di, src);
      const uint32_t delta = static_cast<uint32_t>(
          (reinterpret_cast<uintptr_t>(a.indices + r) & 15u) >> 2);
      mbar_wait(&bars[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const uint32_t* ids = ring + s * kPureStride + delta + lane;
      // prefilter pass bits (yhi <= b2 <=> (yhi >> 1) <= (T >> 33)), then the
      // exact test for the few survivors
      const uint32_t b2 = static_cast<uint32_t>(Tq >> 32) | 1u;
      uint32_t cand = 0;  // bit WPS - 1 - j: position j passed
#pragma unroll 8
#ifdef CB_NO_CARRY_SPLIT
      for (uint32_t j = 0; j < WPS; ++j) cand = shift_in_pass(cand, b2, mix64_yhi(p1, ids[32 * j]));
#else
      for (uint32_t j = 0; j < WPS; ++j)
        cand = shift_in_pass(cand, b2, mix64_yhi_cs(yk, ids[32 * j]));
#endif
      uint32_t km = __brev(cand) >> (32 - WPS);
      ++dbg_tiles;
      dbg_surv += __popc(km);
      for (uint32_t kk = km; kk;) {
        const int j = __ffs(kk) - 1;
        kk &= kk - 1;
        if (!keep_plain(p1, ids[32 * j], Tq)) km &= ~(1u << j);
      }
      uint32_t my_word = 0;
      if (__any_sync(0xffffffffu, km != 0)) {
#pragma unroll
        for (uint32_t j = 0; j < WPS; ++j) {
          const unsigned bal = __ballot_sync(0xffffffffu, (km >> j) & 1u);
          if (lane == j) my_word = bal;
        }
        uint32_t kk = km;
        while (kk) {
          const int j = __ffs(kk) - 1;
          kk &= kk - 1;
          const uint32_t v = ids[32 * j];
          set_bit(a.bits, a.summ, v);
          a.stage[xq + lane + 32 * j] = make_uint2(v, dq);
        }
      }
      if (lane < WPS) a.keep_words[(xq >> 5) + lane] = my_word;
      __syncwarp();  // every lane is done with stage s
      if (im) issue_next(s);
      s = s + 1 == NS ? 0 : s + 1;
    }
  }
  if (a.trace && role % 16 == 0 && (threadIdx.x >> 5) == 0) {  // diagnostics (CB_TRACE)
    const unsigned long long s = warp_sum(dbg_surv);
    if (lane == 0) {
      a.trace[(role / 16) * 8 + 5] = dbg_tiles;
      a.trace[(role / 16) * 8 + 6] = s;
    }
  }
}

// Phase B by warps (CB_MIXED_WARP): each warp takes whole tiles with record
// boundaries (warp gw: the back of the list, entries gw, gw + W, ...), stages
// the tile's records in its own shared memory (the phase-A ring of the same
// warp, so neither phase waits for the CTA) and marks the tile as four spans
// of 32 * IPT positions (mark_span). No CTA barrier anywhere.
template <int IPT>
__device__ __forceinline__ void mark_mixed_warp(const LaborArgs& a, const Variates& v,
                                                uint64_t p1, uint64_t n_mixed, uint64_t total,
                                                unsigned role, unsigned ncta, ActRec* wrec) {
  constexpr uint32_t TILE = kLaborTile;
  constexpr uint32_t WSPAN = 32 * IPT;
  constexpr uint32_t WPC = kMarkNT / 32;
  constexpr uint32_t kRecsW = (kPureStages * kPureStride * 4) / sizeof(ActRec);  // the warp ring
  static_assert(kRecsW >= 32, "the 32-record window fits the warp ring");
  const uint32_t lane = lane_id();
  const uint64_t W = static_cast<uint64_t>(ncta) * WPC;
  const uint64_t gw = static_cast<uint64_t>(role) * WPC + (threadIdx.x >> 5);
  unsigned long long uncert = 0;
  YhiConst yk = yhi_const(p1);
  yk.K0 = opaque(yk.K0);
  yk.K1 = opaque(yk.K1);
  for (uint64_t e = gw; e < n_mixed; e += W) {
    const uint64_t tile = a.tile_list[a.list_cap - 1 - e].x;
    const uint64_t x0 = tile * TILE;
    const uint32_t rend = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), total - x0));
    uint32_t a0, a1;
    tile_records(a.act, a.tile_first, 0, tile, 0, a0, a1);
    const uint32_t nd = a1 - a0 + 1;
    const bool staged = nd <= kRecsW;
    __syncwarp();  // every lane is done with the previous tile's records
    if (staged) {
      const uint4* src = reinterpret_cast<const uint4*>(a.act + a0);
      uint4* dst = reinterpret_cast<uint4*>(wrec);
      for (uint32_t i = lane; i < 2 * nd; i += 32) dst[i] = __ldg(src + i);
      __syncwarp();
    }
    for (uint32_t r0 = 0; r0 < rend; r0 += WSPAN) {
      if (staged) {
        // record of the span's first position: 32-ary search over the starts
        uint32_t lo = 0, hi = nd - 1;
        while (lo < hi) {
          const uint32_t step = (hi - lo + 32) / 32;
          const uint32_t cand = lo + lane * step;
          const bool le = cand <= hi && wrec[cand].pre <= x0 + r0;
          const unsigned m = __ballot_sync(0xffffffffu, le);
          const uint32_t best = lo + (31 - __clz(m)) * step;
          lo = best;
          hi = min(hi, best + step - 1);
          if (step == 1) break;
        }
        mark_span<IPT, false, 1>(a, v, p1, 0, x0, r0, rend, a0, a1, lo, wrec, nd, uncert,
                                    nullptr, yk);
      } else {  // more records than the ring holds: a 32-record window of them
        uint32_t nw;
        const uint32_t cur = rec_window(a.act, a0, a1, x0 + r0, wrec, &nw);
        mark_span<IPT, false, 2>(a, v, p1, 0, x0, r0, rend, a0, a1, cur, wrec, nw, uncert,
                                 nullptr, yk);
      }
    }
  }
}

// labor_mark: tiles of kNT*IPT scan positions, one 32*IPT span per warp.
// Plain stream: phase A (mark_pure) first takes the full single-record tiles;
// phase B then runs the tiles with record boundaries (or a partial last tile),
// listed per CTA from its grid-stride candidates. Smoothed stream: every tile
// in phase B. In phase B a tile's records (when <= kRecs) are staged raw in
// shared memory by cp.async, triple-buffered: records of the next two tiles
// are in flight or staged while one is hashed.
template <int IPT, bool SMOOTH>
__device__ __forceinline__ void mark_body(const LaborArgs& a, unsigned role, unsigned ncta) {
  constexpr int TILE = kMarkNT * IPT;
  static_assert(TILE == kLaborTile, "tile size shared with frontier");
  constexpr uint32_t WSPAN = 32 * IPT;  // contiguous positions owned by one warp
  constexpr int kRecs = kMarkRecs;  // records staged in smem (else global path)
  constexpr int WPC = kMarkNT / 32;
  extern __shared__ __align__(128) unsigned char s_raw[];  // mark_smem_bytes(SMOOTH)
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ __align__(8) uint64_t s_rbar[SMOOTH ? 1 : WPC][kPureStages];
  __shared__ uint32_t s_delta[2];
  MarkSmemB& sb = *reinterpret_cast<MarkSmemB*>(s_raw);
  auto& s_act = sb.act;
  auto& s_ids = sb.ids;
  LayerMeta* meta = a.meta;
  const uint64_t total = meta->scan_total;
  const uint64_t ntiles = (total + TILE - 1) / TILE;
  const Variates v = *a.var;
  // prefix({kStreamLabor, layer}) under z1 (and z2 when smoothed)
  const uint64_t p1 = hstep(hstep(hinit(v.z1), 2ULL), static_cast<uint64_t>(a.layer));
  const uint64_t p2 = SMOOTH ? hstep(hstep(hinit(v.z2), 2ULL), static_cast<uint64_t>(a.layer)) : 0;
  const double* vtab = (SMOOTH && vtab_used(a, total)) ? a.vtab : nullptr;
  const uint32_t warp = threadIdx.x >> 5;
  unsigned long long uncert = 0;
#ifdef CB_TRACE_FIRST  // trace the first 64 CTAs instead (small layers)
  const unsigned trole = role < 64 ? role : 64u;
#else
  const unsigned trole = (role % 16 == 0) ? role / 16 : 64u;  // trace: every 16th CTA
#endif
  tstamp(a.trace, trole, 0);
  // ---- phase A (plain stream with the frontier's tile lists): the
  // single-record tiles, one warp each. Phase B: the tiles with record
  // boundaries (the back of the list), or every tile without lists.
  const bool listed = !SMOOTH && a.tile_list != nullptr;
  uint64_t n_mixed = 0;
  unsigned prole = role;  // this CTA's phase-B slot
  if (listed) {
    const uint64_t n_pure = min(static_cast<uint64_t>(a.list_ctr[0]), ntiles);
    // phase-B tiles start at the first CTA without a phase-A tile, so a small
    // layer's CTA never runs a pure and a mixed tile back to back
    const unsigned off = static_cast<unsigned>(
        min(static_cast<uint64_t>(ncta), (n_pure + WPC - 1) / WPC) % ncta);
    prole = (role + ncta - off) % ncta;
    n_mixed = min(static_cast<uint64_t>(a.list_ctr[1]), ntiles - n_pure);
    MarkSmemA& sa = *reinterpret_cast<MarkSmemA*>(s_raw);
    mark_pure<kPureStages>(a, p1, n_pure, role, ncta, &sa.ring[warp][0][0], s_rbar[warp]);
    // many mixed tiles (every warp gets one or more): one warp per tile, no
    // CTA barriers; few (small layers): four warps per tile, shorter path
    if (n_mixed * kMixedWarpDiv >= static_cast<uint64_t>(ncta) * WPC) {
      tstamp(a.trace, trole, 2);
      mark_mixed_warp<IPT>(a, v, p1, n_mixed, total, role, ncta,
                           reinterpret_cast<ActRec*>(&sa.ring[warp][0][0]));
      tstamp(a.trace, trole, 1);
      tlast(a.trace);
      return;
    }
    __syncthreads();  // the ring memory becomes phase B's
    tstamp(a.trace, trole, 2);
  }
  YhiConst yk = yhi_const(p1);
  yk.K0 = opaque(yk.K0);
  yk.K1 = opaque(yk.K1);
  const uint64_t nb = listed ? (n_mixed > prole ? (n_mixed - prole + ncta - 1) / ncta : 0)
                             : (ntiles > role ? (ntiles - role + ncta - 1) / ncta : 0);
  // tile of phase-B item i
  auto tile_at = [&](uint64_t i) -> uint64_t {
    const uint64_t j = prole + i * ncta;
    return listed ? static_cast<uint64_t>(a.tile_list[a.list_cap - 1 - j].x) : j;
  };
  auto stage = [&](uint32_t a0, uint32_t a1, int buf) {
    const uint32_t nd = a1 - a0 + 1;
    if (nd <= static_cast<uint32_t>(kRecs)) {
      const char* src = reinterpret_cast<const char*>(a.act + a0);
      char* dst = reinterpret_cast<char*>(s_act[buf]);
      for (uint32_t i = threadIdx.x; i < 2 * nd; i += kMarkNT) cp_async16(dst + 16 * i, src + 16 * i);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // ids of tile t (inside record 0 of records buffer rb) -> s_ids[ib] by one
  // bulk copy of the 16-byte-aligned superset; the tile's first id sits at
  // s_ids[ib][s_delta[ib]] (indices carry >= 16 B of tail padding)
  auto stage_ids = [&](uint64_t t, int rb, int ib) {
    const uint64_t x0 = t * TILE;
    const uint32_t rend = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), total - x0));
    const uint32_t* first = a.indices + (s_act[rb][0].a + x0);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~static_cast<uintptr_t>(15);
    const uint32_t delta = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(first) - lo) >> 2);
    const uint32_t bytes = ((rend + delta) * 4u + 15u) & ~15u;
    s_delta[ib] = delta;
    bulk_g2s(s_ids[ib], reinterpret_cast<const void*>(lo), bytes, &s_bar[ib]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0]);
    mbar_init(&s_bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // records of the first two items; tile_first of the third. Record ranges
  // of this item (c), the next (n) and the one after (m) rotate in registers.
  uint32_t c0 = 0, c1 = 0, n0 = 0, n1 = 0, m0 = 0, m1 = 0;
  uint32_t tfa = 0, tfb = 0;
  if (nb > 0) {
    tile_records(a.act, a.tile_first, 0, tile_at(0), 0, c0, c1);
    stage(c0, c1, 0);
  }
  if (nb > 1) {
    tile_records(a.act, a.tile_first, 0, tile_at(1), 0, n0, n1);
    stage(n0, n1, 1);
  }
  if (nb > 2) {
    const uint64_t t2 = tile_at(2);
    tfa = __ldg(&a.tile_first[t2]);
    tfb = __ldg(&a.tile_first[t2 + 1]);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // barriers initialised, first records visible
  tstamp(a.trace, trole, 3);
  uint32_t iphase = 0;  // mbarrier phase bit per id buffer (bit ib)
  uint32_t ipure = 0;   // id buffer ib holds its tile's ids (bit ib)
  if (threadIdx.x == 0 && nb > 0 && c0 == c1) stage_ids(tile_at(0), 0, 0);
  if (nb > 0 && c0 == c1) ipure |= 1u;
  int rb = 0, ib = 0;
  for (uint64_t i = 0; i < nb; ++i) {
    const uint64_t tile = tile_at(i);
    const int rb1 = rb == 2 ? 0 : rb + 1, rb2 = rb1 == 2 ? 0 : rb1 + 1;
    // the item after this one: its ids (single-record tile) one item ahead
    if (i + 1 < nb && n0 == n1) {
      if (threadIdx.x == 0) stage_ids(tile_at(i + 1), rb1, ib ^ 1);
      ipure |= 2u >> ib;  // bit (ib ^ 1)
    } else {
      ipure &= ~(2u >> ib);
    }
    // records of the item after that (buffer of the item two back is free:
    // every warp passed this iteration's trailing barrier of the last one)
    if (i + 2 < nb) {
      tile_decode(tfa, tfb, m0, m1);
      stage(m0, m1, rb2);
      if (i + 3 < nb) {
        const uint64_t t3 = tile_at(i + 3);
        tfa = __ldg(&a.tile_first[t3]);
        tfb = __ldg(&a.tile_first[t3 + 1]);
      }
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const uint64_t x0 = tile * TILE;
    const uint32_t rend = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), total - x0));
    const uint32_t a0 = c0, a1 = c1;
    const uint32_t nd = a1 - a0 + 1;
    const uint32_t r0 = warp * WSPAN;
    if ((ipure >> ib) & 1u) {
      mbar_wait(&s_bar[ib], (iphase >> ib) & 1u);
      iphase ^= 1u << ib;
      if (r0 + WSPAN <= rend) {
        mark_span_smem<IPT, SMOOTH>(a, v, p1, p2, x0, r0, s_ids[ib] + s_delta[ib], s_act[rb][0],
                                    uncert, vtab);
      } else if (r0 < rend) {
        mark_span<IPT, SMOOTH, 1, kCompactSpan>(a, v, p1, p2, x0, r0, rend, a0, a1, 0, s_act[rb], nd, uncert,
                                     vtab, yk);
      }
    } else if (r0 < rend) {
      if (nd <= static_cast<uint32_t>(kRecs)) {
        const ActRec* sa = s_act[rb];
        // record of the warp's first position: 32-ary search over the starts
        uint32_t lo = 0, hi = nd - 1;
        while (lo < hi) {
          const uint32_t step = (hi - lo + 32) / 32;
          const uint32_t cand = lo + lane_id() * step;
          const bool le = cand <= hi && sa[cand].pre <= x0 + r0;
          const unsigned m = __ballot_sync(0xffffffffu, le);
          const uint32_t best = lo + (31 - __clz(m)) * step;
          lo = best;
          hi = min(hi, best + step - 1);
          if (step == 1) break;
        }
        mark_span<IPT, SMOOTH, 1, kCompactSpan>(a, v, p1, p2, x0, r0, rend, a0, a1, lo, sa, nd, uncert,
                                     vtab, yk);
      } else {  // more records than s_act holds: a 32-record window per warp
        static_assert(kRecs >= 32 * (kMarkNT / 32), "one 32-record window per warp");
        uint32_t nw;
        ActRec* win = s_act[rb] + 32 * warp;  // unused by this item (not staged)
        const uint32_t cur = rec_window(a.act, a0, a1, x0 + r0, win, &nw);
        mark_span<IPT, SMOOTH, 2, kCompactSpan>(a, v, p1, p2, x0, r0, rend, a0, a1, cur, win, nw, uncert,
                                  vtab, yk);
      }
    }
    if (i == 0) tstamp(a.trace, trole, 4);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // this item's buffers are free; the next records are visible
    rb = rb1;
    ib ^= 1;
    c0 = n0;
    c1 = n1;
    n0 = m0;
    n1 = m1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (SMOOTH) {
    uncert = warp_sum(uncert);
    if (lane_id() == 0 && uncert) atomicAdd(&meta->uncertified, uncert);
  }
  __syncthreads();
  tstamp(a.trace, trole, 1);
  tlast(a.trace);
}

template <int IPT, bool SMOOTH>
__global__ void __launch_bounds__(kMarkNT, SMOOTH ? 6 : kMarkMinBlocks) labor_mark_kernel(LaborArgs a) {
  pdl_begin();
  mark_body<IPT, SMOOTH>(a, blockIdx.x, gridDim.x);
}

// Emit tiles: 256 keep words (8K positions) per tile for small layers, 2048
// (64K positions) once a layer has > 64K words, so the look-back front never
// walks more than a few thousand tiles.
#ifndef CB_EMIT_WPT
#define CB_EMIT_WPT 8
#endif
constexpr int kEmitWPT = CB_EMIT_WPT;           // max keep words per thread
constexpr int kEmitTileWords = kNT * kEmitWPT;  // max words per tile
constexpr uint64_t kEmitBigLayerWords = 64 * 1024;

// Ordered compaction of the keep words. The tile's kept items are spread
// over all threads (item q -> its word by binary search over the per-word
// output bases in smem); the edge itself was staged by labor_mark at its scan
// position, so each kept edge is one load and one store.
__device__ __forceinline__ void labor_emit_body(const LaborArgs& a, unsigned role,
                                                unsigned ncta,
                                                unsigned long long* trace_in = nullptr) {
  unsigned long long* trace = role < 32 ? trace_in : nullptr;
  __shared__ unsigned long long s_scan[kNT / 32 + 1];
  __shared__ uint32_t s_wbase[kEmitTileWords + 1];
  __shared__ uint32_t s_word[kEmitTileWords];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  LayerMeta* meta = a.meta;
  const uint64_t total = meta->scan_total;
  const uint64_t nwords = (total + 31) / 32;
  const int wpt = nwords > kEmitBigLayerWords ? kEmitWPT : 1;
  const uint32_t tw = kNT * wpt;  // words per tile
  const uint64_t ntiles = (nwords + tw - 1) / tw;
  const unsigned ep = inv_epoch(a.epoch, a.slot);
  tstamp(trace, 32 + role, 0);
  for (unsigned tile = role; tile < ntiles; tile = next_tile_after(a.ticket, &s_tile, ncta, ntiles)) {
    const uint64_t wt = static_cast<uint64_t>(tile) * tw;
    const uint32_t l0 = threadIdx.x * wpt;
    uint32_t wv[kEmitWPT];
    unsigned long long c = 0;
#pragma unroll
    for (int j = 0; j < kEmitWPT; ++j) {
      wv[j] = (j < wpt && wt + l0 + j < nwords) ? a.keep_words[wt + l0 + j] : 0u;
      c += __popc(wv[j]);
    }
    if (tile == role) tstamp(trace, 32 + role, 1);
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<kNT>(c, s_scan, tot);
    if (tile == role) tstamp(trace, 32 + role, 2);
    uint32_t run = static_cast<uint32_t>(ex);
#pragma unroll
    for (int j = 0; j < kEmitWPT; ++j) {
      if (j < wpt) {
        s_word[l0 + j] = wv[j];
        s_wbase[l0 + j] = run;
        run += __popc(wv[j]);
      }
    }
    const unsigned long long gb = tile_prefix<4>(a.status, tile, tot, ep, &s_b);
    if (tile == role) tstamp(trace, 32 + role, 3);
    // (tile_prefix ends with __syncthreads: s_word / s_wbase are visible)
    constexpr int B = 8;  // kept items per thread in flight
    for (uint32_t q0 = threadIdx.x; q0 < tot; q0 += kNT * B) {
      uint2 e[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const uint32_t q = q0 + u * kNT;
        if (q < tot) {
          uint32_t lo = 0, hi = tw - 1;
          while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (s_wbase[mid] <= q) lo = mid;
            else hi = mid - 1;
          }
          uint32_t word = s_word[lo];
          for (uint32_t r = q - s_wbase[lo]; r > 0; --r) word &= word - 1;
          e[u] = __ldg(&a.stage[(wt + lo) * 32 + (__ffs(word) - 1)]);
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const unsigned long long pos = gb + q0 + u * kNT;
        if (q0 + u * kNT < tot && pos < a.cap_edges) a.edges[pos] = e[u];
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      meta->n_edges = gb + tot;
      if (gb + tot > a.cap_edges) atomicExch(a.overflow, 1u);
    }
  }
  tstamp(trace, 32 + role, 4);
  tlast(trace_in);
}

// ---------------------------------------------------------------- NS -------
// Reservoir (samplers.cpp:75-84) restated per slot: the final content of slot
// j is the largest i in [k, d) with floor(U_i*(i+1)) == j, else j. Every
// position is an independent atomicMax, so hub rows split across CTAs.
// NS slot roll r = floor(u * (i + 1)) near an integer (ns_block,
// samplers.cpp:80-82): the host-resolved u when the resolve table has it,
// else counted as uncertified and recorded for the host.
__device__ __noinline__ uint64_t ns_in_band(const Variates& v, int layer, uint32_t s, uint64_t i,
                                            double u, uint64_t r, unsigned long long& uncert) {
  const uint64_t k1 = (static_cast<uint64_t>(v.part) << 48) | (static_cast<uint64_t>(layer) << 32) | s;
  double ex;
  if (resolve_lookup(v.rs, k1, i, ex))
    return __double2ull_rz(__dmul_rn(ex, static_cast<double>(i + 1)));
  ++uncert;
  if (v.rs && v.rs->perturb) {  // test hook: the other side of the integer
    const double y = __dmul_rn(u, static_cast<double>(i + 1));
    const uint64_t n = static_cast<uint64_t>(floor(y + 0.5));
    r = (r == n) ? n - 1 : n;
  }
  resolve_record(v.rs, k1, i, u, static_cast<double>(r));
  return r;
}

template <int IPT, bool SMOOTH>
__global__ void __launch_bounds__(kNT) ns_reservoir_kernel(LaborArgs a) {
  pdl_begin();
  constexpr int TILE = kNT * IPT;
  static_assert(TILE == kLaborTile, "tile size shared with frontier");
  LayerMeta* meta = a.meta;
  const uint64_t total = meta->scan_total;
  const uint64_t n_act = meta->n_active;
  const uint64_t ntiles = (total + TILE - 1) / TILE;
  const Variates v = *a.var;
  constexpr bool smooth = SMOOTH;
  const uint64_t z2p = hstep(hstep(hinit(v.z2), 1ULL), static_cast<uint64_t>(a.layer));
  const uint32_t k = a.k;
  unsigned long long uncert = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t x0 = tile * TILE;
    const uint64_t x1 = min(x0 + TILE, total);
    uint32_t a0, a1;
    tile_records(a.act, a.tile_first, n_act, tile, x1, a0, a1);
#pragma unroll 4
    for (int j = 0; j < IPT; ++j) {
      const uint64_t x = x0 + static_cast<uint64_t>(j) * kNT + threadIdx.x;
      if (x < x1) {
        const uint32_t li = rec_search(a.act, a0, a1, x);
        const ActRec rec = a.act[li];
        const uint64_t i = k + (x - rec.pre);
        const double scale = static_cast<double>(i + 1);
        double u;
        uint64_t r;
        if (!smooth) {
          u = ufb(hstep(rec.b, i));
          r = __double2ull_rz(__dmul_rn(u, scale));
        } else {
          const uint32_t s = a.D[rec.di];
          const uint64_t h2 = hstep(z2p, s);
          u = smooth_finish(v, hstep(rec.b, i), hstep(h2, i));
          const double y = __dmul_rn(u, scale);
          const double fr = y - floor(y + 0.5);
          r = __double2ull_rz(y);
          if (fabs(fr) <= v.guard * y && y >= 0.5) r = ns_in_band(v, a.layer, s, i, u, r, uncert);
        }
        if (r < k) {
          const uint64_t pos = rec.a + r;
          if (pos < a.cap_edges) atomicMax(&a.slots[pos], static_cast<uint32_t>(i));
        }
      }
    }
  }
  if (smooth) {
    uncert = warp_sum(uncert);
    if (lane_id() == 0 && uncert) atomicAdd(&meta->uncertified, uncert);
  }
}

// Emit NS edges, tiled by dst (each dst owns <= k outputs): rows with d<=k
// copy N(s) in CSR order; hubs read N(s)[slots[j]] in slot order.
constexpr int kEmitDst = 256;
__global__ void __launch_bounds__(kNT) ns_emit_kernel(
    const uint32_t* __restrict__ D, const LayerMeta* meta,
    const uint64_t* __restrict__ out_prefix, const uint64_t* __restrict__ indptr,
    const uint32_t* __restrict__ indices, uint32_t k, const uint32_t* __restrict__ slots,
    uint32_t* bits, uint32_t* summ, uint2* edges, uint64_t cap_edges) {
  pdl_begin();
  __shared__ uint64_t s_op[kEmitDst + 1];
  __shared__ uint64_t s_rs[kEmitDst];
  __shared__ uint32_t s_d[kEmitDst];
  const uint64_t n_dst = meta->n_dst;
  if (meta->n_edges > cap_edges) return;
  const uint64_t ntiles = (n_dst + kEmitDst - 1) / kEmitDst;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t d0 = tile * kEmitDst;
    const int cnt = static_cast<int>(min(static_cast<uint64_t>(kEmitDst), n_dst - d0));
    __syncthreads();
    for (int i = threadIdx.x; i <= cnt; i += kNT) s_op[i] = out_prefix[d0 + i];
    for (int i = threadIdx.x; i < cnt; i += kNT) {
      const uint32_t s = D[d0 + i];
      const uint64_t b = indptr[s];
      s_rs[i] = b;
      s_d[i] = static_cast<uint32_t>(indptr[s + 1] - b);
    }
    __syncthreads();
    const uint64_t xe = s_op[cnt];
    for (uint64_t x = s_op[0] + threadIdx.x; x < xe; x += kNT) {
      const int li = seg_search(s_op, 0, cnt, x);
      const uint64_t q = x - s_op[li];
      const uint64_t pos = (s_d[li] <= k) ? q : slots[x];
      const uint32_t t = __ldg(indices + s_rs[li] + pos);
      edges[x] = make_uint2(t, static_cast<uint32_t>(d0 + li));
      set_bit(bits, summ, t);
    }
  }
}

// -------------------------------------------------------------------- RW --
// rw_block (samplers.cpp:202-285): per dst s, rw_walks walks of rw_length
// steps; step j of walk w draws u = U(hash(hash(prefix{3, layer, s}, w), j))
// (smoothed when kappa says so); after the first step a restart coin takes the
// [0,p) slice and the remainder is rescaled; the next vertex is
// indices[beg + (u64)(u*d)]; visits of s itself are not counted; the k most
// visited vertices (ties: smaller id) become the dst's edges, in rank order.
// One warp per dst: lane-strided walks, the visits sorted in shared memory,
// top-k by warp arg-max rounds.
constexpr int kRwWarps = kNT / 32;

template <bool SMOOTH>
__global__ void __launch_bounds__(kNT) rw_walk_kernel(RwArgs a) {
  pdl_begin();
  constexpr uint32_t kDead = 0xfffffffeu, kNone = 0xffffffffu;
  __shared__ uint32_t s_vis[kRwWarps][kRwMaxVisits];  // visit of (step, walk); then ids
  __shared__ uint32_t s_key[kRwWarps][kRwMaxVisits];  // sorted visited ids
  __shared__ uint16_t s_cc[kRwWarps][kRwMaxVisits];   // visit count per candidate
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  uint32_t* vis = s_vis[wib];
  uint32_t* key = s_key[wib];
  uint16_t* cc = s_cc[wib];
  const uint64_t n = a.meta->n_dst;
  const Variates v = *a.var;
  const uint64_t z1p = hstep(hstep(hinit(v.z1), 3ULL), static_cast<uint64_t>(a.layer));
  const uint64_t z2p = SMOOTH ? hstep(hstep(hinit(v.z2), 3ULL), static_cast<uint64_t>(a.layer))
                              : 0ULL;
  const uint32_t nv = a.walks * a.length;
  const double p = a.restart;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kRwWarps;
  for (uint64_t di = static_cast<uint64_t>(blockIdx.x) * kRwWarps + wib; di < n; di += nw) {
    const uint32_t s = a.D[di];
    const uint64_t h1 = hstep(z1p, s), h2 = SMOOTH ? hstep(z2p, s) : 0ULL;
    // round-major walks (samplers.cpp:228-260); the walk's current vertex is
    // its previous visit, kDead once it hit a dead end
    for (uint32_t j = 0; j < a.length; ++j) {
      for (uint32_t w = lane; w < a.walks; w += 32) {
        const uint32_t cur = (j == 0) ? s : vis[(j - 1) * a.walks + w];
        uint32_t out = kDead;
        if (cur != kDead) {
          const uint64_t b1 = hstep(hstep(h1, w), j);
          double u = SMOOTH ? smooth_finish(v, b1, hstep(hstep(h2, w), j)) : ufb(b1);
          uint32_t from = cur;
          if (j > 0 && p > 0.0) {
            if (u < p) {
              from = s;
              u = __ddiv_rn(u, p);
            } else {
              u = __ddiv_rn(__dsub_rn(u, p), __dsub_rn(1.0, p));
            }
          }
          const uint64_t beg = __ldg(a.indptr + from);
          const uint64_t d = __ldg(a.indptr + from + 1) - beg;
          if (d != 0 && a.weights) {
            // pick_neighbor (samplers.cpp:139-165): cdf[i] = weights summed in
            // f64 in CSR order, x = u * cdf.back(), first i with cdf[i] > x
            double tot = 0.0;
            for (uint64_t i = 0; i < d; ++i)
              tot = __dadd_rn(tot, static_cast<double>(__ldg(a.weights + beg + i)));
            const double x = __dmul_rn(u, tot);
            double acc = 0.0;
            uint64_t idx = d - 1;
            for (uint64_t i = 0; i < d; ++i) {
              acc = __dadd_rn(acc, static_cast<double>(__ldg(a.weights + beg + i)));
              if (acc > x) {
                idx = i;
                break;
              }
            }
            out = __ldg(a.indices + beg + idx);
          } else if (d != 0) {
            uint64_t idx = __double2ull_rz(__dmul_rn(u, static_cast<double>(d)));
            if (idx >= d) idx = d - 1;
            out = __ldg(a.indices + beg + idx);
          }
        }
        vis[j * a.walks + w] = out;
      }
      __syncwarp();
    }
    // counted visits: every next != s (samplers.cpp:258)
    for (uint32_t i = lane; i < kRwMaxVisits; i += 32) {
      const uint32_t x = i < nv ? vis[i] : kNone;
      key[i] = (x == s || x == kDead) ? kNone : x;
    }
    __syncwarp();
    // bitonic sort (ascending), whole warp
    for (uint32_t size = 2; size <= kRwMaxVisits; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t t = lane; t < kRwMaxVisits / 2; t += 32) {
          const uint32_t i = 2 * t - (t & (stride - 1));
          const uint32_t jj = i + stride;
          const bool up = ((i & size) == 0);
          const uint32_t x = key[i], y = key[jj];
          if ((x > y) == up) {
            key[i] = y;
            key[jj] = x;
          }
        }
        __syncwarp();
      }
    }
    // distinct ids with their visit counts, compacted (ids -> vis, counts -> cc)
    uint32_t ncand = 0;
    for (uint32_t base = 0; base < kRwMaxVisits; base += 32) {
      const uint32_t i = base + lane;
      const uint32_t x = key[i];
      const bool start = x != kNone && (i == 0 || key[i - 1] != x);
      uint32_t c = 0;
      if (start) {
        uint32_t e = i + 1;
        while (e < kRwMaxVisits && key[e] == x) ++e;
        c = e - i;
      }
      const unsigned m = __ballot_sync(0xffffffffu, start);
      if (start) {
        const uint32_t pos = ncand + __popc(m & lanemask_lt());
        vis[pos] = x;
        cc[pos] = static_cast<uint16_t>(c);
      }
      ncand += __popc(m);
    }
    __syncwarp();
    // top-k by (count desc, id asc) (samplers.cpp:271-281), rank order
    const uint32_t take = min(a.k, ncand);
    for (uint32_t r = 0; r < take; ++r) {
      uint32_t bc = 0, bid = kNone, bpos = kNone;
      for (uint32_t q = lane; q < ncand; q += 32) {
        const uint32_t c = cc[q], id = vis[q];
        if (c > bc || (c == bc && c > 0 && id < bid)) {
          bc = c;
          bid = id;
          bpos = q;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const uint32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
        const uint32_t op = __shfl_xor_sync(0xffffffffu, bpos, o);
        if (oc > bc || (oc == bc && oid < bid)) {
          bc = oc;
          bid = oid;
          bpos = op;
        }
      }
      __syncwarp();  // every lane's reads of cc[] precede the write below
      if (lane == 0) {
        a.slots[di * a.k + r] = bid;
        cc[bpos] = 0;  // taken
        set_bit(a.bits, a.summ, bid);
      }
      __syncwarp();
    }
    if (lane == 0) a.cnt[di] = take;
    __syncwarp();
  }
}

// Edges of the RW picks in dst order (ordered compaction of the per-dst
// counts, decoupled look-back), rank order inside a dst.
__global__ void __launch_bounds__(kNT) rw_emit_kernel(RwArgs a) {
  pdl_begin();
  __shared__ unsigned long long s_scan[kNT / 32 + 1];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  constexpr int IPT = 4;
  constexpr int TILE = kNT * IPT;
  const uint64_t n = a.meta->n_dst;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const unsigned ep = inv_epoch(a.epoch, a.slot);
  for (unsigned tile = blockIdx.x; tile < ntiles;
       tile = next_tile_after(a.ticket, &s_tile, gridDim.x, ntiles)) {
    const uint64_t i0 = static_cast<uint64_t>(tile) * TILE + threadIdx.x * IPT;
    uint64_t c[IPT];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      c[j] = (i0 + j < n) ? a.cnt[i0 + j] : 0;
      sum += c[j];
    }
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<kNT>(sum, s_scan, tot);
    const unsigned long long gb = tile_prefix<4>(a.status, tile, tot, ep, &s_b);
    unsigned long long pos = gb + ex;
#pragma unroll
    for (int j = 0; j < IPT; ++j)
      for (uint64_t r = 0; r < c[j]; ++r, ++pos)
        if (pos < a.cap_edges)
          a.edges[pos] = make_uint2(a.slots[(i0 + j) * a.k + r], static_cast<uint32_t>(i0 + j));
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      a.meta->n_edges = gb + tot;
      if (gb + tot > a.cap_edges) atomicExch(a.overflow, 1u);
    }
  }
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) a.meta->n_edges = 0;
}

// ---------------------------------------------------------------- extract --
// Sorted unique list = set bits in id order; wprefix[w] = rank of word w.
// Words per thread: 2 for small bitmaps (more tiles, short per-thread
// serial bit loops), 8 (two 16 B loads) once the bitmap exceeds 256K words,
// so the look-back chain stays ~ <2K tiles even at 10^8 vertices.
constexpr int kWPTSmall = 2;  // the flat path loads word pairs
constexpr int kWPTBig = 8;
static_assert(kNT * kWPTBig == kExtractTileWords, "extract tile");

__device__ __forceinline__ void extract_flat(const ExtractArgs& a, unsigned role,
                                             unsigned ncta) {
  __shared__ unsigned long long s_scan[kNT / 32 + 1];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  const int wpt = a.words_padded > kExtractBigWords ? kWPTBig : kWPTSmall;
  const uint32_t tw = kNT * wpt;
  const uint64_t ntiles = a.words_padded / tw;
  const unsigned ep = inv_epoch(a.epoch, a.slot);
  unsigned long long* tr = role < 32 ? a.trace : nullptr;
  tstamp(tr, role, 0);
  for (unsigned tile = role; tile < ntiles; tile = next_tile_after(a.ticket, &s_tile, ncta, ntiles)) {
    const uint64_t w0 = static_cast<uint64_t>(tile) * tw + threadIdx.x * wpt;
    uint32_t wv[kWPTBig];
    if (wpt == kWPTBig) {
      const uint4 x = *reinterpret_cast<const uint4*>(a.bits + w0);
      const uint4 y = *reinterpret_cast<const uint4*>(a.bits + w0 + 4);
      wv[0] = x.x; wv[1] = x.y; wv[2] = x.z; wv[3] = x.w;
      wv[4] = y.x; wv[5] = y.y; wv[6] = y.z; wv[7] = y.w;
      if (a.zero_bits) {
        *reinterpret_cast<uint4*>(a.zero_bits + w0) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(a.zero_bits + w0 + 4) = make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      const uint2 x = *reinterpret_cast<const uint2*>(a.bits + w0);
      wv[0] = x.x; wv[1] = x.y;
#pragma unroll
      for (int j = 2; j < kWPTBig; ++j) wv[j] = 0u;
      if (a.zero_bits) *reinterpret_cast<uint2*>(a.zero_bits + w0) = make_uint2(0u, 0u);
    }
    if (a.zero_summ && threadIdx.x < tw / 32)
      a.zero_summ[static_cast<uint64_t>(tile) * (tw / 32) + threadIdx.x] = 0u;
    unsigned long long c = 0;
#pragma unroll
    for (int j = 0; j < kWPTBig; ++j) c += __popc(wv[j]);
    if (tile == role) tstamp(tr, role, 1);
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<kNT>(c, s_scan, tot);
    if (tile == role) tstamp(tr, role, 2);
    const unsigned long long gb = tile_prefix<4>(a.status, tile, tot, ep, &s_b);
    if (tile == role) tstamp(tr, role, 3);
    unsigned long long pos = gb + ex;
    uint32_t pw[kWPTBig];
#pragma unroll
    for (int j = 0; j < kWPTBig; ++j) {
      pw[j] = static_cast<uint32_t>(pos);
      uint32_t x = wv[j];
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        if (pos < a.cap_out) a.out[pos] = static_cast<uint32_t>((w0 + j) * 32 + bit);
        ++pos;
      }
    }
    if (wpt == kWPTBig) {
      *reinterpret_cast<uint4*>(a.wprefix + w0) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
      *reinterpret_cast<uint4*>(a.wprefix + w0 + 4) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
    } else {
      *reinterpret_cast<uint2*>(a.wprefix + w0) = make_uint2(pw[0], pw[1]);
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      *a.count_out = gb + tot;
      if (a.count_out2) *a.count_out2 = gb + tot;
      if (gb + tot > a.cap_out) atomicExch(a.overflow, 1u);
    }
  }
  tstamp(tr, role, 4);
  tlast(a.trace);
}

// Summary-driven extraction for large bitmaps: a tile is kNT summary words
// (8K data words); threads visit only data words whose summary bit is set,
// so the cost follows the frontier, not n. The zeroing of the previous
// layer's bitmap likewise walks its own summary.
__device__ __forceinline__ void extract_summ(const ExtractArgs& a, unsigned role,
                                             unsigned ncta) {
  __shared__ unsigned long long s_scan[kNT / 32 + 1];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  const uint64_t swords = a.words_padded / 32;
  const uint64_t ntiles = (swords + kNT - 1) / kNT;
  const unsigned ep = inv_epoch(a.epoch, a.slot);
  unsigned long long* tr = role < 32 ? a.trace : nullptr;
  tstamp(tr, role, 0);
  for (unsigned tile = role; tile < ntiles; tile = next_tile_after(a.ticket, &s_tile, ncta, ntiles)) {
    const uint64_t sw = static_cast<uint64_t>(tile) * kNT + threadIdx.x;
    const uint32_t sm = sw < swords ? a.summ[sw] : 0u;
    if (a.zero_summ && sw < swords) {
      uint32_t z = a.zero_summ[sw];
      while (z) {
        const int j = __ffs(z) - 1;
        z &= z - 1;
        a.zero_bits[sw * 32 + j] = 0u;
      }
      a.zero_summ[sw] = 0u;
    }
    unsigned long long c = 0;
    {
      uint32_t m = sm;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        c += __popc(a.bits[sw * 32 + j]);
      }
    }
    if (tile == role) tstamp(tr, role, 1);
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<kNT>(c, s_scan, tot);
    if (tile == role) tstamp(tr, role, 2);
    const unsigned long long gb = tile_prefix<4>(a.status, tile, tot, ep, &s_b);
    if (tile == role) tstamp(tr, role, 3);
    unsigned long long pos = gb + ex;
    uint32_t m = sm;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t w = sw * 32 + j;
      uint32_t x = a.bits[w];
      a.wprefix[w] = static_cast<uint32_t>(pos);
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        if (pos < a.cap_out) a.out[pos] = static_cast<uint32_t>(w * 32 + bit);
        ++pos;
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      *a.count_out = gb + tot;
      if (a.count_out2) *a.count_out2 = gb + tot;
      if (gb + tot > a.cap_out) atomicExch(a.overflow, 1u);
    }
  }
  tstamp(tr, role, 4);
  tlast(a.trace);
}

__device__ __forceinline__ bool extract_uses_summary(const ExtractArgs& a) {
  return a.words_padded > kExtractBigWords;
}

__device__ __forceinline__ void extract_body(const ExtractArgs& a, unsigned role,
                                             unsigned ncta) {
  if (extract_uses_summary(a)) extract_summ(a, role, ncta);
  else extract_flat(a, role, ncta);
}

__global__ void __launch_bounds__(kNT) extract_kernel(ExtractArgs a) {
  pdl_begin();
  extract_body(a, blockIdx.x, gridDim.x);
}

// Extract (dedup of the layer) and the ordered LABOR edge emission only
// depend on labor_mark, not on each other: one launch, CTAs split by role.
__global__ void __launch_bounds__(kNT) post_kernel(ExtractArgs e, LaborArgs a, unsigned n_ext) {
  pdl_begin();
  if (blockIdx.x < n_ext) extract_body(e, blockIdx.x, n_ext);
  else labor_emit_body(a, blockIdx.x - n_ext, gridDim.x - n_ext, e.trace);
}

// ---------------------------------------------------------------- relabel --
__global__ void relabel_kernel(RelabelArgs r) {
  pdl_begin();
  relabel_range(r, blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
                static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void rank_kernel(const uint32_t* __restrict__ bits,
                            const uint32_t* __restrict__ wprefix,
                            const uint32_t* __restrict__ ids,
                            const unsigned long long* count, uint32_t* out) {
  pdl_begin();
  const uint64_t n = *count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    out[i] = bm_rank(bits, wprefix, ids[i]);
}

__global__ void clear_kernel(uint32_t* bits, uint32_t* summ, const uint32_t* __restrict__ list,
                             const unsigned long long* count) {
  pdl_begin();
  const uint64_t n = *count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const uint32_t v = list[i];
    bits[v >> 5] = 0u;
    if (summ) summ[v >> 10] = 0u;
  }
}

constexpr int kLaborIPT = kLaborTile / kNT;      // NS reservoir tiles
constexpr int kMarkIPT = kLaborTile / kMarkNT;   // labor_mark

}  // namespace

uint64_t extract_tiles(uint64_t words_padded) {
  if (words_padded > kExtractBigWords) return (words_padded / 32 + kNT - 1) / kNT;
  return words_padded / (kNT * kWPTSmall);
}

// Resident CTAs per SM of a kernel at kNT threads (cached per function).
template <typename K>
int resident_per_sm(K kernel, size_t smem = 0) {
  static std::unordered_map<const void*, int> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(reinterpret_cast<const void*>(kernel));
  if (it != cache.end()) return it->second;
  int n = 0;
  CB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kNT, smem));
  n = std::max(1, n);
  cache.emplace(reinterpret_cast<const void*>(kernel), n);
  return n;
}

int grid_for(uint64_t work_items, int per_block, int max_per_sm) {
  const uint64_t blocks = (work_items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(kNumSMs) * max_per_sm;
  return static_cast<int>(std::max<uint64_t>(1, std::min(blocks, cap)));
}

void launch_batch_begin(const Sync& s, uint32_t* clear_bits, uint32_t* clear_summ,
                        const uint32_t* clear_list, const unsigned long long* clear_count,
                        uint64_t clear_cap, uint64_t nwords, cudaStream_t st) {
  const int grid = grid_for(clear_cap, 256, 4);
  launch_k(batch_begin_kernel, grid, 256, st, s.epoch, s.overflow, s.tickets, Sync::kMaxTickets,
                                           clear_bits, clear_summ, clear_list, clear_count,
                                           clear_cap, nwords);
  CB_LAUNCH("batch_begin");
}

void launch_frontier(const FrontierArgs& a, const RelabelArgs& r, uint64_t cap_dst,
                     uint64_t relabel_work, cudaStream_t st) {
  const int occ = resident_per_sm(frontier_kernel<kFrontierIPT>);
  const int fgrid = grid_for(cap_dst, kNT * kFrontierIPT, occ);
  const int rgrid = r.edges ? grid_for(relabel_work, kNT * 4, occ) : 0;
  launch_k(frontier_kernel<kFrontierIPT>, fgrid + rgrid, kNT, st, a, r,
           static_cast<unsigned>(fgrid));
  CB_LAUNCH("frontier");
}

void launch_labor(const LaborArgs& a, uint64_t max_tiles, bool smooth, cudaStream_t st) {
  if (smooth && a.kind != 0 && a.vtab && a.n_vert) {
    launch_k(vtab_kernel, grid_for(a.n_vert, kNT, 8), kNT, st, a);
    CB_LAUNCH("vtab");
  }
  const int grid = grid_for(max_tiles * kLaborTile, kLaborTile, kMarkCtasPerSM);
  static const bool attrs_set = [] {
    CB_CUDA(cudaFuncSetAttribute(labor_mark_kernel<kMarkIPT, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(mark_smem_bytes(true))));
    CB_CUDA(cudaFuncSetAttribute(labor_mark_kernel<kMarkIPT, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(mark_smem_bytes(false))));
    return true;
  }();
  (void)attrs_set;
  if (smooth && a.kind != 0)
    launch_ks(labor_mark_kernel<kMarkIPT, true>, grid, kMarkNT, mark_smem_bytes(true), st, a);
  else
    launch_ks(labor_mark_kernel<kMarkIPT, false>, grid, kMarkNT, mark_smem_bytes(false), st, a);
  CB_LAUNCH("labor_mark");
}

void launch_labor_post(const LaborArgs& a, uint64_t max_tiles, const ExtractArgs& e,
                       cudaStream_t st) {
  const uint64_t words = (max_tiles * kLaborTile + 31) / 32;
  const int occ = resident_per_sm(post_kernel);
  // both roles share the resident capacity: extract gets what its tiles need
  // (up to half), emit the rest
  const int cap = occ * kNumSMs;
  const int g_ext = std::min(grid_for(extract_tiles(e.words_padded), 1, occ), cap / 2);
  const int g_emit = std::min(grid_for(words, kEmitTileWords, occ), cap - g_ext);
  launch_k(post_kernel, g_emit + g_ext, kNT, st, e, a, static_cast<unsigned>(g_ext));
  CB_LAUNCH("post");
}

void launch_ns(const LaborArgs& a, const uint32_t* D, const uint64_t* out_prefix,
               const uint64_t* indptr, const uint32_t* indices, uint64_t cap_dst, bool smooth,
               cudaStream_t st) {
  if (smooth) launch_k(ns_reservoir_kernel<kLaborIPT, true>, kNumSMs * 8, kNT, st, a);
  else launch_k(ns_reservoir_kernel<kLaborIPT, false>, kNumSMs * 8, kNT, st, a);
  CB_LAUNCH("ns_reservoir");
  const int grid = grid_for(cap_dst, kEmitDst, 8);
  launch_k(ns_emit_kernel, grid, kNT, st, D, a.meta, out_prefix, indptr, indices, a.k, a.slots,
                                       a.bits, a.summ, a.edges, a.cap_edges);
  CB_LAUNCH("ns_emit");
}

void launch_rw(const RwArgs& a, uint64_t cap_dst, bool smooth, cudaStream_t st) {
  const int grid = grid_for(cap_dst, kRwWarps, 4);
  if (smooth) launch_k(rw_walk_kernel<true>, grid, kNT, st, a);
  else launch_k(rw_walk_kernel<false>, grid, kNT, st, a);
  CB_LAUNCH("rw_walk");
  launch_k(rw_emit_kernel, grid_for(cap_dst, kNT * 4, resident_per_sm(rw_emit_kernel)), kNT, st,
           a);
  CB_LAUNCH("rw_emit");
}

void launch_extract(const ExtractArgs& a, cudaStream_t st) {
  const int grid = grid_for(extract_tiles(a.words_padded), 1, resident_per_sm(extract_kernel));
  launch_k(extract_kernel, grid, kNT, st, a);
  CB_LAUNCH("extract");
}

void launch_relabel(const RelabelArgs& r, uint64_t work, cudaStream_t st) {
  const int grid = grid_for(work, 256 * 4, 8);
  launch_k(relabel_kernel, grid, 256, st, r);
  CB_LAUNCH("relabel");
}

void launch_rank(const Bitmap& bm, const uint32_t* ids, const unsigned long long* count,
                 uint32_t* rank_out, cudaStream_t st) {
  launch_k(rank_kernel, kNumSMs * 4, 256, st, bm.bits, bm.wprefix, ids, count, rank_out);
  CB_LAUNCH("rank");
}

void launch_clear(Bitmap& bm, const uint32_t* list, const unsigned long long* count,
                  cudaStream_t st) {
  launch_k(clear_kernel, kNumSMs * 4, 256, st, bm.bits, bm.summ, list, count);
  CB_LAUNCH("clear");
}

}  // namespace cb
