// Frontier expansion kernels: one layer of LABOR-0 / NS / FULL sampling
// (samplers.cpp:62-136, 289-296) plus the bitmap dedup/relabel that replaces
// BlockBuilder::finish (samplers.cpp:28-54).
//
// Per layer the pipeline is
//   frontier  : degree scan of D (scan-space prefix), marks D in the bitmap,
//               clears the previous layer's bitmap words, NS slot init
//   labor/ns  : scan-space tiles over all neighbour positions; keep rule /
//               reservoir; order-preserving compaction via ballot + decoupled
//               look-back (edges land grouped by dst, CSR order inside a dst,
//               slot order for NS hubs — exactly the reference order);
//               kept ids are OR-ed into the bitmap
//   extract   : bitmap popcount scan -> sorted unique src list + word ranks
//   relabel   : edge (t, di) -> (rank(t), di); dst_pos = rank(D)
// No host synchronisation: every count lives in device LayerMeta and all
// kernels are persistent (ticketed) loops bounded by those counts.
#include "cb_internal.h"

namespace cb {
using namespace cbdev;

namespace {

constexpr int kNT = 256;

__device__ __forceinline__ unsigned inv_epoch(const unsigned* ep, int slot) {
  return ((*ep & 0x3ffffu) << 6) | static_cast<unsigned>(slot);
}

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t v) {
  atomicOr(&bits[v >> 5], 1u << (v & 31u));
}

__device__ __forceinline__ uint32_t bm_rank(const uint32_t* bits, const uint32_t* wprefix,
                                            uint32_t v) {
  const uint32_t w = v >> 5;
  return wprefix[w] + __popc(bits[w] & ((1u << (v & 31u)) - 1u));
}

// ------------------------------------------------------------ batch begin --
__global__ void batch_begin_kernel(unsigned* epoch, unsigned* tickets, int n_tickets,
                                   LayerMeta* meta, int n_meta, unsigned long long n_seeds,
                                   unsigned* overflow) {
  const int t = threadIdx.x;
  if (t == 0) {
    *epoch = *epoch + 1;
    *overflow = 0;
  }
  for (int i = t; i < n_tickets; i += blockDim.x) tickets[i] = 0;
  for (int i = t; i < n_meta * 8; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(meta)[i] = 0;
  __syncthreads();
  if (t == 0) meta[0].n_dst = n_seeds;
}

// ---------------------------------------------------------------- frontier --
// kind: 0 FULL, 1 NS, 2 LABOR0 (samplers.hpp:15). Per dst: scan work q
// (LABOR/FULL: d; NS: reservoir positions max(d-k,0)), active flag q>0 and,
// for NS, the output count min(d,k). Three look-back scans give the active
// list (bounded dsts per scan tile), its scan prefix and the NS out prefix.
template <int IPT>
__global__ void __launch_bounds__(kNT) frontier_kernel(
    const uint32_t* __restrict__ D, LayerMeta* meta, const uint64_t* __restrict__ indptr,
    int kind, uint32_t k, uint32_t* set_bits, uint32_t* clear_bits, uint32_t* act_di,
    uint64_t* act_pre, uint64_t* out_prefix, uint32_t* slots, uint64_t cap_edges,
    unsigned* ticket, unsigned long long* st_a, unsigned long long* st_b,
    unsigned long long* st_c, const unsigned* epoch_p, int slot, unsigned* overflow) {
  __shared__ unsigned long long s_scan[3][kNT / 32 + 1];
  __shared__ unsigned long long s_bc[3];
  __shared__ unsigned s_tile;
  const uint64_t n = meta->n_dst;
  constexpr int TILE = kNT * IPT;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const bool is_ns = (kind == 1);
  for (unsigned tile = next_tile(ticket, &s_tile); tile < ntiles;
       tile = next_tile(ticket, &s_tile)) {
    const uint64_t i0 = static_cast<uint64_t>(tile) * TILE + threadIdx.x * IPT;
    unsigned long long q[IPT], o[IPT];
    unsigned long long qs = 0, as = 0, os = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t i = i0 + j;
      q[j] = o[j] = 0;
      if (i < n) {
        const uint32_t v = D[i];
        const uint64_t d = indptr[v + 1] - indptr[v];
        set_bit(set_bits, v);
        if (clear_bits) clear_bits[v >> 5] = 0u;
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
    unsigned long long tq, ta, to = 0;
    unsigned long long eq = block_exclusive_scan<kNT>(qs, s_scan[0], tq);
    unsigned long long ea = block_exclusive_scan<kNT>(as, s_scan[1], ta);
    unsigned long long eo = 0;
    if (is_ns) eo = block_exclusive_scan<kNT>(os, s_scan[2], to);
    const unsigned long long bq = tile_prefix(st_a, tile, tq, inv_epoch(epoch_p, slot), &s_bc[0]);
    const unsigned long long ba =
        tile_prefix(st_b, tile, ta, inv_epoch(epoch_p, slot + 1), &s_bc[1]);
    unsigned long long bo = 0;
    if (is_ns) bo = tile_prefix(st_c, tile, to, inv_epoch(epoch_p, slot + 2), &s_bc[2]);
    eq += bq;
    ea += ba;
    eo += bo;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t i = i0 + j;
      if (i < n) {
        if (q[j] > 0) {
          act_di[ea] = static_cast<uint32_t>(i);
          act_pre[ea] = eq;
          ++ea;
        }
        if (is_ns) {
          out_prefix[i] = eo;
          if (q[j] > 0 && eo + k <= cap_edges)  // hub: slots start as identity
            for (uint32_t r = 0; r < k; ++r) slots[eo + r] = r;
        }
      }
      eq += q[j];
      eo += o[j];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      act_pre[ba + ta] = bq + tq;
      meta->scan_total = bq + tq;
      meta->n_active = ba + ta;
      if (is_ns) {
        out_prefix[n] = bo + to;
        meta->n_edges = bo + to;
        if (bo + to > cap_edges) atomicExch(overflow, 1u);
      }
    }
  }
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    act_pre[0] = 0;
    if (is_ns) out_prefix[0] = 0;
  }
}

// ---------------------------------------------------------- segment tiles --
// Active entries [a0, a1] covering scan positions [x0, x1): at most
// x1-x0 entries because every active dst owns >= 1 position.
__device__ __forceinline__ void tile_segment(const uint64_t* prefix, uint64_t n_act,
                                             uint64_t x0, uint64_t x1, int* s_range) {
  if (threadIdx.x == 0) {
    int lo = 0, hi = static_cast<int>(n_act);
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= x0) lo = mid;
      else hi = mid;
    }
    s_range[0] = lo;
    int lo2 = lo;
    hi = static_cast<int>(n_act);
    while (hi - lo2 > 1) {
      const int mid = (lo2 + hi) >> 1;
      if (prefix[mid] <= x1 - 1) lo2 = mid;
      else hi = mid;
    }
    s_range[1] = lo2;
  }
  __syncthreads();
}

// ------------------------------------------------------------- LABOR/FULL --
// keep(t -> s) iff U(hash(z1,{2,layer,t})) <= k/d_s  (samplers.cpp:117-134);
// plain stream compared in integers: (h>>11) <= floor((k/d)*2^53), exact.
template <int IPT>
__global__ void __launch_bounds__(kNT) labor_kernel(
    const uint32_t* __restrict__ D, LayerMeta* meta, const uint32_t* __restrict__ act_di,
    const uint64_t* __restrict__ act_pre, const uint64_t* __restrict__ indptr,
    const uint32_t* __restrict__ indices, int kind, uint32_t k, int layer,
    const Variates* __restrict__ var, uint32_t* bits, uint2* edges, uint64_t cap_edges,
    unsigned* ticket, unsigned long long* status, const unsigned* epoch_p, int slot,
    unsigned* overflow) {
  constexpr int TILE = kNT * IPT;
  constexpr int NW = kNT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_dp = reinterpret_cast<uint64_t*>(smem_raw);  // [TILE+1]
  uint64_t* s_rs = s_dp + (TILE + 1);                      // [TILE]
  uint64_t* s_th = s_rs + TILE;                            // [TILE]
  uint32_t* s_di = reinterpret_cast<uint32_t*>(s_th + TILE);  // [TILE]
  __shared__ unsigned s_cnt[IPT * NW];
  __shared__ unsigned s_base[IPT * NW];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  __shared__ int s_range[2];
  __shared__ unsigned s_total;

  const uint64_t total = meta->scan_total;
  const uint64_t n_act = meta->n_active;
  const uint64_t ntiles = (total + TILE - 1) / TILE;
  const unsigned ep = inv_epoch(epoch_p, slot);
  const Variates v = *var;
  const bool full = (kind == 0);
  const bool smooth = v.smoothed != 0 && !full;
  // prefix({kStreamLabor, layer}) under z1 (and z2 when smoothed)
  const uint64_t p1 = hstep(hstep(hinit(v.z1), 2ULL), static_cast<uint64_t>(layer));
  const uint64_t p2 = hstep(hstep(hinit(v.z2), 2ULL), static_cast<uint64_t>(layer));
  const unsigned w = threadIdx.x >> 5;
  unsigned long long uncert = 0;

  for (unsigned tile = next_tile(ticket, &s_tile); tile < ntiles;
       tile = next_tile(ticket, &s_tile)) {
    const uint64_t x0 = static_cast<uint64_t>(tile) * TILE;
    const uint64_t x1 = min(x0 + TILE, total);
    tile_segment(act_pre, n_act, x0, x1, s_range);
    const int a0 = s_range[0];
    const int nd = s_range[1] - a0 + 1;
    for (int i = threadIdx.x; i <= nd; i += kNT) s_dp[i] = act_pre[a0 + i];
    __syncthreads();
    for (int i = threadIdx.x; i < nd; i += kNT) {
      const uint32_t di = act_di[a0 + i];
      const uint32_t s = D[di];
      s_di[i] = di;
      s_rs[i] = indptr[s] - s_dp[i];  // indices[s_rs + x] is the neighbour at x
      const uint64_t d = s_dp[i + 1] - s_dp[i];
      if (full) {
        s_th[i] = ~0ULL;
      } else {
        const double thr = __ddiv_rn(static_cast<double>(k), static_cast<double>(d));
        if (smooth) s_th[i] = static_cast<uint64_t>(__double_as_longlong(thr));
        else s_th[i] = (d <= k) ? ~0ULL : __double2ull_rz(__dmul_rn(thr, 0x1.0p53));
      }
    }
    __syncthreads();

    uint32_t tv[IPT];
    uint32_t dv[IPT];
    unsigned keepmask = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t x = x0 + static_cast<uint64_t>(j) * kNT + threadIdx.x;
      bool keep = false;
      tv[j] = 0;
      dv[j] = 0;
      if (x < x1) {
        const int li = seg_search(s_dp, 0, nd, x);
        const uint32_t t = __ldg(indices + s_rs[li] + x);
        tv[j] = t;
        dv[j] = s_di[li];
        const uint64_t th = s_th[li];
        if (!smooth) {
          keep = (th == ~0ULL) || (hstep(p1, t) >> 11) <= th;
        } else {
          const double thr = __longlong_as_double(static_cast<long long>(th));
          if (thr >= 1.0) {
            keep = true;  // r < 1 always (phi of a finite normal)
          } else {
            const double r = smooth_finish(v, hstep(p1, t), hstep(p2, t));
            keep = r <= thr;
            if (fabs(r - thr) <= kGuard * thr) ++uncert;
          }
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane_id() == 0) s_cnt[j * NW + w] = __popc(bal);
      if (keep) keepmask |= 1u << j;
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan over IPT*NW (j-major) counters, 2 per lane
      constexpr int NC = IPT * NW;
      static_assert(NC <= 64, "scan width");
      const unsigned c0 = (2 * lane_id() < NC) ? s_cnt[2 * lane_id()] : 0u;
      const unsigned c1 = (2 * lane_id() + 1 < NC) ? s_cnt[2 * lane_id() + 1] : 0u;
      const unsigned inc = warp_inclusive_scan(c0 + c1);
      const unsigned ex = inc - c0 - c1;
      if (2 * lane_id() < NC) s_base[2 * lane_id()] = ex;
      if (2 * lane_id() + 1 < NC) s_base[2 * lane_id() + 1] = ex + c0;
      if (lane_id() == 31) s_total = inc;
    }
    __syncthreads();
    const unsigned agg = s_total;
    const unsigned long long gb = tile_prefix(status, tile, agg, ep, &s_b);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const bool keep = (keepmask >> j) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const unsigned long long pos = gb + s_base[j * NW + w] + __popc(bal & lanemask_lt());
        if (pos < cap_edges) edges[pos] = make_uint2(tv[j], dv[j]);
        set_bit(bits, tv[j]);
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      meta->n_edges = gb + agg;
      if (gb + agg > cap_edges) atomicExch(overflow, 1u);
    }
  }
  if (smooth) {
    uncert = warp_sum(uncert);
    if (lane_id() == 0 && uncert) atomicAdd(&meta->uncertified, uncert);
  }
}

// ---------------------------------------------------------------- NS -------
// Reservoir (samplers.cpp:75-84) restated per slot: the final content of slot
// j is the largest i in [k, d) with floor(U_i*(i+1)) == j, else j. Every
// position is an independent atomicMax, so hub rows split across CTAs.
template <int IPT>
__global__ void __launch_bounds__(kNT) ns_reservoir_kernel(
    const uint32_t* __restrict__ D, LayerMeta* meta, const uint32_t* __restrict__ act_di,
    const uint64_t* __restrict__ act_pre, const uint64_t* __restrict__ out_prefix,
    uint32_t k, int layer, const Variates* __restrict__ var, uint32_t* slots,
    uint64_t cap_edges) {
  constexpr int TILE = kNT * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_dp = reinterpret_cast<uint64_t*>(smem_raw);  // [TILE+1]
  uint64_t* s_op = s_dp + (TILE + 1);                      // [TILE]
  uint64_t* s_h1 = s_op + TILE;                            // [TILE]
  uint64_t* s_h2 = s_h1 + TILE;                            // [TILE]
  __shared__ int s_range[2];
  const uint64_t total = meta->scan_total;
  const uint64_t n_act = meta->n_active;
  const uint64_t ntiles = (total + TILE - 1) / TILE;
  const Variates v = *var;
  const bool smooth = v.smoothed != 0;
  const uint64_t z1p = hstep(hstep(hinit(v.z1), 1ULL), static_cast<uint64_t>(layer));
  const uint64_t z2p = hstep(hstep(hinit(v.z2), 1ULL), static_cast<uint64_t>(layer));
  unsigned long long uncert = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t x0 = tile * TILE;
    const uint64_t x1 = min(x0 + TILE, total);
    __syncthreads();
    tile_segment(act_pre, n_act, x0, x1, s_range);
    const int a0 = s_range[0];
    const int nd = s_range[1] - a0 + 1;
    for (int i = threadIdx.x; i <= nd; i += kNT) s_dp[i] = act_pre[a0 + i];
    for (int i = threadIdx.x; i < nd; i += kNT) {
      const uint32_t di = act_di[a0 + i];
      const uint32_t s = D[di];
      s_op[i] = out_prefix[di];
      s_h1[i] = hstep(z1p, s);  // prefix({kStreamNs, layer, s})
      s_h2[i] = smooth ? hstep(z2p, s) : 0;
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < IPT; ++j) {
      const uint64_t x = x0 + static_cast<uint64_t>(j) * kNT + threadIdx.x;
      if (x < x1) {
        const int li = seg_search(s_dp, 0, nd, x);
        const uint64_t i = k + (x - s_dp[li]);
        const double scale = static_cast<double>(i + 1);
        double u;
        if (!smooth) {
          u = ufb(hstep(s_h1[li], i));
        } else {
          u = smooth_finish(v, hstep(s_h1[li], i), hstep(s_h2[li], i));
          const double y = __dmul_rn(u, scale);
          const double fr = y - floor(y + 0.5);
          if (fabs(fr) <= kGuard * y && y >= 0.5) ++uncert;
        }
        const uint64_t r = __double2ull_rz(__dmul_rn(u, scale));
        if (r < k) {
          const uint64_t pos = s_op[li] + r;
          if (pos < cap_edges) atomicMax(&slots[pos], static_cast<uint32_t>(i));
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
    uint32_t* bits, uint2* edges, uint64_t cap_edges) {
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
      set_bit(bits, t);
    }
  }
}

// ---------------------------------------------------------------- extract --
// Sorted unique list = set bits in id order; wprefix[w] = rank of word w.
constexpr int kWPT = 8;  // words per thread (two 16-byte loads)
__global__ void __launch_bounds__(kNT) extract_kernel(
    const uint32_t* __restrict__ bits, uint32_t* wprefix, uint64_t words_padded,
    uint32_t* out, uint64_t cap_out, unsigned long long* count_out,
    unsigned long long* count_out2, unsigned* ticket, unsigned long long* status,
    const unsigned* epoch_p, int slot, unsigned* overflow) {
  __shared__ unsigned long long s_scan[kNT / 32 + 1];
  __shared__ unsigned long long s_b;
  __shared__ unsigned s_tile;
  constexpr int TILE = kNT * kWPT;
  const uint64_t ntiles = words_padded / TILE;
  const unsigned ep = inv_epoch(epoch_p, slot);
  for (unsigned tile = next_tile(ticket, &s_tile); tile < ntiles;
       tile = next_tile(ticket, &s_tile)) {
    const uint64_t w0 = static_cast<uint64_t>(tile) * TILE + threadIdx.x * kWPT;
    const uint4 a = *reinterpret_cast<const uint4*>(bits + w0);
    const uint4 b = *reinterpret_cast<const uint4*>(bits + w0 + 4);
    const uint32_t wv[kWPT] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    unsigned long long c = 0;
#pragma unroll
    for (int j = 0; j < kWPT; ++j) c += __popc(wv[j]);
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<kNT>(c, s_scan, tot);
    const unsigned long long gb = tile_prefix(status, tile, tot, ep, &s_b);
    unsigned long long pos = gb + ex;
    uint32_t pw[kWPT];
#pragma unroll
    for (int j = 0; j < kWPT; ++j) {
      pw[j] = static_cast<uint32_t>(pos);
      uint32_t x = wv[j];
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        if (pos < cap_out) out[pos] = static_cast<uint32_t>((w0 + j) * 32 + bit);
        ++pos;
      }
    }
    *reinterpret_cast<uint4*>(wprefix + w0) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    *reinterpret_cast<uint4*>(wprefix + w0 + 4) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      *count_out = gb + tot;
      if (count_out2) *count_out2 = gb + tot;
      if (gb + tot > cap_out) atomicExch(overflow, 1u);
    }
  }
}

// ---------------------------------------------------------------- relabel --
__global__ void relabel_kernel(const uint32_t* __restrict__ bits,
                               const uint32_t* __restrict__ wprefix, const LayerMeta* meta,
                               uint2* edges, uint64_t cap_edges,
                               const uint32_t* __restrict__ D, uint32_t* dst_pos) {
  const uint64_t ne = min(static_cast<uint64_t>(meta->n_edges), cap_edges);
  const uint64_t nd = meta->n_dst;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += stride) {
    uint2 x = edges[e];
    x.x = bm_rank(bits, wprefix, x.x);
    edges[e] = x;
  }
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nd;
       i += stride)
    dst_pos[i] = bm_rank(bits, wprefix, D[i]);
}

__global__ void rank_kernel(const uint32_t* __restrict__ bits,
                            const uint32_t* __restrict__ wprefix,
                            const uint32_t* __restrict__ ids,
                            const unsigned long long* count, uint32_t* out) {
  const uint64_t n = *count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    out[i] = bm_rank(bits, wprefix, ids[i]);
}

__global__ void clear_kernel(uint32_t* bits, const uint32_t* __restrict__ list,
                             const unsigned long long* count) {
  const uint64_t n = *count;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    bits[list[i] >> 5] = 0u;
}

constexpr int kFrontierIPT = 4;
constexpr int kLaborIPT = 4;
constexpr int kNsIPT = 4;

}  // namespace

int grid_for(uint64_t work_items, int per_block, int max_per_sm) {
  const uint64_t blocks = (work_items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(kNumSMs) * max_per_sm;
  return static_cast<int>(std::max<uint64_t>(1, std::min(blocks, cap)));
}

void launch_batch_begin(const Sync& s, LayerMeta* meta, int num_layers, uint64_t n_seeds,
                        cudaStream_t st) {
  batch_begin_kernel<<<1, 256, 0, st>>>(s.epoch, s.tickets, Sync::kMaxTickets, meta,
                                        num_layers, n_seeds, s.overflow);
  CB_LAUNCH("batch_begin");
}

void launch_frontier(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, int kind,
                     uint32_t fanout, Bitmap& set_bm, const Bitmap* clear_bm,
                     const Sync& s, int ticket, int epoch_slot, cudaStream_t st) {
  const int grid = grid_for(b.cap_dst, kNT * kFrontierIPT, 8);
  frontier_kernel<kFrontierIPT><<<grid, kNT, 0, st>>>(
      b.dst, meta, g.indptr, kind, fanout, set_bm.bits, clear_bm ? clear_bm->bits : nullptr,
      b.act_di, b.act_pre, b.out_prefix, b.slots, b.cap_edges, s.tickets + ticket,
      s.status_a, s.status_b, s.status_c, s.epoch, epoch_slot, s.overflow);
  CB_LAUNCH("frontier");
}

void launch_labor(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, int kind,
                  uint32_t fanout, int layer, const cbdev::Variates* var, Bitmap& bm,
                  const Sync& s, int ticket, int epoch_slot, cudaStream_t st) {
  constexpr int TILE = kNT * kLaborIPT;
  const size_t smem = (3 * TILE + 1) * sizeof(uint64_t) + TILE * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    CB_CUDA(cudaFuncSetAttribute(labor_kernel<kLaborIPT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int grid = grid_for(s.max_tiles * TILE, TILE, 6);
  labor_kernel<kLaborIPT><<<grid, kNT, smem, st>>>(
      b.dst, meta, b.act_di, b.act_pre, g.indptr, g.indices, kind, fanout, layer, var,
      bm.bits, b.edges, b.cap_edges, s.tickets + ticket, s.status_a, s.epoch, epoch_slot,
      s.overflow);
  CB_LAUNCH("labor");
}

void launch_ns(const DeviceGraph& g, const LayerBufs& b, LayerMeta* meta, uint32_t fanout,
               int layer, const cbdev::Variates* var, Bitmap& bm, cudaStream_t st) {
  constexpr int TILE = kNT * kNsIPT;
  const size_t smem_r = (4 * TILE + 1) * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    CB_CUDA(cudaFuncSetAttribute(ns_reservoir_kernel<kNsIPT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r));
    attr = true;
  }
  ns_reservoir_kernel<kNsIPT><<<kNumSMs * 4, kNT, smem_r, st>>>(
      b.dst, meta, b.act_di, b.act_pre, b.out_prefix, fanout, layer, var, b.slots,
      b.cap_edges);
  CB_LAUNCH("ns_reservoir");
  const int grid = grid_for(b.cap_dst, kEmitDst, 8);
  ns_emit_kernel<<<grid, kNT, 0, st>>>(b.dst, meta, b.out_prefix, g.indptr, g.indices,
                                       fanout, b.slots, bm.bits, b.edges, b.cap_edges);
  CB_LAUNCH("ns_emit");
}

void launch_extract(const Bitmap& bm, uint32_t* out, uint64_t cap_out,
                    unsigned long long* count_out, unsigned long long* count_out2,
                    const Sync& s, int ticket, int epoch_slot, cudaStream_t st) {
  const int grid = grid_for(bm.words_padded, kNT * kWPT, 8);
  extract_kernel<<<grid, kNT, 0, st>>>(bm.bits, bm.wprefix, bm.words_padded, out, cap_out,
                                       count_out, count_out2, s.tickets + ticket, s.status_a,
                                       s.epoch, epoch_slot, s.overflow);
  CB_LAUNCH("extract");
}

void launch_relabel(const Bitmap& bm, const LayerBufs& b, const LayerMeta* meta,
                    cudaStream_t st) {
  const int grid = grid_for(std::max(b.cap_edges, b.cap_dst), 256, 8);
  relabel_kernel<<<grid, 256, 0, st>>>(bm.bits, bm.wprefix, meta, b.edges, b.cap_edges, b.dst,
                                       b.dst_pos);
  CB_LAUNCH("relabel");
}

void launch_rank(const Bitmap& bm, const uint32_t* ids, const unsigned long long* count,
                 uint32_t* rank_out, cudaStream_t st) {
  rank_kernel<<<kNumSMs * 4, 256, 0, st>>>(bm.bits, bm.wprefix, ids, count, rank_out);
  CB_LAUNCH("rank");
}

void launch_clear(Bitmap& bm, const uint32_t* list, const unsigned long long* count,
                  cudaStream_t st) {
  clear_kernel<<<kNumSMs * 4, 256, 0, st>>>(bm.bits, list, count);
  CB_LAUNCH("clear");
}

}  // namespace cb
