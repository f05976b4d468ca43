// GCN layer kernels of the cooperative training step (see train.h). FP64,
// explicit _rn arithmetic in the reference's accumulation order.
#include "cb_internal.h"
#include "train.h"

namespace cb {
using namespace cbdev;

namespace {

constexpr int kTB = 256;

int grid_n(uint64_t n, int per = kTB) {
  return static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>((n + per - 1) / per, static_cast<uint64_t>(kNumSMs) * 16)));
}

__global__ void in_degrees_kernel(const uint2* __restrict__ edges, uint64_t n, uint32_t* deg) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&deg[edges[e].y], 1u);
}

// warp per dst row; lane c owns columns c, c+32, ...; edges of the row in order
__global__ void aggregate_kernel(const uint2* __restrict__ edges, const uint32_t* __restrict__ deg,
                                 const uint64_t* __restrict__ off,
                                 const uint32_t* __restrict__ dst_pos, uint64_t n_dst,
                                 const double* __restrict__ h, uint32_t dim, double* agg) {
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t di = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32;
       di < n_dst; di += nw) {
    const uint32_t d = deg[di];
    const uint64_t e0 = off[di];
    double* out = agg + di * dim;
    if (d == 0) {
      const double* self = h + static_cast<uint64_t>(dst_pos[di]) * dim;
      for (uint32_t c = lane_id(); c < dim; c += 32) out[c] = self[c];
      continue;
    }
    const double inv = __ddiv_rn(1.0, static_cast<double>(d));
    for (uint32_t c = lane_id(); c < dim; c += 32) {
      double acc = 0.0;
      for (uint64_t e = e0; e < e0 + d; ++e)
        acc = __dadd_rn(acc, h[static_cast<uint64_t>(edges[e].x) * dim + c]);
      out[c] = __dmul_rn(acc, inv);
    }
  }
}

__global__ void dense_kernel(const double* __restrict__ agg, uint64_t rows, uint32_t in_dim,
                             const double* __restrict__ w, uint32_t out_dim, int tanh_act,
                             double* out) {
  const uint64_t total = rows * out_dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = x / out_dim;
    const uint32_t j = static_cast<uint32_t>(x - r * out_dim);
    const double* a = agg + r * in_dim;
    double o = 0.0;
    for (uint32_t i = 0; i < in_dim; ++i) {
      const double ai = a[i];
      if (ai == 0.0) continue;
      o = __dadd_rn(o, __dmul_rn(ai, w[static_cast<uint64_t>(i) * out_dim + j]));
    }
    out[x] = tanh_act ? tanh(o) : o;
  }
}

__global__ void softmax_ce_kernel(const double* __restrict__ z_all, uint64_t rows, uint32_t C,
                                  const uint32_t* __restrict__ row_vertex, uint64_t label_seed,
                                  const uint32_t* __restrict__ labels, double scale,
                                  double* row_loss, double* grad) {
  const uint64_t pfx = hstep(hinit(label_seed), 10ULL);  // {kStreamLabel, v}
  for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double* z = z_all + r * C;
    double* gz = grad + r * C;
    double zmax = z[0];
    for (uint32_t j = 1; j < C; ++j) zmax = fmax(zmax, z[j]);
    double denom = 0.0;
    for (uint32_t j = 0; j < C; ++j) denom = __dadd_rn(denom, exp(__dsub_rn(z[j], zmax)));
    // FeatureStore::labels (coop.hpp:145): given, or synth's hash(seed,{10,v}) mod C
    const uint32_t label = labels ? labels[row_vertex[r]]
                                  : static_cast<uint32_t>(hstep(pfx, row_vertex[r]) % C);
    row_loss[r] = __dsub_rn(log(denom), __dsub_rn(z[label], zmax));
    for (uint32_t j = 0; j < C; ++j) {
      const double p = __ddiv_rn(exp(__dsub_rn(z[j], zmax)), denom);
      gz[j] = __dmul_rn(__dsub_rn(p, j == label ? 1.0 : 0.0), scale);
    }
  }
}

__global__ void tanh_grad_kernel(const double* __restrict__ t, uint64_t n, double* g) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    g[x] = __dmul_rn(g[x], __dsub_rn(1.0, __dmul_rn(t[x], t[x])));
}

__global__ void grad_w_kernel(const double* __restrict__ agg, const double* __restrict__ dp,
                              uint64_t rows, uint32_t in_dim, uint32_t out_dim, double* gw) {
  const uint64_t total = static_cast<uint64_t>(in_dim) * out_dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = static_cast<uint32_t>(x / out_dim), j = static_cast<uint32_t>(x % out_dim);
    double acc = 0.0;
    for (uint64_t r = 0; r < rows; ++r) {
      const double a = agg[r * in_dim + i];
      if (a == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(a, dp[r * out_dim + j]));
    }
    gw[x] = acc;
  }
}

__global__ void grad_agg_kernel(const double* __restrict__ dp, const double* __restrict__ w,
                                uint64_t rows, uint32_t in_dim, uint32_t out_dim, double* dagg) {
  const uint64_t total = rows * in_dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = x / in_dim;
    const uint32_t i = static_cast<uint32_t>(x - r * in_dim);
    const double* d = dp + r * out_dim;
    const double* wr = w + static_cast<uint64_t>(i) * out_dim;
    double acc = 0.0;
    for (uint32_t j = 0; j < out_dim; ++j) acc = __dadd_rn(acc, __dmul_rn(d[j], wr[j]));
    dagg[x] = acc;
  }
}

__global__ void iso_dst_kernel(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ dst_pos,
                               uint64_t n_dst, int64_t* iso) {
  for (uint64_t di = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; di < n_dst;
       di += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (deg[di] == 0) iso[dst_pos[di]] = static_cast<int64_t>(di);
}

// warp per source row
__global__ void grad_h_in_kernel(const uint2* __restrict__ edges,
                                 const uint32_t* __restrict__ by_src,
                                 const uint64_t* __restrict__ src_off,
                                 const uint32_t* __restrict__ deg,
                                 const int64_t* __restrict__ iso, uint64_t n_src,
                                 const double* __restrict__ dagg, uint32_t dim, double* gh) {
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t si = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32;
       si < n_src; si += nw) {
    const uint64_t e0 = src_off[si], e1 = src_off[si + 1];
    const int64_t self = iso[si];
    for (uint32_t c = lane_id(); c < dim; c += 32) {
      double acc = 0.0;
      for (uint64_t k = e0; k < e1; ++k) {
        const uint32_t di = edges[by_src[k]].y;
        const double inv = __ddiv_rn(1.0, static_cast<double>(deg[di]));
        acc = __dadd_rn(acc, __dmul_rn(dagg[static_cast<uint64_t>(di) * dim + c], inv));
      }
      if (self >= 0) acc = __dadd_rn(acc, dagg[static_cast<uint64_t>(self) * dim + c]);
      gh[si * dim + c] = acc;
    }
  }
}

__global__ void row_forward_kernel(const double* const* __restrict__ owner_rows,
                                   const uint32_t* __restrict__ part,
                                   const uint32_t* __restrict__ row, uint64_t n, uint32_t dim,
                                   double* out) {
  const uint64_t total = n * dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = x / dim, c = x - j * dim;
    out[x] = owner_rows[part[j]][static_cast<uint64_t>(row[j]) * dim + c];
  }
}

__global__ void reverse_sum_kernel(const uint64_t* __restrict__ off,
                                   const uint64_t* __restrict__ src, uint64_t n_rows,
                                   const double* __restrict__ req, uint32_t dim, double* out) {
  const uint64_t total = n_rows * dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = x / dim, c = x - k * dim;
    double acc = 0.0;
    for (uint64_t t = off[k]; t < off[k + 1]; ++t) acc = __dadd_rn(acc, req[src[t] * dim + c]);
    out[x] = acc;
  }
}

__global__ void add_kernel(double* a, const double* __restrict__ b, uint64_t n) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a[x] = __dadd_rn(a[x], b[x]);
}

}  // namespace

void launch_in_degrees(const uint2* edges, uint64_t n, uint32_t* deg, cudaStream_t st) {
  if (n) in_degrees_kernel<<<grid_n(n), kTB, 0, st>>>(edges, n, deg);
  CB_LAUNCH("in_degrees");
}
void launch_aggregate(const uint2* edges, const uint32_t* deg, const uint64_t* off,
                      const uint32_t* dst_pos, uint64_t n_dst, const double* h, uint32_t dim,
                      double* agg, cudaStream_t st) {
  if (n_dst) aggregate_kernel<<<grid_n(n_dst * 32), kTB, 0, st>>>(edges, deg, off, dst_pos, n_dst,
                                                                 h, dim, agg);
  CB_LAUNCH("aggregate");
}
void launch_dense(const double* agg, uint64_t rows, uint32_t in_dim, const double* w,
                  uint32_t out_dim, bool tanh_act, double* out, cudaStream_t st) {
  if (rows) dense_kernel<<<grid_n(rows * out_dim), kTB, 0, st>>>(agg, rows, in_dim, w, out_dim,
                                                                 tanh_act ? 1 : 0, out);
  CB_LAUNCH("dense");
}
void launch_softmax_ce(const double* logits, uint64_t rows, uint32_t classes,
                       const uint32_t* row_vertex, uint64_t label_seed, const uint32_t* labels,
                       double scale,
                       double* row_loss, double* grad, cudaStream_t st) {
  if (rows) softmax_ce_kernel<<<grid_n(rows), kTB, 0, st>>>(logits, rows, classes, row_vertex,
                                                           label_seed, labels, scale, row_loss, grad);
  CB_LAUNCH("softmax_ce");
}
void launch_tanh_grad(const double* t, uint64_t n, double* grad, cudaStream_t st) {
  if (n) tanh_grad_kernel<<<grid_n(n), kTB, 0, st>>>(t, n, grad);
  CB_LAUNCH("tanh_grad");
}
void launch_grad_w(const double* agg, const double* dp, uint64_t rows, uint32_t in_dim,
                   uint32_t out_dim, double* gw, cudaStream_t st) {
  grad_w_kernel<<<grid_n(static_cast<uint64_t>(in_dim) * out_dim), kTB, 0, st>>>(
      agg, dp, rows, in_dim, out_dim, gw);
  CB_LAUNCH("grad_w");
}
void launch_grad_agg(const double* dp, const double* w, uint64_t rows, uint32_t in_dim,
                     uint32_t out_dim, double* dagg, cudaStream_t st) {
  if (rows) grad_agg_kernel<<<grid_n(rows * in_dim), kTB, 0, st>>>(dp, w, rows, in_dim, out_dim,
                                                                   dagg);
  CB_LAUNCH("grad_agg");
}
void launch_iso_dst(const uint32_t* deg, const uint32_t* dst_pos, uint64_t n_dst, int64_t* iso,
                    cudaStream_t st) {
  if (n_dst) iso_dst_kernel<<<grid_n(n_dst), kTB, 0, st>>>(deg, dst_pos, n_dst, iso);
  CB_LAUNCH("iso_dst");
}
void launch_grad_h_in(const uint2* edges, const uint32_t* by_src, const uint64_t* src_off,
                      const uint32_t* deg, const int64_t* iso, uint64_t n_src,
                      const double* dagg, uint32_t dim, double* gh, cudaStream_t st) {
  if (n_src) grad_h_in_kernel<<<grid_n(n_src * 32), kTB, 0, st>>>(edges, by_src, src_off, deg,
                                                                  iso, n_src, dagg, dim, gh);
  CB_LAUNCH("grad_h_in");
}
void launch_row_forward(const double* const* owner_rows, const uint32_t* part,
                        const uint32_t* row, uint64_t n, uint32_t dim, double* out,
                        cudaStream_t st) {
  if (n) row_forward_kernel<<<grid_n(n * dim), kTB, 0, st>>>(owner_rows, part, row, n, dim, out);
  CB_LAUNCH("row_forward");
}
void launch_reverse_sum(const uint64_t* off, const uint64_t* src, uint64_t n_rows,
                        const double* req, uint32_t dim, double* out, cudaStream_t st) {
  if (n_rows) reverse_sum_kernel<<<grid_n(n_rows * dim), kTB, 0, st>>>(off, src, n_rows, req,
                                                                       dim, out);
  CB_LAUNCH("reverse_sum");
}
void launch_add(double* a, const double* b, uint64_t n, cudaStream_t st) {
  if (n) add_kernel<<<grid_n(n), kTB, 0, st>>>(a, b, n);
  CB_LAUNCH("add");
}

}  // namespace cb
