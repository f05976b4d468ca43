// GCN forward/backward of the cooperative training step (coop.cpp:161-357,
// 394-610), FP64 on the device. Every reduction keeps the reference's
// summation order (edges in edge order per destination or per source, rows
// in row order per weight entry, parts in part order), so results equal the
// reference up to libm (tanh / exp / log in libdevice vs glibc).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace cb {

// deg[di] = sampled in-edges of dst di (edges grouped by dst, in dst order)
void launch_in_degrees(const uint2* edges, uint64_t n_edges, uint32_t* deg, cudaStream_t st);
// aggregate (coop.cpp:203-226): mean of the in-neighbour rows, own row if none
void launch_aggregate(const uint2* edges, const uint32_t* deg, const uint64_t* off,
                      const uint32_t* dst_pos, uint64_t n_dst, const double* h_in, uint32_t dim,
                      double* agg, cudaStream_t st);
// out = act(agg * W) (coop.cpp:236-255), zero activations skipped as in the reference
void launch_dense(const double* agg, uint64_t rows, uint32_t in_dim, const double* w,
                  uint32_t out_dim, bool tanh_act, double* out, cudaStream_t st);
// softmax cross-entropy rows (coop.cpp:392-414): per-row loss, scaled gradient
void launch_softmax_ce(const double* logits, uint64_t rows, uint32_t classes,
                       const uint32_t* row_vertex, uint64_t label_seed,
                       const uint32_t* labels, double scale, double* row_loss, double* grad,
                       cudaStream_t st);
// dpre = grad * (1 - t^2) for tanh layers (in place)
void launch_tanh_grad(const double* t, uint64_t n, double* grad, cudaStream_t st);
// grad_w[i][j] = sum_r agg[r][i] * dp[r][j] (rows ascending, zero agg skipped)
void launch_grad_w(const double* agg, const double* dp, uint64_t rows, uint32_t in_dim,
                   uint32_t out_dim, double* gw, cudaStream_t st);
// dagg[r][i] = sum_j dp[r][j] * W[i][j]
void launch_grad_agg(const double* dp, const double* w, uint64_t rows, uint32_t in_dim,
                     uint32_t out_dim, double* dagg, cudaStream_t st);
// grad_h_in (coop.cpp:317-331): per source row, its edges in edge order
// (CSC order from a stable sort), then the isolated dst whose own row it is
void launch_grad_h_in(const uint2* edges, const uint32_t* edge_by_src, const uint64_t* src_off,
                      const uint32_t* deg, const int64_t* iso_dst, uint64_t n_src,
                      const double* dagg, uint32_t dim, double* gh, cudaStream_t st);
// iso_dst[dst_pos[di]] = di for every dst with no sampled in-edge (else -1)
void launch_iso_dst(const uint32_t* deg, const uint32_t* dst_pos, uint64_t n_dst,
                    int64_t* iso_dst, cudaStream_t st);
// rows[j] = owner_rows[part[j]][row[j]] (all_to_all_forward, coop.cpp:145-159)
void launch_row_forward(const double* const* owner_rows, const uint32_t* loc_part,
                        const uint32_t* loc_row, uint64_t n, uint32_t dim, double* out,
                        cudaStream_t st);
// owner rows from a sorted contribution list (all_to_all_reverse_sum,
// coop.cpp:177-194): out[k] = sum over contribs in (part, index) order
void launch_reverse_sum(const uint64_t* contrib_off, const uint64_t* contrib_src,
                        uint64_t n_owner_rows, const double* requester_rows, uint32_t dim,
                        double* out, cudaStream_t st);
// a += b elementwise (part-ordered gradient sums)
void launch_add(double* a, const double* b, uint64_t n, cudaStream_t st);

}  // namespace cb
