// C-ABI: host-buffer forms of the path's data movement and GCN block ops, for
// the C++ drop-in (paper_2310_12403_b200/dropin/), whose reference signatures
// take and return host std::vectors. Each call uploads its operands, runs the
// same kernels the device-resident step uses, and copies the result back.
#include "capi_internal.h"
#include "train.h"
#include "train_util.cuh"
#include "gather.h"
#include "cb_device.cuh"

using namespace cb_train_util;

namespace {

// owner rows of a requester-side contribution list, stable by (part, index)
struct Contribs {
  uint64_t* off = nullptr;  // [n_owner + 1] contribution ranges per owner row
  uint64_t* src = nullptr;  // contribution -> requester row (global)
};

// owner_base[q] = first global owner row of part q; requester row j of part
// p (global index req_off[p] + j) contributes to owner_base[part] + row.
Contribs sort_contribs(uint32_t P, const uint64_t* loc_off, const uint32_t* d_part,
                       const uint32_t* d_row, const uint64_t* owner_base_h, uint64_t n_owner,
                       TmpArena& A, cudaStream_t st) {
  const uint64_t total = loc_off[P];
  uint64_t* d_obase = A.get<uint64_t>(P + 1);
  CB_CUDA(cudaMemcpyAsync(d_obase, owner_base_h, (P + 1) * 8, cudaMemcpyHostToDevice, st));
  uint32_t* cnt = A.get<uint32_t>(n_owner);
  CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(n_owner, 1) * 4, st));
  uint64_t* key = A.get<uint64_t>(total);
  uint64_t* val = A.get<uint64_t>(total);
  uint64_t* key2 = A.get<uint64_t>(total);
  uint64_t* val2 = A.get<uint64_t>(total);
  if (total)
    owner_key_kernel<<<grid_of_n(total), 256, 0, st>>>(d_part, d_row, total, d_obase, 0, cnt, key,
                                                       val);
  CB_LAUNCH("owner_key");
  Contribs c;
  c.off = A.get<uint64_t>(n_owner + 1);
  scan_counts(cnt, n_owner, c.off, A, st);
  cub::DoubleBuffer<uint64_t> kb(key, key2), vb(val, val2);
  size_t bytes = 0;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, static_cast<int64_t>(total), 0,
                                          64, st));
  void* tmp = A.get<unsigned char>(bytes);
  CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int64_t>(total), 0, 64,
                                          st));
  c.src = vb.Current();
  return c;
}

// all_to_all_reverse (coop.cpp:161-176): owner row k = the last requester row
// written to it in (part, index) order, zeros if none
__global__ void reverse_last_kernel(const uint64_t* __restrict__ off,
                                    const uint64_t* __restrict__ src, uint64_t n_owner,
                                    const double* __restrict__ req, uint32_t dim, double* out) {
  const uint64_t total = n_owner * dim;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = x / dim, c = x % dim;
    out[x] = off[k + 1] > off[k] ? req[src[off[k + 1] - 1] * dim + c] : 0.0;
  }
}

void check_record(uint32_t P, const uint64_t* loc_off, const uint32_t* loc_part,
                  const uint64_t* loc_row, const uint64_t* owner_rows) {
  require(P >= 1, "exchange: no parts");
  require(loc_off[0] == 0, "exchange: offsets must start at 0");
  for (uint32_t p = 0; p < P; ++p) require(loc_off[p + 1] >= loc_off[p], "exchange: offsets");
  for (uint64_t j = 0; j < loc_off[P]; ++j) {
    require(loc_part[j] < P, "exchange: src_location part out of range");
    require(loc_row[j] < owner_rows[loc_part[j]], "exchange: src_location row out of range");
  }
}

// (dst, edge index) keys of a block's edges, for a stable grouping by dst
__global__ void dst_key_kernel(const uint2* __restrict__ e, uint64_t n, uint32_t* key,
                               uint32_t* val) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    key[i] = e[i].y;
    val[i] = static_cast<uint32_t>(i);
  }
}

__global__ void permute_edges_kernel(const uint2* __restrict__ e, const uint32_t* __restrict__ perm,
                                     uint64_t n, uint2* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = e[perm[i]];
}

__global__ void labels_kernel(uint64_t seed, uint32_t classes, uint64_t v0, uint64_t n,
                              uint32_t* out) {
  const uint64_t pfx = cbdev::hstep(cbdev::hinit(seed), 10ULL);  // {kStreamLabel, v}
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(cbdev::hstep(pfx, v0 + i) % classes);
}

}  // namespace

extern "C" {

// FeatureStore::synth (coop.cpp:359-376) computed on the device, delivered to
// host memory: values[v * dim + j] = 2 * hash_uniform(seed, {9, v, j}) - 1 in
// f64, labels[v] = hash_bits(seed, {10, v}) mod classes (either may be null).
int cb_synth_host(int device, uint64_t n, uint32_t dim, uint32_t classes, uint64_t seed,
                  double* values, uint32_t* labels) {
  return guard([&] {
    require(classes >= 1 || labels == nullptr, "synth: num_classes must be >= 1");
    DeviceGuard dg(device);
    cudaStream_t st = 0;
    const uint64_t chunk = std::max<uint64_t>(1, (64ULL << 20) / std::max<uint32_t>(dim, 1));
    TmpArena A;
    double* d_v = values ? A.get<double>(std::min(n, chunk) * dim) : nullptr;
    uint32_t* d_l = labels ? A.get<uint32_t>(std::min(n, chunk)) : nullptr;
    for (uint64_t v0 = 0; v0 < n; v0 += chunk) {
      const uint64_t c = std::min(chunk, n - v0);
      if (values && dim) {
        launch_synth(seed, dim, CB_F64, c, nullptr, v0, d_v, st);
        CB_CUDA(cudaMemcpyAsync(values + v0 * dim, d_v, c * dim * 8, cudaMemcpyDeviceToHost, st));
      }
      if (labels) {
        labels_kernel<<<grid_of_n(c), 256, 0, st>>>(seed, classes, v0, c, d_l);
        CB_LAUNCH("labels");
        CB_CUDA(cudaMemcpyAsync(labels + v0, d_l, c * 4, cudaMemcpyDeviceToHost, st));
      }
      CB_CUDA(cudaStreamSynchronize(st));
    }
  });
}


int cb_op_forward_rows(int device, uint32_t P, const uint64_t* loc_off, const uint32_t* loc_part,
                       const uint64_t* loc_row, const uint64_t* owner_row_counts, uint32_t dim,
                       const double* owner_flat, double* out_flat) {
  NvtxRange nvtx_("cb.op_forward_rows");
  return guard([&] {
    require(loc_off && owner_row_counts && (dim == 0 || (owner_flat || loc_off[P] == 0)),
            "null argument");
    check_record(P, loc_off, loc_part, loc_row, owner_row_counts);
    DeviceGuard dg(device);
    cudaStream_t st = 0;
    TmpArena A;
    const uint64_t nreq = loc_off[P];
    if (nreq == 0 || dim == 0) return;
    std::vector<uint64_t> obase(P + 1, 0);
    for (uint32_t q = 0; q < P; ++q) obase[q + 1] = obase[q] + owner_row_counts[q];
    double* d_own = A.get<double>(obase[P] * dim);
    CB_CUDA(cudaMemcpyAsync(d_own, owner_flat, obase[P] * dim * 8, cudaMemcpyHostToDevice, st));
    std::vector<const double*> bases(P);
    for (uint32_t q = 0; q < P; ++q) bases[q] = d_own + obase[q] * dim;
    const double** d_bases = A.get<const double*>(P);
    CB_CUDA(cudaMemcpyAsync(d_bases, bases.data(), P * sizeof(void*), cudaMemcpyHostToDevice, st));
    std::vector<uint32_t> rows32(nreq);
    for (uint64_t j = 0; j < nreq; ++j) rows32[j] = static_cast<uint32_t>(loc_row[j]);
    uint32_t* d_part = A.get<uint32_t>(nreq);
    uint32_t* d_row = A.get<uint32_t>(nreq);
    CB_CUDA(cudaMemcpyAsync(d_part, loc_part, nreq * 4, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaMemcpyAsync(d_row, rows32.data(), nreq * 4, cudaMemcpyHostToDevice, st));
    double* d_out = A.get<double>(nreq * dim);
    launch_row_forward(d_bases, d_part, d_row, nreq, dim, d_out, st);
    CB_CUDA(cudaMemcpyAsync(out_flat, d_out, nreq * dim * 8, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

int cb_op_reverse_rows(int device, uint32_t P, const uint64_t* loc_off, const uint32_t* loc_part,
                       const uint64_t* loc_row, const uint64_t* owner_row_counts, uint32_t dim,
                       const double* requester_flat, int sum, double* owner_out_flat) {
  NvtxRange nvtx_("cb.op_reverse_rows");
  return guard([&] {
    require(loc_off && owner_row_counts, "null argument");
    check_record(P, loc_off, loc_part, loc_row, owner_row_counts);
    DeviceGuard dg(device);
    cudaStream_t st = 0;
    TmpArena A;
    const uint64_t nreq = loc_off[P];
    std::vector<uint64_t> obase(P + 1, 0);
    for (uint32_t q = 0; q < P; ++q) obase[q + 1] = obase[q] + owner_row_counts[q];
    const uint64_t no = obase[P];
    if (no == 0 || dim == 0) return;
    double* d_out = A.get<double>(no * dim);
    if (nreq == 0) {
      CB_CUDA(cudaMemsetAsync(d_out, 0, no * dim * 8, st));
    } else {
      std::vector<uint32_t> rows32(nreq);
      for (uint64_t j = 0; j < nreq; ++j) rows32[j] = static_cast<uint32_t>(loc_row[j]);
      uint32_t* d_part = A.get<uint32_t>(nreq);
      uint32_t* d_row = A.get<uint32_t>(nreq);
      CB_CUDA(cudaMemcpyAsync(d_part, loc_part, nreq * 4, cudaMemcpyHostToDevice, st));
      CB_CUDA(cudaMemcpyAsync(d_row, rows32.data(), nreq * 4, cudaMemcpyHostToDevice, st));
      double* d_req = A.get<double>(nreq * dim);
      CB_CUDA(cudaMemcpyAsync(d_req, requester_flat, nreq * dim * 8, cudaMemcpyHostToDevice, st));
      const Contribs c = sort_contribs(P, loc_off, d_part, d_row, obase.data(), no, A, st);
      if (sum) {
        launch_reverse_sum(c.off, c.src, no, d_req, dim, d_out, st);
      } else {
        reverse_last_kernel<<<grid_of_n(no * dim), 256, 0, st>>>(c.off, c.src, no, d_req, dim,
                                                                 d_out);
        CB_LAUNCH("reverse_last");
      }
    }
    CB_CUDA(cudaMemcpyAsync(owner_out_flat, d_out, no * dim * 8, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

// gcn_forward / gcn_backward of one block (coop.cpp:236-331) on host buffers:
// edges are (src_idx, dst_idx) pairs in any order (the reference accumulates in edge order).
int cb_op_gcn_block(int device, uint64_t n_src, uint64_t n_dst, uint64_t n_edges,
                    const uint32_t* edges, const uint32_t* dst_pos, const double* h_in,
                    uint32_t in_dim, const double* w, uint32_t out_dim, int tanh_act,
                    const double* grad_out, double* out, double* grad_h_in, double* grad_w) {
  NvtxRange nvtx_("cb.op_gcn_block");
  return guard([&] {
    for (uint64_t e = 0; e < n_edges; ++e)
      require(edges[2 * e] < n_src && edges[2 * e + 1] < n_dst, "gcn: edge index out of range");
    for (uint64_t d = 0; d < n_dst; ++d)
      require(dst_pos[d] < n_src, "gcn: dst_pos_in_src out of range");
    bool grouped = true;
    for (uint64_t e = 1; e < n_edges && grouped; ++e) grouped = edges[2 * e + 1] >= edges[2 * e - 1];
    DeviceGuard dg(device);
    cudaStream_t st = 0;
    TmpArena A;
    uint2* d_e = A.get<uint2>(n_edges);
    uint32_t* d_dp = A.get<uint32_t>(n_dst);
    double* d_h = A.get<double>(n_src * in_dim);
    double* d_w = A.get<double>(static_cast<uint64_t>(in_dim) * out_dim);
    if (n_edges) CB_CUDA(cudaMemcpyAsync(d_e, edges, n_edges * 8, cudaMemcpyHostToDevice, st));
    if (n_dst) CB_CUDA(cudaMemcpyAsync(d_dp, dst_pos, n_dst * 4, cudaMemcpyHostToDevice, st));
    if (n_src * in_dim)
      CB_CUDA(cudaMemcpyAsync(d_h, h_in, n_src * in_dim * 8, cudaMemcpyHostToDevice, st));
    if (in_dim * out_dim)
      CB_CUDA(cudaMemcpyAsync(d_w, w, static_cast<uint64_t>(in_dim) * out_dim * 8,
                              cudaMemcpyHostToDevice, st));
    // The aggregate walks each destination's edges in edge order; a block
    // whose edges are not grouped by destination is grouped by a stable sort
    // (the gradient scatter keeps the original order per source).
    uint2* d_eg = d_e;
    if (!grouped) {
      uint32_t* key = A.get<uint32_t>(n_edges);
      uint32_t* val = A.get<uint32_t>(n_edges);
      uint32_t* key2 = A.get<uint32_t>(n_edges);
      uint32_t* val2 = A.get<uint32_t>(n_edges);
      dst_key_kernel<<<grid_of_n(n_edges), 256, 0, st>>>(d_e, n_edges, key, val);
      CB_LAUNCH("dst_key");
      cub::DoubleBuffer<uint32_t> kb(key, key2), vb(val, val2);
      size_t bytes = 0;
      CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb,
                                              static_cast<int64_t>(n_edges), 0, 32, st));
      void* tmp = A.get<unsigned char>(bytes);
      CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int64_t>(n_edges),
                                              0, 32, st));
      d_eg = A.get<uint2>(n_edges);
      permute_edges_kernel<<<grid_of_n(n_edges), 256, 0, st>>>(d_e, vb.Current(), n_edges, d_eg);
      CB_LAUNCH("permute_edges");
    }
    uint32_t* deg = A.get<uint32_t>(n_dst);
    CB_CUDA(cudaMemsetAsync(deg, 0, std::max<uint64_t>(n_dst, 1) * 4, st));
    launch_in_degrees(d_e, n_edges, deg, st);
    uint64_t* off = A.get<uint64_t>(n_dst + 1);
    scan_counts(deg, n_dst, off, A, st);
    double* agg = A.get<double>(n_dst * in_dim);
    launch_aggregate(d_eg, deg, off, d_dp, n_dst, d_h, in_dim, agg, st);
    double* o = A.get<double>(n_dst * out_dim);
    launch_dense(agg, n_dst, in_dim, d_w, out_dim, tanh_act != 0, o, st);
    if (out && n_dst * out_dim)
      CB_CUDA(cudaMemcpyAsync(out, o, n_dst * out_dim * 8, cudaMemcpyDeviceToHost, st));
    if (grad_out) {
      const uint64_t nw = static_cast<uint64_t>(in_dim) * out_dim;
      double* dp = A.get<double>(n_dst * out_dim);
      if (n_dst * out_dim)
        CB_CUDA(cudaMemcpyAsync(dp, grad_out, n_dst * out_dim * 8, cudaMemcpyHostToDevice, st));
      if (tanh_act) launch_tanh_grad(o, n_dst * out_dim, dp, st);
      double* gw = A.get<double>(nw);
      launch_grad_w(agg, dp, n_dst, in_dim, out_dim, gw, st);
      double* dagg = A.get<double>(n_dst * in_dim);
      launch_grad_agg(dp, d_w, n_dst, in_dim, out_dim, dagg, st);
      uint32_t* cnt = A.get<uint32_t>(n_src);
      CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(n_src, 1) * 4, st));
      uint32_t* key = A.get<uint32_t>(n_edges);
      uint32_t* val = A.get<uint32_t>(n_edges);
      uint32_t* key2 = A.get<uint32_t>(n_edges);
      uint32_t* val2 = A.get<uint32_t>(n_edges);
      if (n_edges)
        src_hist_kernel<<<grid_of_n(n_edges), 256, 0, st>>>(d_e, n_edges, cnt, key, val);
      CB_LAUNCH("src_hist");
      uint64_t* soff = A.get<uint64_t>(n_src + 1);
      scan_counts(cnt, n_src, soff, A, st);
      cub::DoubleBuffer<uint32_t> kb(key, key2), vb(val, val2);
      size_t bytes = 0;
      CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb,
                                              static_cast<int64_t>(n_edges), 0, 32, st));
      void* tmp = A.get<unsigned char>(bytes);
      CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int64_t>(n_edges),
                                              0, 32, st));
      int64_t* iso = A.get<int64_t>(n_src);
      CB_CUDA(cudaMemsetAsync(iso, 0xff, std::max<uint64_t>(n_src, 1) * 8, st));
      launch_iso_dst(deg, d_dp, n_dst, iso, st);
      double* gh = A.get<double>(n_src * in_dim);
      launch_grad_h_in(d_e, vb.Current(), soff, deg, iso, n_src, dagg, in_dim, gh, st);
      if (grad_h_in && n_src * in_dim)
        CB_CUDA(cudaMemcpyAsync(grad_h_in, gh, n_src * in_dim * 8, cudaMemcpyDeviceToHost, st));
      if (grad_w && nw) CB_CUDA(cudaMemcpyAsync(grad_w, gw, nw * 8, cudaMemcpyDeviceToHost, st));
    }
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

// A feature table from host rows (FeatureStore::values, coop.hpp:140-155):
// n_rows x dim of dtype, identity row map.
int cb_features_from_host(int device, uint64_t n_rows, uint32_t dim, int dtype, const void* rows,
                          cb_features** out) {
  return guard([&] {
    require(out != nullptr && (rows != nullptr || n_rows == 0), "null argument");
    require(dim >= 1, "feature dim must be >= 1");
    require(dtype == CB_F64 || dtype == CB_F32 || dtype == CB_F16, "unknown dtype");
    DeviceGuard dg(device);
    auto f = std::make_unique<cb_features>();
    f->device = device;
    f->dim = dim;
    f->dtype = dtype;
    const uint64_t es = dtype == CB_F64 ? 8 : (dtype == CB_F32 ? 4 : 2);
    f->row_bytes = es * dim;
    f->n_rows = n_rows;
    f->table = f->mem.alloc<unsigned char>(std::max<uint64_t>(n_rows, 1) * f->row_bytes);
    if (n_rows)
      h2d_sync(f->table, rows, n_rows * f->row_bytes);
    *out = f.release();
  });
}

// FeatureStore::labels (coop.hpp:145) for the training step's softmax
// (instead of synth's hash(seed, {10, v}) mod C); nullptr clears.
int cb_features_set_labels(cb_features* f, const uint32_t* labels) {
  return guard([&] {
    require(f != nullptr, "null features");
    DeviceGuard dg(f->device);
    if (!labels) {
      f->labels = nullptr;
      return;
    }
    if (!f->labels) f->labels = f->mem.alloc<uint32_t>(std::max<uint64_t>(f->n_rows, 1));
    if (f->n_rows)
      h2d_sync(f->labels, labels, f->n_rows * 4);
  });
}

// The caller's host rows, read in place by the device: the range is pinned
// and mapped (cudaHostRegister) until cb_features_destroy. For a table that
// lives in host memory (the reference's FeatureStore::values, coop.hpp:144);
// the gather reads rows over the host link instead of copying the table.
int cb_features_wrap_host(int device, uint64_t n_rows, uint32_t dim, int dtype,
                          const void* rows, cb_features** out) {
  return guard([&] {
    require(out != nullptr && (rows != nullptr || n_rows == 0), "null argument");
    require(dim >= 1, "feature dim must be >= 1");
    require(dtype == CB_F64 || dtype == CB_F32 || dtype == CB_F16, "unknown dtype");
    DeviceGuard dg(device);
    auto f = std::make_unique<cb_features>();
    f->device = device;
    f->dim = dim;
    f->dtype = dtype;
    const uint64_t es = dtype == CB_F64 ? 8 : (dtype == CB_F32 ? 4 : 2);
    f->row_bytes = es * dim;
    f->n_rows = n_rows;
    require(reinterpret_cast<uintptr_t>(rows) % es == 0, "host rows are not element-aligned");
    if (n_rows) {
      void* h = const_cast<void*>(rows);
      CB_CUDA(cudaHostRegister(h, n_rows * f->row_bytes,
                               cudaHostRegisterMapped | cudaHostRegisterPortable));
      f->registered = h;
      CB_CUDA(cudaHostGetDevicePointer(&f->table, h, 0));
    } else {
      f->table = f->mem.alloc<unsigned char>(f->row_bytes);
    }
    *out = f.release();
  });
}

// FeatureStore::load_rows (coop.hpp:151, coop.cpp:378-388) from host ids into
// host rows: out[i] = row ids[i]; ids must be < n_rows (the reference reads
// past its table otherwise).
int cb_op_load_rows(const cb_features* f, const uint32_t* ids, uint64_t n, void* out) {
  return guard([&] {
    require(f != nullptr && ((ids != nullptr && out != nullptr) || n == 0), "null argument");
    require(f->shard_rows == 0 && f->row_map == nullptr, "load_rows needs a whole, unsharded table");
    if (!n) return;
    for (uint64_t i = 0; i < n; ++i)
      if (ids[i] >= f->n_rows)
        throw cb::Error(kInput, "load_rows: vertex id " + std::to_string(ids[i]) +
                                    " out of range [0, " + std::to_string(f->n_rows) + ")");
    DeviceGuard dg(f->device);
    auto* fm = const_cast<cb_features*>(f);  // scratch only; the table is not modified
    if (!fm->op_stream) CB_CUDA(cudaStreamCreateWithFlags(&fm->op_stream, cudaStreamNonBlocking));
    cudaStream_t st = fm->op_stream;
    if (fm->op_cap < n) {
      if (fm->op_ids) CB_CUDA(cudaFree(fm->op_ids));
      if (fm->op_out) CB_CUDA(cudaFree(fm->op_out));
      fm->op_cap = n + n / 4;
      CB_CUDA(cudaMalloc(&fm->op_ids, fm->op_cap * 4));
      CB_CUDA(cudaMalloc(&fm->op_out, fm->op_cap * f->row_bytes));
    }
    CB_CUDA(cudaMemcpyAsync(fm->op_ids, ids, n * 4, cudaMemcpyHostToDevice, st));
    launch_gather(f->table, vec_bytes_for(f->row_bytes), f->row_bytes,
                  static_cast<uint32_t*>(fm->op_ids), nullptr, n, nullptr, fm->op_out, st);
    CB_LAUNCH("load_rows");
    CB_CUDA(cudaMemcpyAsync(out, fm->op_out, n * f->row_bytes, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
