// C-ABI: GCN training step (f1) over the plan's last batch.
#include "capi_internal.h"

// ------------------------------------------------- GCN training step (f1) --
// GcnModel (coop.hpp:105-135) on the device and coop_train_step /
// indep_train_step (coop.cpp:438-610) over the plan's last batch: the
// forward pass mean-aggregates each block's sampled in-neighbours, applies
// W and tanh (identity at block 0), moves hidden rows to the requesters with
// the batch's exchange records (all_to_all_forward), takes the softmax
// cross-entropy of the seeds, and runs the backward pass with the owner-side
// gradient sums (all_to_all_reverse_sum). FP64 in the reference's
// accumulation order (train.cu).
struct cb_model {
  int device = 0;
  int L = 0;
  bool tanh_hidden = true;
  std::vector<uint32_t> rows, cols;
  std::vector<double*> w;
  ~cb_model() {
    for (double* p : w) if (p) cudaFree(p);
  }
};

#include "train_util.cuh"
using namespace cb_train_util;

extern "C" {

int cb_gcn_model_init(int device, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                      int num_layers, uint64_t seed, cb_model** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    require(num_layers >= 1, "GcnModel: num_layers must be >= 1");
    require(in_dim >= 1 && hidden >= 1 && classes >= 1, "GcnModel: dims must be >= 1");
    DeviceGuard dg(device);
    auto m = std::make_unique<cb_model>();
    m->device = device;
    m->L = num_layers;
    for (int l = 0; l < num_layers; ++l) {
      // GcnModel::init (coop.cpp:334-357): weights[l] is used at block l
      const uint32_t rows = (l == num_layers - 1) ? in_dim : hidden;
      const uint32_t cols = (l == 0) ? classes : hidden;
      std::vector<double> w(static_cast<uint64_t>(rows) * cols);
      const double scale = 1.0 / std::sqrt(static_cast<double>(rows));
      const uint64_t pfx = cbdev::hstep(cbdev::hstep(cbdev::hinit(seed), 11ULL),
                                        static_cast<uint64_t>(l));
      for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
          const double u = cbdev::ufb(cbdev::hstep(cbdev::hstep(pfx, i), j));
          volatile double t = 2.0 * u;  // no contraction: (2u - 1) * scale as two roundings
          w[i * cols + j] = (t - 1.0) * scale;
        }
      double* d = nullptr;
      CB_CUDA(cudaMalloc(&d, w.size() * 8));
      h2d_sync(d, w.data(), w.size() * 8);
      m->rows.push_back(rows);
      m->cols.push_back(cols);
      m->w.push_back(d);
    }
    *out = m.release();
  });
}

// A model of any layer shapes (GcnModel::weights as given, coop.hpp:126-135),
// weights uploaded from host row-major matrices back to back.
int cb_gcn_model_create(int device, int num_layers, const uint32_t* rows, const uint32_t* cols,
                        int tanh_hidden, const double* weights, cb_model** out) {
  return guard([&] {
    require(out != nullptr && rows != nullptr && cols != nullptr, "null argument");
    require(num_layers >= 1, "GcnModel: num_layers must be >= 1");
    DeviceGuard dg(device);
    auto m = std::make_unique<cb_model>();
    m->device = device;
    m->L = num_layers;
    m->tanh_hidden = tanh_hidden != 0;
    uint64_t o = 0;
    for (int l = 0; l < num_layers; ++l) {
      m->rows.push_back(rows[l]);
      m->cols.push_back(cols[l]);
      const uint64_t n = static_cast<uint64_t>(rows[l]) * cols[l];
      double* p = nullptr;
      CB_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * 8));
      m->w.push_back(p);
      if (weights && n) h2d_sync(p, weights + o, n * 8);
      o += n;
    }
    *out = m.release();
  });
}

int cb_gcn_model_weights(cb_model* m, int layer, double* host, int upload, uint64_t* rows,
                         uint64_t* cols) {
  return guard([&] {
    require(m != nullptr, "null model");
    require(layer >= 0 && layer < m->L, "layer index out of range");
    DeviceGuard dg(m->device);
    const uint64_t n = static_cast<uint64_t>(m->rows[layer]) * m->cols[layer];
    if (rows) *rows = m->rows[layer];
    if (cols) *cols = m->cols[layer];
    if (!host) return;
    if (upload) h2d_sync(m->w[layer], host, n * 8);
    else CB_CUDA(cudaMemcpy(host, m->w[layer], n * 8, cudaMemcpyDeviceToHost));
  });
}

void cb_gcn_model_destroy(cb_model* m) {
  if (!m) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  delete m;
  cudaSetDevice(prev);
}

int cb_train_step(cb_plan* pl, const cb_features* f, uint32_t classes, cb_model* m,
                  double* loss_out, double* grad_w_out) {
  NvtxRange nvtx_("cb.train_step");
  return guard([&] {
    require(pl != nullptr && f != nullptr && m != nullptr && loss_out != nullptr,
            "null argument");
    require(pl->have_batch, "no sampled batch in this plan");
    require_full_table(f);
    require(f->dtype == CB_F64, "train step: the feature table must be f64 (FeatureStore)");
    require(m->L == pl->L, "train step: model depth does not match layer count");
    require(m->rows[pl->L - 1] == f->dim, "train step: model input dim does not match store");
    require(classes >= 1 && m->cols[0] == classes, "train step: class count mismatch");
    DeviceGuard dg(pl->device);
    check_overflow(pl);
    const uint32_t P = pl->P;
    const int L = pl->L;
    const bool coop = pl->coop_active();
    cudaStream_t st = pl->stream;
    TmpArena A;
    // counts of the batch (one host read)
    std::vector<std::vector<LayerMeta>> M(P, std::vector<LayerMeta>(L + 1));
    for (uint32_t p = 0; p < P; ++p)
      CB_CUDA(cudaMemcpy(M[p].data(), pl->meta_at(p, 0), sizeof(LayerMeta) * (L + 1),
                         cudaMemcpyDeviceToHost));
    uint64_t total_seeds = 0;
    for (uint32_t p = 0; p < P; ++p) total_seeds += M[p][0].n_dst;
    require(total_seeds > 0, coop ? "coop_train_step: no seeds" : "indep_train_step: no seeds");
    auto dst_of = [&](uint32_t p, int l) -> const uint32_t* {
      if (l == 0) return pl->seeds + pl->seeds_off[p];
      return pl->own_dst() ? pl->pe[p].L[l].dst : pl->pe[p].L[l - 1].src;
    };
    // input rows of every part, requester-aligned (load_rows + all_to_all_forward)
    prepare_rows(pl, f);
    enqueue_gather(pl, f);
    std::vector<std::vector<double*>> hin(L, std::vector<double*>(P)), agg(L, std::vector<double*>(P)),
        out(L, std::vector<double*>(P));
    std::vector<std::vector<uint32_t*>> deg(L, std::vector<uint32_t*>(P));
    for (int l = L - 1; l >= 0; --l) {
      const uint32_t din = m->rows[l], dout = m->cols[l];
      const bool act = (l > 0) && m->tanh_hidden;
      for (uint32_t p = 0; p < P; ++p) {
        const LayerBufs& b = pl->pe[p].L[l];
        const uint64_t nd = M[p][l].n_dst, ne = M[p][l].n_edges;
        if (l == L - 1) hin[l][p] = static_cast<double*>(pl->pe[p].rows);
        else if (!coop) hin[l][p] = out[l + 1][p];
        deg[l][p] = A.get<uint32_t>(nd);
        CB_CUDA(cudaMemsetAsync(deg[l][p], 0, std::max<uint64_t>(nd, 1) * 4, st));
        launch_in_degrees(b.edges, ne, deg[l][p], st);
        uint64_t* off = A.get<uint64_t>(nd + 1);
        scan_counts(deg[l][p], nd, off, A, st);
        agg[l][p] = A.get<double>(nd * din);
        launch_aggregate(b.edges, deg[l][p], off, b.dst_pos, nd, hin[l][p], din, agg[l][p], st);
        out[l][p] = A.get<double>(nd * dout);
        launch_dense(agg[l][p], nd, din, m->w[l], dout, act, out[l][p], st);
      }
      if (coop && l > 0) {  // all_to_all_forward of block l's outputs to block l-1's sources
        const double** owners = A.get<const double*>(P);
        std::vector<const double*> h(out[l].begin(), out[l].end());
        CB_CUDA(cudaMemcpyAsync(owners, h.data(), P * sizeof(void*), cudaMemcpyHostToDevice, st));
        CB_CUDA(cudaStreamSynchronize(st));
        for (uint32_t p = 0; p < P; ++p) {
          const uint64_t ns = M[p][l - 1].n_src;
          hin[l - 1][p] = A.get<double>(ns * dout);
          launch_row_forward(owners, pl->pe[p].loc_part[l - 1], pl->pe[p].loc_row[l - 1], ns,
                             dout, hin[l - 1][p], st);
        }
      }
    }
    // loss on the seeds, gradient rows scaled by the global mean
    const double scale = 1.0 / static_cast<double>(total_seeds);
    const uint32_t C = classes;
    std::vector<std::vector<double*>> grad(L + 1, std::vector<double*>(P, nullptr));
    double loss_sum = 0.0;
    for (uint32_t p = 0; p < P; ++p) {
      const uint64_t n0 = M[p][0].n_dst;
      double* rl = A.get<double>(n0);
      grad[0][p] = A.get<double>(n0 * C);
      launch_softmax_ce(out[0][p], n0, C, dst_of(p, 0), f->seed, f->labels, scale, rl, grad[0][p],
                        st);
      std::vector<double> h(n0);
      if (n0) CB_CUDA(cudaMemcpyAsync(h.data(), rl, n0 * 8, cudaMemcpyDeviceToHost, st));
      CB_CUDA(cudaStreamSynchronize(st));
      for (double x : h) loss_sum += x;
    }
    *loss_out = loss_sum * scale;
    // backward with owner-side gradient accumulation between layers
    uint64_t gw_off = 0;
    for (int l = 0; l < L; ++l) {
      const uint32_t din = m->rows[l], dout = m->cols[l];
      const bool act = (l > 0) && m->tanh_hidden;
      const uint64_t nw = static_cast<uint64_t>(din) * dout;
      double* gw = A.get<double>(nw);
      CB_CUDA(cudaMemsetAsync(gw, 0, nw * 8, st));
      double* gwp = A.get<double>(nw);
      uint64_t req_total = 0;
      std::vector<uint64_t> req_off(P + 1, 0);
      for (uint32_t p = 0; p < P; ++p) req_off[p + 1] = req_off[p] + M[p][l].n_src;
      req_total = req_off[P];
      double* gh_all = A.get<double>(req_total * din);
      for (uint32_t p = 0; p < P; ++p) {
        const LayerBufs& b = pl->pe[p].L[l];
        const uint64_t nd = M[p][l].n_dst, ne = M[p][l].n_edges, ns = M[p][l].n_src;
        double* dp = grad[l][p];
        if (act) launch_tanh_grad(out[l][p], nd * dout, dp, st);
        launch_grad_w(agg[l][p], dp, nd, din, dout, gwp, st);
        launch_add(gw, gwp, nw, st);  // parts in order (the simulated all-reduce)
        double* dagg = A.get<double>(nd * din);
        launch_grad_agg(dp, m->w[l], nd, din, dout, dagg, st);
        // sources' edges in edge order (stable CSC) + the isolated dst of each source
        uint32_t* cnt = A.get<uint32_t>(ns);
        CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(ns, 1) * 4, st));
        uint32_t* key = A.get<uint32_t>(ne);
        uint32_t* val = A.get<uint32_t>(ne);
        uint32_t* key2 = A.get<uint32_t>(ne);
        uint32_t* val2 = A.get<uint32_t>(ne);
        if (ne) src_hist_kernel<<<grid_of_n(ne), 256, 0, st>>>(b.edges, ne, cnt, key, val);
        CB_LAUNCH("src_hist");
        uint64_t* soff = A.get<uint64_t>(ns + 1);
        scan_counts(cnt, ns, soff, A, st);
        cub::DoubleBuffer<uint32_t> kb(key, key2), vb(val, val2);
        size_t bytes = 0;
        CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, static_cast<int64_t>(ne), 0,
                                                32, st));
        void* tmp = A.get<unsigned char>(bytes);
        CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int64_t>(ne), 0, 32,
                                                st));
        int64_t* iso = A.get<int64_t>(ns);
        CB_CUDA(cudaMemsetAsync(iso, 0xff, std::max<uint64_t>(ns, 1) * 8, st));
        launch_iso_dst(deg[l][p], b.dst_pos, nd, iso, st);
        launch_grad_h_in(b.edges, vb.Current(), soff, deg[l][p], iso, ns, dagg, din,
                         gh_all + req_off[p] * din, st);
      }
      if (grad_w_out)
        CB_CUDA(cudaMemcpyAsync(grad_w_out + gw_off, gw, nw * 8, cudaMemcpyDeviceToHost, st));
      gw_off += nw;
      if (l + 1 < L) {
        if (!coop) {
          for (uint32_t p = 0; p < P; ++p) grad[l + 1][p] = gh_all + req_off[p] * din;
        } else {  // all_to_all_reverse_sum over the exchange of layer l
          std::vector<uint64_t> obase(P + 1, 0);
          for (uint32_t q = 0; q < P; ++q) obase[q + 1] = obase[q] + M[q][l + 1].n_dst;
          const uint64_t no = obase[P];
          uint64_t* d_obase = A.get<uint64_t>(P + 1);
          CB_CUDA(cudaMemcpyAsync(d_obase, obase.data(), (P + 1) * 8, cudaMemcpyHostToDevice, st));
          uint32_t* cnt = A.get<uint32_t>(no);
          CB_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(no, 1) * 4, st));
          uint64_t* key = A.get<uint64_t>(req_total);
          uint64_t* val = A.get<uint64_t>(req_total);
          uint64_t* key2 = A.get<uint64_t>(req_total);
          uint64_t* val2 = A.get<uint64_t>(req_total);
          for (uint32_t p = 0; p < P; ++p) {
            const uint64_t ns = M[p][l].n_src;
            if (ns)
              owner_key_kernel<<<grid_of_n(ns), 256, 0, st>>>(
                  pl->pe[p].loc_part[l], pl->pe[p].loc_row[l], ns, d_obase, req_off[p], cnt, key,
                  val);
            CB_LAUNCH("owner_key");
          }
          uint64_t* ooff = A.get<uint64_t>(no + 1);
          scan_counts(cnt, no, ooff, A, st);
          cub::DoubleBuffer<uint64_t> kb(key, key2), vb(val, val2);
          size_t bytes = 0;
          CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb,
                                                  static_cast<int64_t>(req_total), 0, 64, st));
          void* tmp = A.get<unsigned char>(bytes);
          CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb,
                                                  static_cast<int64_t>(req_total), 0, 64, st));
          double* oall = A.get<double>(no * din);
          launch_reverse_sum(ooff, vb.Current(), no, gh_all, din, oall, st);
          for (uint32_t q = 0; q < P; ++q) grad[l + 1][q] = oall + obase[q] * din;
        }
      }
    }
    CB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
