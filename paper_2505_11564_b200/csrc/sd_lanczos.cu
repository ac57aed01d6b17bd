// Device Lanczos engine: lanczos_run of SPEC.md:257-265 / PAPER.md Alg. 2 with
// full reorthogonalisation as two classical Gram-Schmidt passes over every
// stored column. Each step is:
//   r = op(q_k)                                        (HVP / dense apply)
//   pass A: r -= beta_{k-1} q_{k-1};  partial <q_k, r>   -> alpha_k
//   pass B: r -= alpha_k q_k           [no reorth: partial <r, r> -> beta_k]
//   CGS 1 : partials <Q_i, r>                           -> c   (j columns)
//   CGS 2 : r -= sum_i c_i Q_i (sequential); <Q_i, r>    -> c'
//   CGS 3 : r -= sum_i c'_i Q_i;            <r, r>       -> beta_k
//   q_{k+1} = (1/beta_k) r
// Scalars never leave the device inside a step; partials are exchanged with
// one all-gather per scalar set and folded in rank order (bitwise equal to
// the reference's coordinator fold for any rank count). alpha/beta reach the
// host once per step for the breakdown test (beta < eps).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "sd_common.cuh"
#include "sd_engine.h"

namespace {

constexpr uint64_t kAlign = 256;
uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Plan {
  uint64_t P = 0, ldq = 0, esize = 0, ncols_alloc = 0, pstride = 0, m_max = 0, maxlen = 0;
  uint64_t off_Q = 0, off_r = 0, off_xfull = 0, off_send = 0, off_recv = 0, off_scal = 0, off_part = 0,
           total_bytes = 0;
  bool tree = false;
};

Plan make_plan(const uint64_t* begins, const uint64_t* ends, uint64_t total, const sd_lanczos_config* cfg, int nranks,
               int rank) {
  Plan p;
  if (!cfg) sd::fail(SD_CONFIG_ERROR, "null lanczos config");
  if (cfg->k_max < 1) sd::fail(SD_CONFIG_ERROR, "k_max must be >= 1");
  if (cfg->prec != SD_F32 && cfg->prec != SD_F64) sd::fail(SD_CONFIG_ERROR, "precision must be f32 or f64");
  if (cfg->reorth != SD_REORTH_NONE && cfg->reorth != SD_REORTH_FULL && cfg->reorth != SD_REORTH_SELECTIVE)
    sd::fail(SD_CONFIG_ERROR, "reorth must be none, full or selective");
  if (cfg->reorth == SD_REORTH_SELECTIVE && cfg->selective_window < 2)
    sd::fail(SD_CONFIG_ERROR, "selective reorthogonalisation needs a window >= 2");
  if (cfg->reduction != SD_REDUCE_ORDERED && cfg->reduction != SD_REDUCE_TREE)
    sd::fail(SD_CONFIG_ERROR, "reduction must be ordered or tree");
  if (nranks < 1 || rank < 0 || rank >= nranks) sd::fail(SD_ARGUMENT_ERROR, "bad rank/size");
  uint64_t at = 0;
  for (int r = 0; r < nranks; ++r) {
    if (begins[r] != at || !(ends[r] > begins[r])) sd::fail(SD_LAYOUT_ERROR, "shard bounds leave a gap or overlap");
    at = ends[r];
    p.pstride = std::max<uint64_t>(p.pstride, sd::partial_shape(begins[r], ends[r], total).len());
    p.maxlen = std::max<uint64_t>(p.maxlen, ends[r] - begins[r]);
  }
  if (at != total) sd::fail(SD_LAYOUT_ERROR, "shard bounds do not cover total_dim");
  p.P = ends[rank] - begins[rank];
  p.ldq = (p.P + 31) / 32 * 32;  // 128-byte aligned columns (TMA boxes in tree mode)
  p.esize = cfg->prec == SD_F32 ? 4 : 8;
  p.tree = cfg->reduction == SD_REDUCE_TREE;
  const bool keep = cfg->reorth == SD_REORTH_FULL;
  const bool sel = cfg->reorth == SD_REORTH_SELECTIVE;
  const uint64_t W = std::min<uint64_t>(cfg->selective_window, cfg->k_max + 1);
  p.ncols_alloc = keep ? cfg->k_max + 1 : (sel ? std::max<uint64_t>(W, 2) : 2);
  p.m_max = keep ? cfg->k_max + 1 : (sel ? std::max<uint64_t>(W, 2) : 1);
  if (p.tree) {
    p.m_max = std::max<uint64_t>(p.m_max, 2);
    if (p.ncols_alloc > 256)
      sd::fail(SD_CONFIG_ERROR, "tree reduction keeps at most 256 basis columns (k_max <= 255 with full reorth)");
  }
  uint64_t o = 0;
  p.off_Q = o;
  o = align_up(o + p.ncols_alloc * p.ldq * p.esize);
  p.off_r = o;
  o = align_up(o + p.P * p.esize);
  p.off_xfull = o;
  o = align_up(o + (nranks > 1 ? (uint64_t(nranks) * p.maxlen + total) * p.esize : 0));
  p.off_send = o;
  o = align_up(o + p.m_max * p.pstride * 8);
  p.off_recv = o;
  o = align_up(o + (nranks > 1 ? uint64_t(nranks) * p.m_max * p.pstride * 8 : 0));
  p.off_scal = o;
  o = align_up(o + (4 + 2 * cfg->k_max + 2 * p.m_max) * 8);
  p.off_part = o;
  if (p.tree) o = align_up(o + sd::tree_part_bytes(p.P));
  p.total_bytes = o;
  return p;
}

}  // namespace

struct sd_lanczos_s {
  sd_operator op = nullptr;
  sd_comm comm = nullptr;
  int nranks = 1, rank = 0;
  std::vector<uint64_t> rb, re;
  uint64_t total = 0;
  sd_lanczos_config cfg{};
  Plan plan;
  char* ws = nullptr;
  cudaStream_t s = nullptr;
  double eps = 0;
  uint64_t k = 0, ncols = 0;
  bool done = false, breakdown = false, failure = false;
  std::vector<double> alphas, betas;
  double* h_scal = nullptr;  // pinned: [alpha, beta]
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double ms_apply = 0, ms_rec = 0, ms_reorth = 0;

  // full: column i in slot i; selective: a ring of W slots (column i in slot
  // i % W, swept in slot order -- oracle/src/core.cpp lanczos_run); none: 2 slots
  void* col(uint64_t i) const {
    const uint64_t slot = cfg.reorth == SD_REORTH_FULL ? i
                          : cfg.reorth == SD_REORTH_SELECTIVE ? i % plan.ncols_alloc
                                                              : (i & 1);
    return ws + plan.off_Q + slot * plan.ldq * plan.esize;
  }
  uint64_t slot_of(uint64_t i) const {
    return cfg.reorth == SD_REORTH_FULL ? i : cfg.reorth == SD_REORTH_SELECTIVE ? i % plan.ncols_alloc : (i & 1);
  }
  double* part() const { return reinterpret_cast<double*>(ws + plan.off_part); }
  unsigned* counter() const {
    return reinterpret_cast<unsigned*>(ws + plan.off_part + sd::tree_part_bytes(plan.P) - 256);
  }
  void* r() const { return ws + plan.off_r; }
  double* send() const { return reinterpret_cast<double*>(ws + plan.off_send); }
  double* recv() const { return reinterpret_cast<double*>(ws + plan.off_recv); }
  double* scal() const { return reinterpret_cast<double*>(ws + plan.off_scal); }
  double* d_alpha() const { return scal() + 4; }                    // [k_max]
  double* d_beta() const { return scal() + 4 + cfg.k_max; }         // [k_max]
  double* d_c1() const { return scal() + 4 + 2 * cfg.k_max; }       // [m_max]
  double* d_c2() const { return d_c1() + plan.m_max; }              // [m_max]
  double* d_norm() const { return scal(); }
  uint64_t begin() const { return rb[rank]; }
  uint64_t end() const { return re[rank]; }

  // all-gather the m partial sequences and fold them in rank order
  void reduce(uint64_t m, double* out, int post_sqrt) {
    const double* parts = send();
    if (nranks > 1) {
      sd::comm_allgather(comm, send(), recv(), m * plan.pstride * 8, s);
      parts = recv();
    }
    sd::combine_device(uint64_t(nranks), rb.data(), re.data(), total, m, plan.pstride, parts, out, s, post_sqrt);
  }

  void apply(const void* x, void* y) {
    if (sd::operator_needs_full(op)) {
      const void* xf = x;
      if (nranks > 1) {
        // gather (operators.cpp:35): fixed-size all-gather of padded shards, then compact
        const uint64_t maxlen = plan.maxlen;
        char* gat = ws + plan.off_xfull;
        char* full = gat + uint64_t(nranks) * maxlen * plan.esize;
        char* sendbuf = gat + uint64_t(rank) * maxlen * plan.esize;
        SD_CUDA(cudaMemcpyAsync(sendbuf, x, plan.P * plan.esize, cudaMemcpyDeviceToDevice, s));
        sd::comm_allgather(comm, sendbuf, gat, maxlen * plan.esize, s);
        for (int q = 0; q < nranks; ++q)
          SD_CUDA(cudaMemcpyAsync(full + rb[q] * plan.esize, gat + uint64_t(q) * maxlen * plan.esize,
                                  (re[q] - rb[q]) * plan.esize, cudaMemcpyDeviceToDevice, s));
        xf = full;
      }
      sd::operator_apply(op, x, y, cfg.prec, s, begin(), end(), xf);
    } else {
      sd::operator_apply(op, x, y, cfg.prec, s, begin(), end(), nullptr);
    }
  }

  void start() {
    const uint64_t B = begin(), E = end();
    void* q0 = col(0);
    sd::probe_fill(q0, B, E, cfg.probe_seed, cfg.probe_dist, 0, cfg.prec, s);
    // normalise: n = norm2(q0); !(n > 0) -> numerical_error; q0 = scale(q0, 1/n) (sharded.cpp:77-81)
    sd::axpy_dot(nullptr, q0, nullptr, nullptr, B, E, total, cfg.prec, send(), s);
    reduce(1, d_norm(), 1);
    SD_CUDA(cudaMemcpyAsync(h_scal, d_norm(), 8, cudaMemcpyDeviceToHost, s));
    sd::comm_wait(comm, s);
    if (!(h_scal[0] > 0.0)) sd::fail(SD_NUMERICAL_ERROR, "probe has zero norm");
    sd::scale(q0, q0, plan.P, d_norm(), 1, cfg.prec, s);
    ncols = 1;
  }

  // one tree-mode pass over `jb` slots starting at slot 0; m results land in
  // `out` (rank-ordered fold of the ranks' results when sharded)
  void tpass(int mode, int jb, int ucol, int xcol, const double* coef, double* out, int m, int post_sqrt,
             double* alpha_out, int alpha_col, const void* base = nullptr) {
    const void* Q = base ? base : col(0);
    if (nranks == 1) {
      sd::tree_pass(cfg.prec, mode, Q, plan.ldq, jb, r(), plan.P, coef, ucol, xcol, part(), counter(), out, alpha_out,
                    alpha_col, post_sqrt, s);
      return;
    }
    sd::tree_pass(cfg.prec, mode, Q, plan.ldq, jb, r(), plan.P, coef, ucol, xcol, part(), counter(), send(), nullptr,
                  -1, 0, s);
    sd::comm_allgather(comm, send(), recv(), uint64_t(m) * 8, s);
    sd::tree_rank_fold(recv(), nranks, m, out, post_sqrt, alpha_out, alpha_col, s);
  }

  void step_tree() {
    void* q = col(k);
    SD_CUDA(cudaEventRecord(ev[0], s));
    apply(q, r());
    SD_CUDA(cudaEventRecord(ev[1], s));
    const int up = k > 0 ? int(slot_of(k - 1)) : -1;
    const double* bcoef = k > 0 ? d_beta() + (k - 1) : nullptr;
    if (cfg.reorth == SD_REORTH_NONE) {
      // r -= beta q_{k-1}; dots with {slot 0, slot 1}; alpha = the q_k one
      const int jb = k > 0 ? 2 : 1;
      tpass(0, jb, up, -1, bcoef, d_c1(), jb, 0, d_alpha() + k, int(slot_of(k)));
      SD_CUDA(cudaEventRecord(ev[2], s));
      // r -= alpha q_k (in f64: the dominant column); beta = ||r||
      tpass(2, 1, 0, 0, d_alpha() + k, d_beta() + k, 1, 1, nullptr, -1, q);
    } else {
      const int jb = int(ncols);
      tpass(0, jb, up, -1, bcoef, d_c1(), jb, 0, d_alpha() + k, int(slot_of(k)));
      SD_CUDA(cudaEventRecord(ev[2], s));
      // first Gram-Schmidt pass: q_k's coefficient (alpha) is the dominant one
      tpass(1, jb, 0, int(slot_of(k)), d_c1(), d_c2(), jb, 0, nullptr, -1);
      tpass(2, jb, 0, -1, d_c2(), d_beta() + k, 1, 1, nullptr, -1);
    }
    SD_CUDA(cudaEventRecord(ev[3], s));
  }

  void step() {
    if (done) return;
    if (plan.tree) {
      step_tree();
      finish_step();
      return;
    }
    const uint64_t B = begin(), E = end();
    void* q = col(k);
    void* qp = k > 0 ? col(k - 1) : nullptr;
    SD_CUDA(cudaEventRecord(ev[0], s));
    apply(q, r());
    SD_CUDA(cudaEventRecord(ev[1], s));
    // pass A: r = axpy(-beta_{k-1}, q_{k-1}, r); alpha = dot(q_k, r)
    sd::axpy_dot(qp, r(), q, k > 0 ? d_beta() + (k - 1) : nullptr, B, E, total, cfg.prec, send(), s);
    reduce(1, d_alpha() + k, 0);
    if (cfg.reorth == SD_REORTH_NONE) {
      // pass B: r = axpy(-alpha, q_k, r); beta = norm2(r)
      sd::axpy_dot(q, r(), nullptr, d_alpha() + k, B, E, total, cfg.prec, send(), s);
      reduce(1, d_beta() + k, 1);
      SD_CUDA(cudaEventRecord(ev[2], s));
    } else {
      sd::axpy_dot(q, r(), nullptr, d_alpha() + k, B, E, total, cfg.prec, nullptr, s);
      SD_CUDA(cudaEventRecord(ev[2], s));
      const uint64_t j = ncols;
      sd::cgs(col(0), plan.ldq, j, r(), nullptr, 1, B, E, total, cfg.prec, send(), plan.pstride, s);
      reduce(j, d_c1(), 0);
      sd::cgs(col(0), plan.ldq, j, r(), d_c1(), 1, B, E, total, cfg.prec, send(), plan.pstride, s);
      reduce(j, d_c2(), 0);
      sd::cgs(col(0), plan.ldq, j, r(), d_c2(), 2, B, E, total, cfg.prec, send(), plan.pstride, s);
      reduce(1, d_beta() + k, 1);
    }
    SD_CUDA(cudaEventRecord(ev[3], s));
    finish_step();
  }

  // alpha/beta to the host, breakdown test, q_{k+1} = scale(r, 1/beta)
  void finish_step() {
    SD_CUDA(cudaMemcpyAsync(h_scal, d_alpha() + k, 8, cudaMemcpyDeviceToHost, s));
    SD_CUDA(cudaMemcpyAsync(h_scal + 1, d_beta() + k, 8, cudaMemcpyDeviceToHost, s));
    sd::comm_wait(comm, s);  // NCCL: async errors / timeouts -> SD_NCCL_ERROR, not a hang
    float t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t12, ev[1], ev[2]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    ms_apply += t01;
    ms_rec += t12;
    ms_reorth += t23;
    const double alpha = h_scal[0], beta = h_scal[1];
    if (!std::isfinite(alpha)) {
      failure = done = true;
      return;
    }
    alphas.push_back(alpha);
    if (!std::isfinite(beta)) {
      failure = done = true;
      return;
    }
    if (beta < eps) {
      breakdown = done = true;
      return;
    }
    if (k + 1 == cfg.k_max) {
      done = true;
      return;
    }
    betas.push_back(beta);
    // q_{k+1} = scale(r, 1/beta)
    sd::scale(r(), col(k + 1), plan.P, d_beta() + k, 1, cfg.prec, s);
    ++k;
    if (cfg.reorth == SD_REORTH_FULL) ++ncols;
    if (cfg.reorth == SD_REORTH_SELECTIVE) ncols = std::min<uint64_t>(ncols + 1, plan.ncols_alloc);
  }

  ~sd_lanczos_s() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (h_scal) cudaFreeHost(h_scal);
  }
};

namespace sd {
bool operator_needs_full(sd_operator op);
}

extern "C" {

uint64_t sd_lanczos_workspace_bytes(const uint64_t* begins, const uint64_t* ends, uint64_t total,
                                    const sd_lanczos_config* cfg, int nranks, int rank) {
  try {
    return make_plan(begins, ends, total, cfg, nranks, rank).total_bytes;
  } catch (const std::exception& e) {
    sd::set_last_error(e.what());
    return 0;
  }
}

sd_status sd_lanczos_begin(sd_operator op, sd_comm comm, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                           const sd_lanczos_config* cfg, void* workspace, uint64_t workspace_bytes, sd_stream s,
                           sd_lanczos* out) {
  return sd::guard([&] {
    if (!op) sd::fail(SD_ARGUMENT_ERROR, "null operator");
    const int nr = sd::comm_size(comm), rk = sd::comm_rank(comm);
    auto L = std::make_unique<sd_lanczos_s>();
    L->plan = make_plan(begins, ends, total, cfg, nr, rk);
    if (sd_operator_dim(op) != total) sd::fail(SD_LAYOUT_ERROR, "operator/vector dimension mismatch");
    if (total < 2) sd::fail(SD_ARGUMENT_ERROR, "operator dimension must be >= 2");
    if (workspace_bytes < L->plan.total_bytes) sd::fail(SD_ARGUMENT_ERROR, "lanczos workspace too small");
    L->op = op;
    L->comm = comm;
    L->nranks = nr;
    L->rank = rk;
    L->rb.assign(begins, begins + nr);
    L->re.assign(ends, ends + nr);
    L->total = total;
    L->cfg = *cfg;
    L->ws = static_cast<char*>(workspace);
    L->s = (cudaStream_t)s;
    L->eps = cfg->eps > 0 ? cfg->eps : (cfg->prec == SD_F64 ? 1e-12 : 1e-7);
    SD_CUDA(cudaMallocHost(&L->h_scal, 2 * sizeof(double)));
    if (L->plan.tree) SD_CUDA(cudaMemsetAsync(L->counter(), 0, 256, L->s));
    for (auto& e : L->ev) SD_CUDA(cudaEventCreate(&e));
    L->start();
    *out = L.release();
  });
}

sd_status sd_lanczos_step(sd_lanczos L, int* done) {
  return sd::guard([&] {
    L->step();
    if (done) *done = L->done ? 1 : 0;
  });
}

sd_status sd_lanczos_result(sd_lanczos L, double* alphas, double* betas, sd_lanczos_info* info) {
  return sd::guard([&] {
    for (size_t i = 0; i < L->alphas.size(); ++i) alphas[i] = L->alphas[i];
    for (size_t i = 0; i < L->betas.size(); ++i) betas[i] = L->betas[i];
    if (info) {
      info->n_alpha = L->alphas.size();
      info->n_beta = L->betas.size();
      info->breakdown = L->breakdown;
      info->numerical_failure = L->failure;
      info->ms_apply = L->ms_apply;
      info->ms_recurrence = L->ms_rec;
      info->ms_reorth = L->ms_reorth;
      info->ms_comm = 0;
    }
  });
}

const void* sd_lanczos_current(sd_lanczos L) { return L ? L->col(L->k) : nullptr; }
uint64_t sd_lanczos_basis_ld(sd_lanczos L) { return L ? L->plan.ldq : 0; }

sd_status sd_lanczos_basis(sd_lanczos L, const void** basis, uint64_t* ncols) {
  return sd::guard([&] {
    if (L->cfg.reorth != SD_REORTH_FULL) sd::fail(SD_STATE_ERROR, "basis was not stored (reorth = none)");
    *basis = L->col(0);
    *ncols = L->ncols;
  });
}

// loss_of_orthogonality: max_{i != j} |q_i^T q_j| over the
// stored columns, every dot the reference's blocked f64 fold (rank-ordered
// across shards); column i is dotted against columns 0..i-1 in one pass.
sd_status sd_lanczos_orthogonality(sd_lanczos L, double* out) {
  return sd::guard([&] {
    if (!L || !out) sd::fail(SD_ARGUMENT_ERROR, "null argument");
    if (L->cfg.reorth != SD_REORTH_FULL) sd::fail(SD_STATE_ERROR, "basis was not stored (reorth = none)");
    const uint64_t B = L->begin(), E = L->end();
    double worst = 0.0;
    std::vector<double> h(L->plan.m_max);
    for (uint64_t i = 1; i < L->ncols; ++i) {
      sd::cgs(L->col(0), L->plan.ldq, i, L->col(i), nullptr, 1, B, E, L->total, L->cfg.prec, L->send(),
              L->plan.pstride, L->s);
      L->reduce(i, L->d_c1(), 0);
      SD_CUDA(cudaMemcpyAsync(h.data(), L->d_c1(), i * sizeof(double), cudaMemcpyDeviceToHost, L->s));
      SD_CUDA(cudaStreamSynchronize(L->s));
      for (uint64_t j = 0; j < i; ++j) worst = std::max(worst, std::fabs(h[j]));
    }
    *out = worst;
  });
}

sd_status sd_lanczos_end(sd_lanczos L) {
  return sd::guard([&] { delete L; });
}

sd_status sd_lanczos_run(sd_operator op, sd_comm comm, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                         const sd_lanczos_config* cfg, void* workspace, uint64_t workspace_bytes, double* alphas,
                         double* betas, sd_lanczos_info* info, sd_stream s) {
  sd_lanczos L = nullptr;
  sd_status st = sd_lanczos_begin(op, comm, begins, ends, total, cfg, workspace, workspace_bytes, s, &L);
  if (st != SD_OK) return st;
  int done = 0;
  while (!done && st == SD_OK) st = sd_lanczos_step(L, &done);
  if (st == SD_OK) st = sd_lanczos_result(L, alphas, betas, info);
  if (st == SD_OK && L->failure) {
    sd::set_last_error("non-finite alpha or beta (partial tridiagonal returned)");
    st = SD_NUMERICAL_ERROR;
  }
  delete L;
  return st;
}

}  // extern "C"
