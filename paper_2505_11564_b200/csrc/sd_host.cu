// Host side of libspecden_b200: error plumbing, layout bookkeeping, the
// tridiagonal eigensolve + quadrature (stays on the host),
// NCCL communicators, operator handles and the device Lanczos engine
// (Alg. 2) that drives the kernels of sd_vector.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <cmath>
#include <chrono>
#include <cstring>
#include <thread>
#include <memory>
#include <string>
#include <vector>

#include "sd_common.cuh"
#include "sd_engine.h"

namespace sd {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------------ layout
static void validate(uint64_t total, uint64_t n, const uint64_t* b, const uint64_t* e) {
  if (total == 0) fail(SD_LAYOUT_ERROR, "layout covers zero dimensions");
  if (n == 0) fail(SD_LAYOUT_ERROR, "layout has no shards");
  uint64_t at = 0;
  for (uint64_t w = 0; w < n; ++w) {
    if (b[w] != at) fail(SD_LAYOUT_ERROR, "shard bounds leave a gap or overlap");
    if (!(e[w] > b[w])) fail(SD_LAYOUT_ERROR, "empty shard range");
    at = e[w];
  }
  if (at != total) fail(SD_LAYOUT_ERROR, "shard bounds do not cover total_dim");
}

// ------------------------------------------------------------- quadrature
// Implicit-shift QL on the symmetric tridiagonal with accumulated rotations
// (the textbook tql2/tqli iteration), f64. Returns eigenvalues ascending and
// the full eigenvector matrix (column-major k x k).
static void tridiag_ql(std::vector<double>& d, std::vector<double> e, std::vector<double>& z) {
  const size_t k = d.size();
  z.assign(k * k, 0.0);
  for (size_t i = 0; i < k; ++i) z[i * k + i] = 1.0;
  e.resize(k, 0.0);
  for (size_t l = 0; l < k; ++l) {
    int iter = 0;
    size_t m;
    do {
      for (m = l; m + 1 < k; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= std::numeric_limits<double>::epsilon() * dd) break;
      }
      if (m != l) {
        if (iter++ == 200) fail(SD_NUMERICAL_ERROR, "tridiagonal QL did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        bool early = false;
        for (size_t ii = m; ii-- > l;) {
          double f = s * e[ii];
          const double b = c * e[ii];
          r = std::hypot(f, g);
          e[ii + 1] = r;
          if (r == 0.0) {
            d[ii + 1] -= p;
            e[m] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[ii + 1] - p;
          r = (d[ii] - g) * s + 2.0 * c * b;
          p = s * r;
          d[ii + 1] = g + p;
          g = c * r - b;
          for (size_t row = 0; row < k; ++row) {  // column-major: z[col*k + row]
            f = z[(ii + 1) * k + row];
            z[(ii + 1) * k + row] = s * z[ii * k + row] + c * f;
            z[ii * k + row] = c * z[ii * k + row] - s * f;
          }
        }
        if (early) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
}

void ritz(uint64_t k, const double* al, const double* be, double* vals, double* wts, double* resid) {
  if (k == 0) fail(SD_ARGUMENT_ERROR, "ritz_decompose needs k >= 1");
  for (uint64_t i = 0; i < k; ++i)
    if (!std::isfinite(al[i]) || (i + 1 < k && !std::isfinite(be[i])))
      fail(SD_NUMERICAL_ERROR, "non-finite tridiagonal entry");
  std::vector<double> d(al, al + k), e(be, be + (k - 1)), z;
  tridiag_ql(d, e, z);
  std::vector<size_t> idx(k);
  for (size_t i = 0; i < k; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return d[a] < d[b]; });
  double tnorm = 0.0;
  for (uint64_t i = 0; i < k; ++i)
    tnorm = std::max(tnorm, std::fabs(al[i]) + (i ? std::fabs(be[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(be[i]) : 0.0));
  double worst = 0.0;
  for (size_t o = 0; o < k; ++o) {
    const size_t c = idx[o];
    const double* y = &z[c * k];
    double n2 = 0.0;
    for (size_t r = 0; r < k; ++r) n2 += y[r] * y[r];
    vals[o] = d[c];
    wts[o] = y[0] * y[0] / n2;
    double res = 0.0;
    for (size_t r = 0; r < k; ++r) {
      double ty = al[r] * y[r];
      if (r > 0) ty += be[r - 1] * y[r - 1];
      if (r + 1 < k) ty += be[r] * y[r + 1];
      const double dlt = ty - d[c] * y[r];
      res += dlt * dlt;
    }
    worst = std::max(worst, std::sqrt(res / n2));
  }
  if (resid) *resid = tnorm > 0 ? worst / tnorm : worst;
}

void density(uint64_t k, const double* v, const double* w, double sigma, uint64_t npts, double* grid, double* dens,
             double* sig_used) {
  if (k == 0) fail(SD_ARGUMENT_ERROR, "degenerate spectrum (k = 0)");
  if (npts < 2) fail(SD_ARGUMENT_ERROR, "grid_points must be >= 2");
  const double lo = *std::min_element(v, v + k), hi = *std::max_element(v, v + k);
  if (!(sigma > 0)) sigma = (hi - lo) / 100.0;
  if (!(sigma > 0)) sigma = 1.0;
  const double a = lo - 5 * sigma, b = hi + 5 * sigma;
  const double norm = 1.0 / (sigma * std::sqrt(2.0 * M_PI));
  for (uint64_t g = 0; g < npts; ++g) {
    const double x = a + (b - a) * double(g) / double(npts - 1);
    double acc = 0.0;
    for (uint64_t i = 0; i < k; ++i) {
      const double t = (x - v[i]) / sigma;
      acc += w[i] * norm * std::exp(-0.5 * t * t);
    }
    grid[g] = x;
    dens[g] = acc;
  }
  if (sig_used) *sig_used = sigma;
}

// ------------------------------------------------------------------- NCCL
// NCCL is resolved at run time from the process (torch has usually loaded
// libnccl.so.2 already); the library never links a second copy.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};
static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(h, "ncclReduceScatter");
    a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.CommGetAsyncError = (decltype(a.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    a.CommAbort = (decltype(a.CommAbort))dlsym(h, "ncclCommAbort");
    return a;
  }();
  if (!api.CommInitRank) fail(SD_NCCL_ERROR, "libnccl.so.2 not loadable");
  return api;
}
static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SD_NCCL_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace sd

// In-process worker group (sd_comm_local_create): the reference's WorkerPool
// model -- n workers of ONE process, each a host thread with its own stream on
// the same device, exchanging through device copies between host barriers.
// No kernel ever waits on another worker's kernel: every exchange first
// synchronises the caller's stream, meets the other workers at a host
// barrier, then copies/reduces published buffers in rank order.
struct LocalMsg {
  const float* p = nullptr;
  uint64_t n = 0;
  bool done = false;
};
struct LocalGroup {
  int n = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> slot;
  // point-to-point: FIFO of posted sends per (src, dst); a send completes when
  // the receiver has copied it (blocking semantics, like NCCL's)
  std::vector<std::vector<std::deque<LocalMsg*>>> q;
  // a worker that fails outside a collective aborts the group, so that the
  // others leave their waits with a protocol error instead of hanging
  bool aborted = false;
  void check_abort() const {
    if (aborted) sd::fail(SD_PROTOCOL_ERROR, "worker group aborted by another worker's failure");
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    check_abort();
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      check_abort();
    }
  }
  void abort() {
    {
      std::lock_guard<std::mutex> lk(m);
      aborted = true;
    }
    cv.notify_all();
  }
};

struct LocalP2p {
  bool send;
  const float* sp;
  float* rp;
  uint64_t n;
  int peer;
};
struct sd_comm_s {
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  bool aborted = false;            // NCCL: aborted after an async error / timeout
  std::shared_ptr<LocalGroup> local;
  const float** d_ptrs = nullptr;  // local group: device copy of the published pointers
  bool in_group = false;           // local group: deferred point-to-point ops of a group
  std::vector<LocalP2p> pending;
  // NCCL rank-ordered reductions: receive slots of every rank's contribution
  float* ord_buf = nullptr;
  uint64_t ord_cap = 0;            // floats
  float* ord_tmp = nullptr;
  uint64_t ord_tmp_cap = 0;
};

namespace {
// out[i] = sum over q (rank order) of src[q][off + i]
__global__ void k_sum_ranks(const float* const* __restrict__ src, int nranks, uint64_t off, uint64_t n,
                            float* __restrict__ out) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  float acc = src[0][off + i];
  for (int q = 1; q < nranks; ++q) acc += src[q][off + i];
  out[i] = acc;
}

void local_publish(sd_comm c, const void* p, cudaStream_t s) {
  SD_CUDA(cudaStreamSynchronize(s));
  c->local->slot[c->rank] = p;
  c->local->barrier();
}

// rank-ordered sum of the published f32 buffers (at element offset off) into out
void local_sum(sd_comm c, uint64_t off, uint64_t n, float* out, cudaStream_t s) {
  if (!c->d_ptrs) SD_CUDA(cudaMalloc(&c->d_ptrs, sizeof(float*) * c->nranks));
  std::vector<const float*> h(c->nranks);
  for (int q = 0; q < c->nranks; ++q) h[q] = static_cast<const float*>(c->local->slot[q]);
  SD_CUDA(cudaMemcpyAsync(c->d_ptrs, h.data(), sizeof(float*) * c->nranks, cudaMemcpyHostToDevice, s));
  if (n) k_sum_ranks<<<unsigned((n + 255) / 256), 256, 0, s>>>(c->d_ptrs, c->nranks, off, n, out);
  SD_CUDA(cudaGetLastError());
}
// Point-to-point between in-process workers: all sends of a unit are posted
// (after the stream has produced them), then every receive waits for its
// matching send, copies it on the receiver's stream and acknowledges, then the
// unit waits for its own sends to be acknowledged. A group is one unit (the
// NCCL group semantics the 1F1B schedule relies on); a lone op is its own.
void local_p2p(sd_comm c, std::vector<LocalP2p>& ops, cudaStream_t s) {
  LocalGroup& g = *c->local;
  SD_CUDA(cudaStreamSynchronize(s));
  std::vector<LocalMsg> msgs(ops.size());
  {
    std::lock_guard<std::mutex> lk(g.m);
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].send) {
        msgs[i].p = ops[i].sp, msgs[i].n = ops[i].n;
        g.q[c->rank][ops[i].peer].push_back(&msgs[i]);
      }
  }
  g.cv.notify_all();
  for (auto& o : ops) {
    if (o.send) continue;
    LocalMsg* m = nullptr;
    {
      std::unique_lock<std::mutex> lk(g.m);
      g.cv.wait(lk, [&] { return !g.q[o.peer][c->rank].empty() || g.aborted; });
      g.check_abort();
      m = g.q[o.peer][c->rank].front();
      g.q[o.peer][c->rank].pop_front();
    }
    if (m->n != o.n) sd::fail(SD_PROTOCOL_ERROR, "point-to-point size mismatch");
    SD_CUDA(cudaMemcpyAsync(o.rp, m->p, o.n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    SD_CUDA(cudaStreamSynchronize(s));
    {
      std::lock_guard<std::mutex> lk(g.m);
      m->done = true;
    }
    g.cv.notify_all();
  }
  std::unique_lock<std::mutex> lk(g.m);
  for (size_t i = 0; i < ops.size(); ++i)
    if (ops[i].send) {
      g.cv.wait(lk, [&] { return msgs[i].done || g.aborted; });
      if (!msgs[i].done) {
        // withdraw the un-received message (it lives on this stack frame)
        for (auto& qq : g.q[c->rank])
          for (auto it = qq.begin(); it != qq.end();)
            it = (*it == &msgs[i]) ? qq.erase(it) : it + 1;
        g.check_abort();
      }
    }
}
}  // namespace

namespace sd {

// No communicator: single rank, the collectives are identities. A real
// communicator (even of one rank) always goes through NCCL.
void comm_allgather(sd_comm c, const void* send, void* recv, uint64_t bytes, cudaStream_t s) {
  if (!c) {
    if (recv != send) SD_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->local) {
    local_publish(c, send, s);
    for (int q = 0; q < c->nranks; ++q)
      SD_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + uint64_t(q) * bytes, c->local->slot[q], bytes,
                              cudaMemcpyDeviceToDevice, s));
    SD_CUDA(cudaStreamSynchronize(s));
    c->local->barrier();  // every worker has read every slot
    return;
  }
  nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, c->comm, s), "ncclAllGather");
}

// NCCL's own sum order depends on its algorithm (ring, tree, NVLS), so the
// engine's reductions over NCCL are rank-ordered instead (SD_NCCL_ORDERED=0
// restores ncclReduceScatter / ncclAllReduce): every rank sends each peer the
// slice it owns (one grouped send/recv round: the reduce-scatter's bytes) and
// sums the received contributions in ascending rank order -- the same fold as
// the in-process workers' k_sum_ranks, so Hv and everything downstream is
// bitwise independent of the transport and of NCCL's algorithm choice.
static bool nccl_ordered() {
  static const bool on = [] {
    const char* e = std::getenv("SD_NCCL_ORDERED");
    return !(e && e[0] == '0');
  }();
  return on;
}
static float* grow(float*& p, uint64_t& cap, uint64_t n) {
  if (cap < n) {
    if (p) SD_CUDA(cudaFree(p));
    SD_CUDA(cudaMalloc(&p, n * sizeof(float)));
    cap = n;
  }
  return p;
}
static void nccl_reducescatter_ordered(sd_comm c, const float* send, float* recv, uint64_t n, cudaStream_t s) {
  const int N = c->nranks;
  float* slots = grow(c->ord_buf, c->ord_cap, uint64_t(N) * n);
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < N; ++q) {
    nccl_check(nccl().Send(send + uint64_t(q) * n, n, ncclFloat32, q, c->comm, s), "ncclSend");
    nccl_check(nccl().Recv(slots + uint64_t(q) * n, n, ncclFloat32, q, c->comm, s), "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  if (!c->d_ptrs) SD_CUDA(cudaMalloc(&c->d_ptrs, sizeof(float*) * N));
  std::vector<const float*> h(N);
  for (int q = 0; q < N; ++q) h[q] = slots + uint64_t(q) * n;
  SD_CUDA(cudaMemcpyAsync(c->d_ptrs, h.data(), sizeof(float*) * N, cudaMemcpyHostToDevice, s));
  if (n) k_sum_ranks<<<unsigned((n + 255) / 256), 256, 0, s>>>(c->d_ptrs, N, 0, n, recv);
  SD_CUDA(cudaGetLastError());
}

void comm_allreduce_f32(sd_comm c, float* buf, uint64_t n, cudaStream_t s) {
  if (!c) return;
  if (c->comm && nccl_ordered() && c->nranks > 1) {
    // ordered reduce-scatter of padded chunks, then all-gather of the sums
    const int N = c->nranks;
    const uint64_t ch = (n + N - 1) / N;
    float* tmp = grow(c->ord_tmp, c->ord_tmp_cap, 2 * uint64_t(N) * ch);
    float *pad = tmp, *mine = tmp + uint64_t(N) * ch;
    SD_CUDA(cudaMemsetAsync(pad, 0, uint64_t(N) * ch * sizeof(float), s));
    SD_CUDA(cudaMemcpyAsync(pad, buf, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    nccl_reducescatter_ordered(c, pad, mine, ch, s);
    nccl_check(nccl().AllGather(mine, pad, ch, ncclFloat32, c->comm, s), "ncclAllGather");
    SD_CUDA(cudaMemcpyAsync(buf, pad, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->local) {
    float* tmp = nullptr;
    SD_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), s));
    local_publish(c, buf, s);
    local_sum(c, 0, n, tmp, s);
    SD_CUDA(cudaStreamSynchronize(s));
    c->local->barrier();  // all sums formed before any buffer is overwritten
    SD_CUDA(cudaMemcpyAsync(buf, tmp, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    SD_CUDA(cudaFreeAsync(tmp, s));
    return;
  }
  nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, c->comm, s), "ncclAllReduce");
}

// sum over ranks of send[r * n .. r * n + n) lands in rank r's recv[0 .. n)
void comm_reducescatter_f32(sd_comm c, const float* send, float* recv, uint64_t n, cudaStream_t s) {
  if (!c) {
    if (recv != send) SD_CUDA(cudaMemcpyAsync(recv, send, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->local) {
    local_publish(c, send, s);
    local_sum(c, uint64_t(c->rank) * n, n, recv, s);
    SD_CUDA(cudaStreamSynchronize(s));
    c->local->barrier();
    return;
  }
  if (nccl_ordered() && c->nranks > 1) return nccl_reducescatter_ordered(c, send, recv, n, s);
  if (!nccl().ReduceScatter) fail(SD_NCCL_ERROR, "ncclReduceScatter unavailable");
  nccl_check(nccl().ReduceScatter(send, recv, n, ncclFloat32, ncclSum, c->comm, s), "ncclReduceScatter");
}

// Variable-length exchanges of a sharded vector, straight between the slices
// (no padded slots): NCCL moves each slice with one grouped send/recv round,
// the in-process workers copy from the published buffers. The reduction sums
// the ranks' contributions in ascending rank order like k_sum_ranks above.
void comm_allgatherv_f32(sd_comm c, const float* mine, float* full, const uint64_t* rb, const uint64_t* re,
                         cudaStream_t s) {
  const int me = c ? c->rank : 0;
  if (full + rb[me] != mine && re[me] > rb[me])
    SD_CUDA(cudaMemcpyAsync(full + rb[me], mine, (re[me] - rb[me]) * sizeof(float), cudaMemcpyDeviceToDevice, s));
  if (!c || c->nranks == 1) return;
  if (c->local) {
    local_publish(c, mine, s);
    for (int q = 0; q < c->nranks; ++q)
      if (q != me && re[q] > rb[q])
        SD_CUDA(cudaMemcpyAsync(full + rb[q], c->local->slot[q], (re[q] - rb[q]) * sizeof(float),
                                cudaMemcpyDeviceToDevice, s));
    SD_CUDA(cudaStreamSynchronize(s));
    c->local->barrier();  // every worker has read every slice
    return;
  }
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < c->nranks; ++q) {
    if (q == me) continue;
    if (re[me] > rb[me]) nccl_check(nccl().Send(mine, re[me] - rb[me], ncclFloat32, q, c->comm, s), "ncclSend");
    if (re[q] > rb[q]) nccl_check(nccl().Recv(full + rb[q], re[q] - rb[q], ncclFloat32, q, c->comm, s), "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

void comm_reducescatterv_f32(sd_comm c, const float* full, float* mine, const uint64_t* rb, const uint64_t* re,
                             cudaStream_t s) {
  const int me = c ? c->rank : 0;
  const uint64_t n = re[me] - rb[me];
  if (!c || c->nranks == 1) {
    if (n && full + rb[me] != mine)
      SD_CUDA(cudaMemcpyAsync(mine, full + rb[me], n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->local) {
    local_publish(c, full, s);
    local_sum(c, rb[me], n, mine, s);
    SD_CUDA(cudaStreamSynchronize(s));
    c->local->barrier();
    return;
  }
  const int N = c->nranks;
  float* slots = grow(c->ord_buf, c->ord_cap, uint64_t(N) * n);
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < N; ++q) {
    if (q == me) continue;
    if (re[q] > rb[q]) nccl_check(nccl().Send(full + rb[q], re[q] - rb[q], ncclFloat32, q, c->comm, s), "ncclSend");
    if (n) nccl_check(nccl().Recv(slots + uint64_t(q) * n, n, ncclFloat32, q, c->comm, s), "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  if (!c->d_ptrs) SD_CUDA(cudaMalloc(&c->d_ptrs, sizeof(float*) * N));
  std::vector<const float*> h(N);
  for (int q = 0; q < N; ++q) h[q] = q == me ? full + rb[me] : slots + uint64_t(q) * n;
  SD_CUDA(cudaMemcpyAsync(c->d_ptrs, h.data(), sizeof(float*) * N, cudaMemcpyHostToDevice, s));
  if (n) k_sum_ranks<<<unsigned((n + 255) / 256), 256, 0, s>>>(c->d_ptrs, N, 0, n, mine);
  SD_CUDA(cudaGetLastError());
}

// Point-to-point (pipeline stages): f32 payloads to/from a peer rank; between
// group_begin/group_end the sends and receives progress together (NCCL group
// semantics), which is what makes the 1F1B exchanges deadlock-free.
void comm_send_f32(sd_comm c, const float* buf, uint64_t n, int peer, cudaStream_t s) {
  if (c && c->local) {
    if (peer < 0 || peer >= c->nranks || peer == c->rank) fail(SD_ARGUMENT_ERROR, "bad peer");
    c->pending.push_back({true, buf, nullptr, n, peer});
    if (!c->in_group) {
      local_p2p(c, c->pending, s);
      c->pending.clear();
    }
    return;
  }
  if (!c || !c->comm) fail(SD_STATE_ERROR, "point-to-point send without a communicator");
  nccl_check(nccl().Send(buf, n, ncclFloat32, peer, c->comm, s), "ncclSend");
}
void comm_recv_f32(sd_comm c, float* buf, uint64_t n, int peer, cudaStream_t s) {
  if (c && c->local) {
    if (peer < 0 || peer >= c->nranks || peer == c->rank) fail(SD_ARGUMENT_ERROR, "bad peer");
    c->pending.push_back({false, nullptr, buf, n, peer});
    if (!c->in_group) {
      local_p2p(c, c->pending, s);
      c->pending.clear();
    }
    return;
  }
  if (!c || !c->comm) fail(SD_STATE_ERROR, "point-to-point receive without a communicator");
  nccl_check(nccl().Recv(buf, n, ncclFloat32, peer, c->comm, s), "ncclRecv");
}
void comm_group_begin(sd_comm c) {
  if (c && c->local) c->in_group = true;
  if (c && c->comm) nccl_check(nccl().GroupStart(), "ncclGroupStart");
}
void comm_group_end(sd_comm c, cudaStream_t s) {
  if (c && c->local) {
    c->in_group = false;
    local_p2p(c, c->pending, s);
    c->pending.clear();
  }
  if (c && c->comm) nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

// Waits for the stream; over NCCL it polls ncclCommGetAsyncError meanwhile and
// aborts the communicator on an asynchronous error (a failed or vanished peer)
// or after SD_NCCL_TIMEOUT_S seconds (default 1800) without completion, so a
// dead rank surfaces as SD_NCCL_ERROR on the survivors instead of a hang.
void comm_wait(sd_comm c, cudaStream_t s) {
  if (!c || !c->comm) {
    SD_CUDA(cudaStreamSynchronize(s));
    return;
  }
  static const double timeout = [] {
    const char* e = std::getenv("SD_NCCL_TIMEOUT_S");
    return e ? std::atof(e) : 1800.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) SD_CUDA(e);
    ncclResult_t ae = ncclSuccess;
    if (nccl().CommGetAsyncError) nccl().CommGetAsyncError(c->comm, &ae);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ae != ncclSuccess && ae != ncclInProgress) || (timeout > 0 && el > timeout)) {
      if (nccl().CommAbort) nccl().CommAbort(c->comm);
      c->comm = nullptr;
      c->aborted = true;
      fail(SD_NCCL_ERROR, ae != ncclSuccess && ae != ncclInProgress
                              ? std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ae)
                              : std::string("NCCL collective timed out (SD_NCCL_TIMEOUT_S)"));
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int comm_rank(sd_comm c) { return c ? c->rank : 0; }
int comm_size(sd_comm c) { return c ? c->nranks : 1; }

}  // namespace sd

// --------------------------------------------------------------- operators
struct sd_operator_s {
  uint64_t dim = 0;
  int kind = 0;  // 0 custom, 1 dense, 2 diagonal
  const void* diag = nullptr;  // kind 2: caller-owned device diagonal (this rank's shard)
  int diag_prec = 0;
  sd_apply_fn fn = nullptr;
  void* ctx = nullptr;
  double* a_dev = nullptr;
  void* xfull = nullptr;  // gather scratch (dense)
  size_t xfull_bytes = 0;
  void (*dtor)(void*) = nullptr;  // releases ctx (operators built by the engines)
};

namespace sd {
void operator_set_dtor(sd_operator op, void (*dtor)(void*)) {
  if (op) op->dtor = dtor;
}
}  // namespace sd

namespace sd {

bool operator_needs_full(sd_operator op) { return op->kind == 1; }

// Dense apply needs the gathered x (operators.cpp:35): single rank here, the
// shard IS the full vector; multi-rank gathers through the engine.
void operator_apply(sd_operator op, const void* x, void* y, int prec, cudaStream_t s, uint64_t row_begin,
                    uint64_t row_end, const void* x_full) {
  if (op->kind == 1) {
    dense_apply(op->a_dev, op->dim, x_full ? x_full : x, y, row_begin, row_end, prec, s);
  } else if (op->kind == 2) {
    if (prec != op->diag_prec) fail(SD_LAYOUT_ERROR, "diagonal operator precision mismatch");
    diag_apply(op->diag, x, y, row_end - row_begin, prec, s);
  } else {
    const sd_status st = op->fn(op->ctx, x, y, (sd_stream)s);
    if (st != SD_OK) fail(st, std::string("operator apply failed: ") + sd_last_error());
  }
}

}  // namespace sd

using namespace sd;

extern "C" {

const char* sd_last_error(void) { return g_last_error.c_str(); }
uint64_t sd_launch_count(void) { return g_launches.load(); }
int sd_abi_version(void) { return 1; }

uint64_t sd_keyed_counter(uint64_t seed, uint64_t counter) { return keyed_counter_k(mix64(seed), counter); }
double sd_rademacher(uint64_t seed, uint64_t i) { return (sd_keyed_counter(seed, i) & 1ull) ? 1.0 : -1.0; }
uint64_t sd_uniform_index(uint64_t seed, uint64_t i, uint64_t n) { return sd_keyed_counter(seed, i) % n; }

sd_status sd_split_evenly(uint64_t dim, uint64_t n, uint64_t* begins, uint64_t* ends, uint64_t* count) {
  return guard([&] {
    if (dim == 0 || n == 0) fail(SD_LAYOUT_ERROR, "split_evenly needs dim > 0 and n > 0");
    const uint64_t w = std::min(dim, n), q = dim / w, rem = dim % w;
    uint64_t at = 0;
    for (uint64_t i = 0; i < w; ++i) {
      begins[i] = at;
      at += q + (i < rem ? 1 : 0);
      ends[i] = at;
    }
    *count = w;
    validate(dim, w, begins, ends);
  });
}

// One-forward-one-backward pipeline schedule of `stage` among `n_stages` for
// `n_micro` micro-batches: (kind, micro-batch) pairs, kinds SD_PIPE_*. Warm-up
// forwards (n_stages - stage - 1 of them), then alternating F/B with the
// boundary exchanges grouped as {send F, recv B} and {send B, recv F} so that
// neighbouring stages post matching groups, then the cool-down backwards.
// Micro-batches finish in order, so a stage holds at most n_stages - stage of
// them (its activation sets). ops == NULL: only *count is returned.
sd_status sd_pipeline_schedule(int n_stages, int stage, int n_micro, int* ops, uint64_t cap, uint64_t* count) {
  return guard([&] {
    if (n_stages < 1 || stage < 0 || stage >= n_stages || n_micro < 1)
      fail(SD_ARGUMENT_ERROR, "pipeline schedule: need 0 <= stage < n_stages and n_micro >= 1");
    std::vector<int> v;
    auto op = [&](int k, int m) { v.push_back(k), v.push_back(m); };
    const bool has_prev = stage > 0, has_next = stage < n_stages - 1;
    const int warm = std::min(n_stages - stage - 1, n_micro), rest = n_micro - warm;
    for (int i = 0; i < warm; ++i) {
      if (has_prev) op(SD_PIPE_RECV_F, i);
      op(SD_PIPE_F, i);
      if (has_next) op(SD_PIPE_SEND_F, i);
    }
    if (rest > 0 && has_prev) op(SD_PIPE_RECV_F, warm);
    for (int i = 0; i < rest; ++i) {
      op(SD_PIPE_F, warm + i);
      if (has_next) {
        op(SD_PIPE_GROUP_BEGIN, -1), op(SD_PIPE_SEND_F, warm + i), op(SD_PIPE_RECV_B, i), op(SD_PIPE_GROUP_END, -1);
      }
      op(SD_PIPE_B, i);
      if (has_prev) {
        if (i == rest - 1) {
          op(SD_PIPE_SEND_B, i);
        } else {
          op(SD_PIPE_GROUP_BEGIN, -1), op(SD_PIPE_SEND_B, i), op(SD_PIPE_RECV_F, warm + i + 1);
          op(SD_PIPE_GROUP_END, -1);
        }
      }
    }
    for (int i = rest; i < n_micro; ++i) {
      if (has_next) op(SD_PIPE_RECV_B, i);
      op(SD_PIPE_B, i);
      if (has_prev) op(SD_PIPE_SEND_B, i);
    }
    *count = v.size() / 2;
    if (ops) {
      if (cap < v.size() / 2) fail(SD_ARGUMENT_ERROR, "pipeline schedule: output too small");
      std::copy(v.begin(), v.end(), ops);
    }
  });
}

sd_status sd_validate_layout(uint64_t total, uint64_t n, const uint64_t* begins, const uint64_t* ends) {
  return guard([&] { validate(total, n, begins, ends); });
}

sd_status sd_layout_owner(uint64_t n, const uint64_t* ends, uint64_t i, uint64_t* owner) {
  return guard([&] {
    for (uint64_t w = 0; w < n; ++w)
      if (ends[w] > i) {
        *owner = w;
        return;
      }
    fail(SD_ARGUMENT_ERROR, "index out of range in ShardLayout::owner");
  });
}

sd_status sd_partial_shape(uint64_t begin, uint64_t end, uint64_t total, uint64_t* h, uint64_t* s, uint64_t* t) {
  return guard([&] {
    if (!(end > begin) || end > total) fail(SD_LAYOUT_ERROR, "bad shard range");
    const PartialShape p = partial_shape(begin, end, total);
    *h = p.n_head;
    *s = p.n_sums;
    *t = p.n_tail;
  });
}

uint64_t sd_partial_len(uint64_t begin, uint64_t end, uint64_t total) {
  return partial_shape(begin, end, total).len();
}

sd_status sd_combine_partials_host(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                                   const double* const* parts, double* out) {
  return guard([&] {
    double closed = 0.0, open = 0.0;
    uint64_t at = 0;
    auto grid_end = [&](uint64_t i) { return std::min(total, (i / kBlock + 1) * kBlock); };
    auto feed = [&](double t) {
      open += t;
      ++at;
      if (at == grid_end(at - 1)) {
        closed += open;
        open = 0.0;
      }
    };
    for (uint64_t r = 0; r < nranks; ++r) {
      if (begins[r] != at) fail(SD_PROTOCOL_ERROR, "blocked partials are not contiguous in worker order");
      const PartialShape p = partial_shape(begins[r], ends[r], total);
      const double* x = parts[r];
      for (uint64_t i = 0; i < p.n_head; ++i) feed(x[i]);
      for (uint64_t i = 0; i < p.n_sums; ++i) {
        if (at % kBlock != 0) fail(SD_PROTOCOL_ERROR, "blocked partial misaligned with the reduction grid");
        closed += x[p.n_head + i];
        at = grid_end(at);
      }
      for (uint64_t i = 0; i < p.n_tail; ++i) feed(x[p.n_head + p.n_sums + i]);
      if (at != ends[r]) fail(SD_PROTOCOL_ERROR, "blocked partial does not cover its range");
    }
    if (at != total) fail(SD_PROTOCOL_ERROR, "blocked partials do not cover the vector");
    *out = closed;
  });
}

sd_status sd_ritz_decompose(uint64_t k, const double* alphas, const double* betas, double* values, double* weights,
                            double* resid) {
  return guard([&] { ritz(k, alphas, betas, values, weights, resid); });
}

sd_status sd_smooth_density(uint64_t k, const double* values, const double* weights, double sigma, uint64_t npts,
                            double* grid, double* dens, double* sigma_used) {
  return guard([&] { density(k, values, weights, sigma, npts, grid, dens, sigma_used); });
}

// wigner_dense / spiked_dense (operators.cpp:50-102): host construction of the
// dense test operators (setup, not the hot path), keyed counter Gaussians.
static double host_gaussian(uint64_t seed, uint64_t i) {
  const uint64_t key = mix64(seed);
  const double a = double(keyed_counter_k(key, 2 * i) >> 11) * 0x1p-53 + 0x1p-54;
  const double b = double(keyed_counter_k(key, 2 * i + 1) >> 11) * 0x1p-53 + 0x1p-54;
  return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
}

sd_status sd_wigner_dense(uint64_t n, double sigma, uint64_t seed, double* out) {
  return guard([&] {
    if (n < 2) fail(SD_ARGUMENT_ERROR, "dense operators need n >= 2");
    if (n > 2048) fail(SD_ARGUMENT_ERROR, "dense operator size exceeds the desk-scale cap (2048)");
    if (!(sigma > 0.0)) fail(SD_ARGUMENT_ERROR, "wigner sigma must be positive");
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t j = i; j < n; ++j) out[i * n + j] = out[j * n + i] = sigma * host_gaussian(seed, i * n + j);
  });
}

sd_status sd_spiked_dense(uint64_t n, double sigma, const double* spikes, uint64_t ns, uint64_t seed, double* out) {
  return guard([&] {
    if (!(n > ns)) fail(SD_ARGUMENT_ERROR, "spiked operator needs n > number of spikes");
    const sd_status st = sd_wigner_dense(n, sigma, seed, out);
    if (st != SD_OK) fail(st, g_last_error);
    const uint64_t dseed = mix64(seed ^ 0x5eedd1ce5ull);
    std::vector<std::vector<double>> dirs;
    for (uint64_t sp = 0; sp < ns; ++sp) {
      std::vector<double> u(n);
      for (uint64_t i = 0; i < n; ++i) u[i] = host_gaussian(dseed, sp * n + i);
      for (const auto& w : dirs) {
        double c = 0.0;
        for (uint64_t i = 0; i < n; ++i) c += w[i] * u[i];
        for (uint64_t i = 0; i < n; ++i) u[i] -= c * w[i];
      }
      double nn = 0.0;
      for (uint64_t i = 0; i < n; ++i) nn += u[i] * u[i];
      nn = std::sqrt(nn);
      if (!(nn > 0.0)) fail(SD_NUMERICAL_ERROR, "degenerate spike direction");
      for (uint64_t i = 0; i < n; ++i) u[i] /= nn;
      for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j) out[i * n + j] += spikes[sp] * (u[i] * u[j]);
      dirs.push_back(std::move(u));
    }
  });
}

sd_status sd_nccl_unique_id(unsigned char out_id[128]) {
  return guard([&] {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out_id, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  });
}

sd_status sd_comm_nccl_create(const unsigned char id[128], int nranks, int rank, sd_comm* out) {
  return guard([&] {
    auto c = std::make_unique<sd_comm_s>();
    c->nranks = nranks;
    c->rank = rank;
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SD_ARGUMENT_ERROR, "bad rank/size");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().CommInitRank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

sd_status sd_comm_destroy(sd_comm c) {
  return guard([&] {
    if (c && c->comm) nccl_check(nccl().CommDestroy(c->comm), "ncclCommDestroy");
    if (c && c->d_ptrs) cudaFree(c->d_ptrs);
    if (c && c->ord_buf) cudaFree(c->ord_buf);
    if (c && c->ord_tmp) cudaFree(c->ord_tmp);
    delete c;
  });
}

// a failing worker / rank releases the others: in-process groups leave their
// barriers with SD_PROTOCOL_ERROR; an NCCL communicator is aborted
// (ncclCommAbort), which makes the peers' pending collectives fail
sd_status sd_comm_abort(sd_comm c) {
  return guard([&] {
    if (c && c->local) c->local->abort();
    if (c && c->comm) {
      if (nccl().CommAbort) nccl().CommAbort(c->comm);
      c->comm = nullptr;
      c->aborted = true;
    }
  });
}

sd_status sd_comm_wait(sd_comm c, sd_stream s) {
  return guard([&] { comm_wait(c, (cudaStream_t)s); });
}

// n in-process workers sharing one device (the reference's WorkerPool,
// pool.hpp:47-94): out[r] is worker r's communicator, to be driven by its own
// host thread with its own stream.
sd_status sd_comm_local_create(int nranks, sd_comm* out) {
  return guard([&] {
    if (nranks < 1 || !out) fail(SD_ARGUMENT_ERROR, "bad worker count");
    auto g = std::make_shared<LocalGroup>();
    g->n = nranks;
    g->slot.assign(nranks, nullptr);
    g->q.assign(nranks, std::vector<std::deque<LocalMsg*>>(nranks));
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<sd_comm_s>();
      c->nranks = nranks, c->rank = r, c->local = g;
      out[r] = c.release();
    }
  });
}

sd_status sd_comm_allreduce_f32(sd_comm c, float* buf, uint64_t n, sd_stream s) {
  return guard([&] { comm_allreduce_f32(c, buf, n, (cudaStream_t)s); });
}

sd_status sd_comm_allgather(sd_comm c, const void* send, void* recv, uint64_t bytes, sd_stream s) {
  return guard([&] { comm_allgather(c, send, recv, bytes, (cudaStream_t)s); });
}

sd_status sd_operator_custom(uint64_t dim, sd_apply_fn fn, void* ctx, sd_operator* out) {
  return guard([&] {
    if (!fn) fail(SD_ARGUMENT_ERROR, "operator apply function is null");
    auto op = std::make_unique<sd_operator_s>();
    op->dim = dim;
    op->fn = fn;
    op->ctx = ctx;
    *out = op.release();
  });
}

sd_status sd_operator_dense(uint64_t n, const double* a_host, sd_operator* out) {
  return guard([&] {
    if (n < 2) fail(SD_ARGUMENT_ERROR, "dense operators need n >= 2");
    if (n > 2048) fail(SD_ARGUMENT_ERROR, "dense operator size exceeds the desk-scale cap (2048)");
    auto op = std::make_unique<sd_operator_s>();
    op->dim = n;
    op->kind = 1;
    SD_CUDA(cudaMalloc(&op->a_dev, n * n * sizeof(double)));
    SD_CUDA(cudaMemcpy(op->a_dev, a_host, n * n * sizeof(double), cudaMemcpyHostToDevice));
    *out = op.release();
  });
}

sd_status sd_operator_diag(uint64_t dim, const void* d_dev, int prec, sd_operator* out) {
  return guard([&] {
    auto op = std::make_unique<sd_operator_s>();
    op->dim = dim;
    op->kind = 2;
    op->diag = d_dev;
    op->diag_prec = prec;
    *out = op.release();
  });
}

sd_status sd_operator_apply(sd_operator op, const void* x, void* y, int prec, sd_stream s) {
  return guard([&] { operator_apply(op, x, y, prec, (cudaStream_t)s, 0, op->dim, nullptr); });
}

uint64_t sd_operator_dim(sd_operator op) { return op ? op->dim : 0; }

sd_status sd_operator_destroy(sd_operator op) {
  return guard([&] {
    if (!op) return;
    if (op->a_dev) cudaFree(op->a_dev);
    if (op->dtor) op->dtor(op->ctx);
    delete op;
  });
}

}  // extern "C"
