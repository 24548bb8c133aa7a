// Multi-GPU BFM solver with a C++ host: one process per GPU,
// axis-0 slab decomposition, exchanges as NCCL grouped send/recv issued from
// the library on the solver's own stream (pack/unpack by this file's kernels),
// rank-ordered double-double scalar merges. The reference has no distributed
// mode; every rank runs the loop of bfm::Solver (solver.hpp:146-368) on its
// rows, and the results equal the single-GPU solver bit for bit:
//  * c-transform: phi rows -> columns (one all-to-all), pass 0 on the column
//    slab (bfm_slab_ct_cols), (q, chain) columns -> rows as ONE packed
//    all-to-all, passes 1..d-1 on the rows (bfm_slab_ct_rows);
//  * Neumann solve: DCT-II along axes d-1..1 on rows, rows -> columns, the
//    fused axis-0 [DCT-II, divide, DCT-III], columns -> rows, DCT-III;
//  * pushforward: halo rows from the neighbours, deposit records routed to
//    the owners of their target rows (counts exchange + all-to-all-v); the
//    concatenation in sender order is the global source order, so every
//    target folds in the reference's sequential order;
//  * scalars: per-rank double-double partials, all-gathered and merged in
//    rank order (deterministic on every rank).
// Communicators: NCCL (libnccl.so.2 loaded at first use), or an in-process
// group of ranks as threads on one device whose exchanges go through host
// synchronisation (no kernel waits on another rank) — how the single-GPU test
// box checks P > 1.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bfm_b200.h"
#include "common.cuh"

namespace bfmgpu {
namespace {

// ---- NCCL, resolved at run time ------------------------------------------------
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool done = false;
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  if (done) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw std::runtime_error("NCCL (libnccl.so.2) is not available");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
  api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
  api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
  api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
  api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
  api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
  api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
  done = true;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string("NCCL error in ") + what + ": " + nccl().errorString(r));
}

// ---- communicators -------------------------------------------------------------
class Comm {
 public:
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // byte all-to-all-v between device buffers, ordered on stream s
  virtual void alltoallv(const void* send, const std::vector<size_t>& scnt, const std::vector<size_t>& soff,
                         void* recv, const std::vector<size_t>& rcnt, const std::vector<size_t>& roff,
                         cudaStream_t s) = 0;
  // every rank's n host doubles -> all[size * n] (synchronous)
  virtual void allgather(const double* mine, int n, double* all, cudaStream_t s) = 0;
  // send[q] host longs for rank q -> recv[q] what rank q sent here (synchronous)
  virtual void alltoall_counts(const long* send, long* recv, cudaStream_t s) = 0;
};

class NcclComm : public Comm {
 public:
  NcclComm(const unsigned char* id, int r, int n) {
    rank = r;
    size = n;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().commInitRank(&comm_, n, uid, r), "ncclCommInitRank");
    BFM_CUDA(dmalloc(&scratch_, sizeof(double) * 64 * static_cast<size_t>(n + 1)));
    BFM_CUDA(cudaMallocHost(&host_, sizeof(double) * 64 * static_cast<size_t>(n + 1)));
  }
  ~NcclComm() override {
    if (comm_) nccl().commDestroy(comm_);
    if (scratch_) dfree(scratch_);
    if (host_) cudaFreeHost(host_);
  }
  void alltoallv(const void* send, const std::vector<size_t>& scnt, const std::vector<size_t>& soff, void* recv,
                 const std::vector<size_t>& rcnt, const std::vector<size_t>& roff, cudaStream_t s) override {
    const NcclApi& A = nccl();
    nccl_check(A.groupStart(), "ncclGroupStart");
    for (int q = 0; q < size; ++q) {
      if (scnt[q])
        nccl_check(A.send(static_cast<const char*>(send) + soff[q], scnt[q], ncclUint8, q, comm_, s), "ncclSend");
      if (rcnt[q])
        nccl_check(A.recv(static_cast<char*>(recv) + roff[q], rcnt[q], ncclUint8, q, comm_, s), "ncclRecv");
    }
    nccl_check(A.groupEnd(), "ncclGroupEnd");
  }
  void allgather(const double* mine, int n, double* all, cudaStream_t s) override {
    if (n > 64) throw std::invalid_argument("allgather: at most 64 values");
    std::memcpy(host_, mine, sizeof(double) * n);
    BFM_CUDA(cudaMemcpyAsync(scratch_, host_, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    nccl_check(nccl().allGather(scratch_, scratch_ + 64, n, ncclDouble, comm_, s), "ncclAllGather");
    BFM_CUDA(cudaMemcpyAsync(host_ + 64, scratch_ + 64, sizeof(double) * n * size, cudaMemcpyDeviceToHost, s));
    BFM_CUDA(cudaStreamSynchronize(s));
    std::memcpy(all, host_ + 64, sizeof(double) * n * size);
  }
  void alltoall_counts(const long* send, long* recv, cudaStream_t s) override {
    static_assert(sizeof(long) == sizeof(double), "long is 8 bytes");
    std::vector<size_t> c(size, sizeof(long)), off(size);
    for (int q = 0; q < size; ++q) off[q] = q * sizeof(long);
    std::memcpy(host_, send, sizeof(long) * size);
    BFM_CUDA(cudaMemcpyAsync(scratch_, host_, sizeof(long) * size, cudaMemcpyHostToDevice, s));
    alltoallv(scratch_, c, off, scratch_ + 64, c, off, s);
    BFM_CUDA(cudaMemcpyAsync(host_ + 64, scratch_ + 64, sizeof(long) * size, cudaMemcpyDeviceToHost, s));
    BFM_CUDA(cudaStreamSynchronize(s));
    std::memcpy(recv, host_ + 64, sizeof(long) * size);
  }

 private:
  ncclComm_t comm_ = nullptr;
  double* scratch_ = nullptr;
  double* host_ = nullptr;
};

// Ranks as threads of one process on one device. Every exchange is host
// synchronised: post, barrier, copy from the peers' buffers, barrier.
struct LocalGroup {
  explicit LocalGroup(int n) : size(n), posts(n) {}
  struct Post {
    const void* send = nullptr;
    const size_t* scnt = nullptr;
    const size_t* soff = nullptr;
    const double* vals = nullptr;
    const long* counts = nullptr;
  };
  int size;
  std::vector<Post> posts;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == size) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int r) : g_(std::move(g)) {
    rank = r;
    size = g_->size;
  }
  void alltoallv(const void* send, const std::vector<size_t>& scnt, const std::vector<size_t>& soff, void* recv,
                 const std::vector<size_t>& rcnt, const std::vector<size_t>& roff, cudaStream_t s) override {
    BFM_CUDA(cudaStreamSynchronize(s));
    g_->posts[rank].send = send;
    g_->posts[rank].scnt = scnt.data();
    g_->posts[rank].soff = soff.data();
    g_->barrier();
    for (int q = 0; q < size; ++q) {
      const LocalGroup::Post& p = g_->posts[q];
      if (p.scnt[rank] != rcnt[q]) throw std::runtime_error("local all-to-all: count mismatch");
      if (rcnt[q])
        BFM_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + roff[q], static_cast<const char*>(p.send) + p.soff[rank],
                                 rcnt[q], cudaMemcpyDeviceToDevice, s));
    }
    BFM_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
  }
  void allgather(const double* mine, int n, double* all, cudaStream_t) override {
    g_->posts[rank].vals = mine;
    g_->barrier();
    for (int q = 0; q < size; ++q) std::memcpy(all + q * n, g_->posts[q].vals, sizeof(double) * n);
    g_->barrier();
  }
  void alltoall_counts(const long* send, long* recv, cudaStream_t) override {
    g_->posts[rank].counts = send;
    g_->barrier();
    for (int q = 0; q < size; ++q) recv[q] = g_->posts[q].counts[rank];
    g_->barrier();
  }

 private:
  std::shared_ptr<LocalGroup> g_;
};

// ---- layout ----------------------------------------------------------------------
void split(long n, int parts, std::vector<long>& start, std::vector<long>& size) {
  start.assign(parts, 0);
  size.assign(parts, 0);
  const long base = n / parts, rem = n % parts;
  long s = 0;
  for (int r = 0; r < parts; ++r) {
    size[r] = base + (r < rem ? 1 : 0);
    start[r] = s;
    s += size[r];
  }
}

struct Layout {
  int d = 2;
  int ext[3] = {1, 1, 1};
  int P = 1;
  long n0 = 0, M = 0, N = 0;
  double vol = 1.0;
  std::vector<long> row0, nrows, col0, ncols;
  Layout(int dim, const int* e, int parts) : d(dim), P(parts) {
    if (dim < 2) throw std::invalid_argument("slab decomposition needs d >= 2");
    for (int a = 0; a < dim; ++a) ext[a] = e[a];
    n0 = e[0];
    M = 1;
    for (int a = 1; a < dim; ++a) M *= e[a];
    N = n0 * M;
    if (n0 < P || M < P) throw std::invalid_argument("grid too small for the number of ranks");
    for (int a = 0; a < dim; ++a) vol *= 1.0 / e[a];  // grid.hpp:71
    split(n0, P, row0, nrows);
    split(M, P, col0, ncols);
  }
};

// ---- pack / unpack kernels -------------------------------------------------------
// rows -> columns: element (i, c) of the row slab (nr x M) goes to the rank q
// owning column c, at q's block offset + i * nc_q + (c - col0_q)
__global__ void pack_rows_to_cols(const double* x, long nr, long M, int P, const long* col0,
                                  const long* ncols, const long* boff, double* out) {
  const long total = nr * M;
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const long i = e / M, c = e - i * M;
    int q = 0;
    while (q + 1 < P && col0[q + 1] <= c) ++q;
    out[boff[q] + i * ncols[q] + (c - col0[q])] = x[e];
  }
}

// columns -> rows (doubles): block from rank q (nr x nc_q) lands in columns
// [col0_q, col0_q + nc_q) of the row slab
__global__ void unpack_cols_to_rows(const double* in, long nr, long M, int P, const long* col0,
                                    const long* ncols, const long* boff, double* out) {
  const long total = nr * M;
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const long i = e / M, c = e - i * M;
    int q = 0;
    while (q + 1 < P && col0[q + 1] <= c) ++q;
    out[e] = in[boff[q] + i * ncols[q] + (c - col0[q])];
  }
}

// column slab (n0 x nc) -> per destination rank q one block [q values
// (8 * cnt_q) | chain values (4 * cnt_q), padded to 8 bytes], rows of q in
// order: ONE message carries both outputs of pass 0
__global__ void pack_qchain(const double* qv, const uint32_t* ch, long n0, long nc, int P, const long* row0,
                            const long* nrows, const long* boff_bytes, unsigned char* out) {
  const long total = n0 * nc;
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const long i = e / nc;
    int q = 0;
    while (q + 1 < P && row0[q + 1] <= i) ++q;
    const long local = e - row0[q] * nc;
    const long cnt = nrows[q] * nc;
    unsigned char* b = out + boff_bytes[q];
    reinterpret_cast<double*>(b)[local] = qv[e];
    reinterpret_cast<uint32_t*>(b + 8 * cnt)[local] = ch[e];
  }
}

__global__ void unpack_qchain(const unsigned char* in, long nr, long M, int P, const long* col0,
                              const long* ncols, const long* boff_bytes, double* qv, uint32_t* ch) {
  const long total = nr * M;
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const long i = e / M, c = e - i * M;
    int q = 0;
    while (q + 1 < P && col0[q + 1] <= c) ++q;
    const long cnt = nr * ncols[q];
    const long local = i * ncols[q] + (c - col0[q]);
    const unsigned char* b = in + boff_bytes[q];
    qv[e] = reinterpret_cast<const double*>(b)[local];
    ch[e] = reinterpret_cast<const uint32_t*>(b + 8 * cnt)[local];
  }
}

unsigned ew_blocks(long n) {
  long b = (n + 255) / 256;
  return static_cast<unsigned>(std::max<long>(1, std::min<long>(b, 148L * 16)));
}

void ck(int rc) {
  if (rc != BFM_OK) throw std::runtime_error(bfm_last_error());
}

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  ~DArr() {
    if (p) dfree(p);
  }
  T* get(size_t count) {
    if (count > n) {
      if (p) dfree(p);
      p = nullptr;
      BFM_CUDA(dmalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
      n = count;
    }
    return p;
  }
};

void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

}  // namespace
}  // namespace bfmgpu

using namespace bfmgpu;

struct bfm_comm {
  std::unique_ptr<Comm> c;
};

struct bfm_dist_solver {
  Layout L;
  Comm* comm;
  int rank;
  long nr = 0, nc = 0, nloc = 0;
  bfm_config cfg;
  cudaStream_t stream = nullptr;
  bfm_slab* slab = nullptr;
  DArr<double> mu, nu, phi, psi, dir, dir2, r, t1, t2, cols_a, cols_b, halo, wbuf, wmap, packed, rpacked, rmass, rw;
  DArr<uint32_t> chain_c, chain_r, key, rkeys;
  DArr<uint8_t> cmask, rcmask;
  DArr<unsigned char> qsend, qrecv;
  DArr<long> meta;  // col0, ncols, boff(r2c), boff(c2r), row0, nrows, boff qchain send, recv
  std::vector<long> boff_r2c, boff_c2r, qboff_send, qboff_recv;
  double sigma = 0.0, last_pair = 0.0, prev_dual = std::numeric_limits<double>::quiet_NaN();
  double probe_dual = 0.0, probe_gn = 0.0;
  bool fresh = false;
  int iteration = 0, stall = 0;
  std::vector<bfm_iteration_stats> trace;
  std::chrono::steady_clock::time_point start;
  // report (host, full grid, every rank)
  std::vector<double> rep_phi, rep_psi, rep_map;
  bool has_report = false;

  bfm_dist_solver(Comm* c, int dim, const int* ext) : L(dim, ext, c->size), comm(c), rank(c->rank) {}
  ~bfm_dist_solver() {
    if (slab) bfm_slab_destroy(slab);
    if (stream) cudaStreamDestroy(stream);
  }
  void* st() const { return stream; }

  // ---- exchanges -------------------------------------------------------------------
  const long* dmeta(int which) const { return meta.p + which * (L.P + 1); }

  void rows_to_cols(const double* rows, double* cols) {
    pack_rows_to_cols<<<ew_blocks(nloc), 256, 0, stream>>>(rows, nr, L.M, L.P, dmeta(0), dmeta(1), dmeta(2),
                                                          wbuf.p);
    BFM_LAUNCH_CHECK("pack_rows_to_cols");
    std::vector<size_t> sc(L.P), so(L.P), rc(L.P), ro(L.P);
    for (int q = 0; q < L.P; ++q) {
      sc[q] = 8 * nr * L.ncols[q];
      so[q] = 8 * boff_r2c[q];
      rc[q] = 8 * L.nrows[q] * nc;
      ro[q] = 8 * L.row0[q] * nc;
    }
    comm->alltoallv(wbuf.p, sc, so, cols, rc, ro, stream);
  }
  void cols_to_rows(const double* cols, double* rows) {
    std::vector<size_t> sc(L.P), so(L.P), rc(L.P), ro(L.P);
    for (int q = 0; q < L.P; ++q) {
      sc[q] = 8 * L.nrows[q] * nc;
      so[q] = 8 * L.row0[q] * nc;
      rc[q] = 8 * nr * L.ncols[q];
      ro[q] = 8 * boff_c2r[q];
    }
    comm->alltoallv(cols, sc, so, wbuf.p, rc, ro, stream);
    unpack_cols_to_rows<<<ew_blocks(nloc), 256, 0, stream>>>(wbuf.p, nr, L.M, L.P, dmeta(0), dmeta(1), dmeta(3),
                                                            rows);
    BFM_LAUNCH_CHECK("unpack_cols_to_rows");
  }

  // ---- operators -------------------------------------------------------------------
  void ctransform(const double* u, double* out) {  // transforms.hpp:396-432
    rows_to_cols(u, cols_a.p);
    ck(bfm_slab_ct_cols(slab, cols_a.p, chain_c.p, cols_b.p, st()));
    pack_qchain<<<ew_blocks(L.n0 * nc), 256, 0, stream>>>(cols_b.p, chain_c.p, L.n0, nc, L.P, dmeta(4), dmeta(5),
                                                          dmeta(6), qsend.p);
    BFM_LAUNCH_CHECK("pack_qchain");
    std::vector<size_t> sc(L.P), so(L.P), rc(L.P), ro(L.P);
    for (int q = 0; q < L.P; ++q) {
      sc[q] = static_cast<size_t>(qboff_send[q + 1] - qboff_send[q]);
      so[q] = static_cast<size_t>(qboff_send[q]);
      rc[q] = static_cast<size_t>(qboff_recv[q + 1] - qboff_recv[q]);
      ro[q] = static_cast<size_t>(qboff_recv[q]);
    }
    comm->alltoallv(qsend.p, sc, so, qrecv.p, rc, ro, stream);
    unpack_qchain<<<ew_blocks(nloc), 256, 0, stream>>>(qrecv.p, nr, L.M, L.P, dmeta(0), dmeta(1), dmeta(7), t1.p,
                                                      chain_r.p);
    BFM_LAUNCH_CHECK("unpack_qchain");
    ck(bfm_slab_ct_rows(slab, chain_r.p, t1.p, out, st()));
  }
  void solve_neumann(const double* rhs, double* out) {  // poisson.hpp:87-106
    ck(bfm_slab_poisson_rows_forward(slab, rhs, t2.p, st()));
    rows_to_cols(t2.p, cols_a.p);
    ck(bfm_slab_poisson_cols(slab, cols_a.p, cols_b.p, st()));
    cols_to_rows(cols_b.p, out);
    ck(bfm_slab_poisson_rows_inverse(slab, out, st()));
  }
  void make_halo(const double* u) {  // rows r0-1 .. r0+nr of u (zeros outside the grid)
    double* h = halo.p;
    BFM_CUDA(cudaMemcpyAsync(h + L.M, u, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, stream));
    std::vector<size_t> sc(L.P, 0), so(L.P, 0), rc(L.P, 0), ro(L.P, 0);
    if (rank > 0) {
      sc[rank - 1] = 8 * L.M;
      so[rank - 1] = 8 * L.M;  // first own row
      rc[rank - 1] = 8 * L.M;
      ro[rank - 1] = 0;
    } else {
      BFM_CUDA(cudaMemsetAsync(h, 0, sizeof(double) * L.M, stream));
    }
    if (rank < L.P - 1) {
      sc[rank + 1] = 8 * L.M;
      so[rank + 1] = 8 * nr * L.M;  // last own row
      rc[rank + 1] = 8 * L.M;
      ro[rank + 1] = 8 * (nr + 1) * L.M;
    } else {
      BFM_CUDA(cudaMemsetAsync(h + (nr + 1) * L.M, 0, sizeof(double) * L.M, stream));
    }
    comm->alltoallv(h, sc, so, h, rc, ro, stream);
  }
  // solver.hpp:251-253: r = target - pushforward(map(u), source)
  void pushforward_residual(const double* u, const double* source, const double* target, double* out,
                            double* disp = nullptr) {
    make_halo(u);
    ck(bfm_slab_pf_map(slab, halo.p, source, key.p, wmap.p, cmask.p, disp, st()));
    if (!out) return;
    const int rec = 3 + L.d;
    std::vector<long> counts(L.P), rcounts(L.P);
    ck(bfm_slab_pf_route(slab, key.p, wmap.p, cmask.p, source, packed.p, counts.data(), st()));
    comm->alltoall_counts(counts.data(), rcounts.data(), stream);
    std::vector<size_t> sc(L.P), so(L.P), rc(L.P), ro(L.P);
    size_t s0 = 0, r0 = 0;
    for (int q = 0; q < L.P; ++q) {
      sc[q] = 8 * rec * counts[q];
      so[q] = s0;
      s0 += sc[q];
      rc[q] = 8 * rec * rcounts[q];
      ro[q] = r0;
      r0 += rc[q];
    }
    const long nrec = static_cast<long>(r0 / (8 * rec));
    double* rp = rpacked.get(static_cast<size_t>(nrec) * rec);
    comm->alltoallv(packed.p, sc, so, rp, rc, ro, stream);
    uint32_t* k = rkeys.get(nrec);
    double* m = rmass.get(nrec);
    double* w = rw.get(static_cast<size_t>(L.d) * nrec);
    uint8_t* cm = rcmask.get(nrec);
    ck(bfm_slab_pf_unpack(slab, nrec, rp, k, m, w, cm, st()));
    ck(bfm_slab_pf_gather(slab, nrec, k, m, w, cm, target, out, st()));
  }
  double dot(const double* a1, const double* b1, const double* a2, const double* b2) {
    double mine[4];
    ck(bfm_slab_dot(slab, a1, b1, a2, b2, mine, st()));
    std::vector<double> all(4 * L.P);
    comm->allgather(mine, 4, all.data(), stream);
    double s1 = 0, c1 = 0, s2 = 0, c2 = 0;  // rank-ordered merge (reduce.cu dd_merge)
    for (int q = 0; q < L.P; ++q) {
      double s, e;
      two_sum(s1, all[4 * q], s, e);
      s1 = s;
      c1 = (c1 + all[4 * q + 1]) + e;
      two_sum(s2, all[4 * q + 2], s, e);
      s2 = s;
      c2 = (c2 + all[4 * q + 3]) + e;
    }
    double v = (s1 + c1) * L.vol;
    if (a2) v = v + (s2 + c2) * L.vol;
    return v;
  }
  double pair_value() { return dot(phi.p, nu.p, psi.p, mu.p); }  // solver.hpp:240
  double ascent(const double* u, const double* source, const double* target, double* d) {
    pushforward_residual(u, source, target, r.p);
    solve_neumann(r.p, d);
    return dot(r.p, d, nullptr, nullptr);
  }
  double update_sigma(double s, double inc, double gn) const {  // solver.hpp:68-76
    const double pred = s * gn;
    if (inc < cfg.beta_1 * pred) s *= cfg.alpha_2;
    else if (inc > cfg.beta_2 * pred) s *= cfg.alpha_1;
    return std::max(s, cfg.sigma_min);
  }
  [[noreturn]] void blowup() { throw BlowupError(); }
  struct BlowupError {};

  void ensure_probe() {  // solver.hpp:264-280
    if (fresh) return;
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      ctransform(phi.p, psi.p);
      const double v = pair_value();
      if (v < last_pair - 1e-10) blowup();
      last_pair = v;
      probe_dual = v;
    } else {
      probe_dual = last_pair;
    }
    probe_gn = ascent(psi.p, mu.p, nu.p, dir.p);
    fresh = true;
  }
  bfm_iteration_stats step() {  // solver.hpp:189-207,286-328
    ensure_probe();
    bfm_iteration_stats s;
    std::memset(&s, 0, sizeof(s));
    s.iteration = iteration + 1;
    s.residual = std::sqrt(std::max(probe_gn, 0.0));
    s.sigma_first = sigma;
    s.grad_norm_sq_first = probe_gn;
    ck(bfm_slab_axpy(slab, phi.p, sigma, dir.p, st()));
    ctransform(phi.p, psi.p);
    const double v2 = probe_dual, v3 = pair_value();
    s.increase_first = v3 - v2;
    sigma = update_sigma(sigma, s.increase_first, probe_gn);
    ctransform(psi.p, phi.p);
    const double v4 = pair_value();
    if (v4 < v3 - 1e-10) blowup();
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      const double gn2 = ascent(phi.p, nu.p, mu.p, dir2.p);
      s.sigma_second = sigma;
      s.grad_norm_sq_second = gn2;
      ck(bfm_slab_axpy(slab, psi.p, sigma, dir2.p, st()));
      ctransform(psi.p, phi.p);
      const double v5 = pair_value();
      s.increase_second = v5 - v4;
      sigma = update_sigma(sigma, s.increase_second, gn2);
      s.dual_value = v5;
    } else {
      s.dual_value = v4;
    }
    last_pair = s.dual_value;
    fresh = false;
    ++iteration;
    if (std::abs(s.dual_value - prev_dual) < 1e-12) ++stall;
    else stall = 0;
    prev_dual = s.dual_value;
    trace.push_back(s);
    return s;
  }
  // every rank's rows of a device field -> the full field on every host
  void gather_full(const double* rows, std::vector<double>& full) {
    full.resize(L.N);
    double* all = cols_b.get(static_cast<size_t>(L.N));
    std::vector<size_t> sc(L.P), so(L.P, 0), rc(L.P), ro(L.P);
    for (int q = 0; q < L.P; ++q) {
      sc[q] = 8 * nloc;
      rc[q] = 8 * L.nrows[q] * L.M;
      ro[q] = 8 * L.row0[q] * L.M;
    }
    comm->alltoallv(rows, sc, so, all, rc, ro, stream);
    BFM_CUDA(cudaMemcpyAsync(full.data(), all, sizeof(double) * L.N, cudaMemcpyDeviceToHost, stream));
    BFM_CUDA(cudaStreamSynchronize(stream));
  }
  void finish(int term, double residual, bfm_report* rep) {  // solver.hpp:330-349
    rep->termination = term;
    rep->iterations = iteration;
    rep->dual_value = probe_dual;
    rep->residual = residual;
    gather_full(phi.p, rep_phi);
    gather_full(psi.p, rep_psi);
    double s = 0.0, c = 0.0;  // grid.hpp:124-133,179-183: the reference's sequential Kahan
    for (double v : rep_phi) {
      const double y = v - c;
      const double t = s + y;
      c = (t - s) - y;
      s = t;
    }
    const double shift = s * L.vol;
    for (double& v : rep_phi) v = v - shift;
    for (double& v : rep_psi) v = v + shift;
    BFM_CUDA(cudaMemcpyAsync(t1.p, rep_psi.data() + L.row0[rank] * L.M, sizeof(double) * nloc,
                             cudaMemcpyHostToDevice, stream));
    double* disp = cols_a.get(static_cast<size_t>(L.d) * nloc);
    pushforward_residual(t1.p, mu.p, nullptr, nullptr, disp);
    double mine[2];
    ck(bfm_slab_primal(slab, disp, mu.p, mine, st()));
    std::vector<double> all(2 * L.P);
    comm->allgather(mine, 2, all.data(), stream);
    double ps = 0, pc = 0;
    for (int q = 0; q < L.P; ++q) {
      double a, e;
      two_sum(ps, all[2 * q], a, e);
      ps = a;
      pc = (pc + all[2 * q + 1]) + e;
    }
    rep->primal_cost = (ps + pc) * L.vol;
    rep_map.resize(static_cast<size_t>(L.d) * L.N);
    std::vector<double> comp;
    for (int a = 0; a < L.d; ++a) {
      gather_full(disp + a * nloc, comp);
      std::copy(comp.begin(), comp.end(), rep_map.begin() + static_cast<long>(a) * L.N);
    }
    rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    has_report = true;
  }
  void run(bfm_report* rep) {  // solver.hpp:211-226
    while (true) {
      ensure_probe();
      const double residual = std::sqrt(std::max(probe_gn, 0.0));
      if (cfg.tolerance >= 0.0 && residual <= cfg.tolerance) return finish(BFM_TERM_TOLERANCE_MET, residual, rep);
      if (cfg.has_exact_cost && cfg.exact_tolerance > 0.0 && std::abs(probe_dual - cfg.exact_cost) <= cfg.exact_tolerance)
        return finish(BFM_TERM_COST_TARGET_MET, residual, rep);
      if (iteration >= cfg.max_iterations) return finish(BFM_TERM_MAX_ITERATIONS, residual, rep);
      if (stall >= 10) return finish(BFM_TERM_DUAL_STALLED, residual, rep);
      step();
    }
  }

  void setup(const double* mu_rows, const double* nu_rows, const bfm_config& c) {
    cfg = c;
    start = std::chrono::steady_clock::now();
    nr = L.nrows[rank];
    nc = L.ncols[rank];
    nloc = nr * L.M;
    BFM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    ck(bfm_slab_create(L.d, L.ext, static_cast<int>(L.row0[rank]), static_cast<int>(nr), L.col0[rank],
                       static_cast<int>(nc), &slab));
    std::vector<int> starts(L.P + 1);
    for (int q = 0; q < L.P; ++q) starts[q] = static_cast<int>(L.row0[q]);
    starts[L.P] = static_cast<int>(L.n0);
    ck(bfm_slab_set_partition(slab, L.P, starts.data()));
    for (auto* b : {&mu, &nu, &phi, &psi, &dir, &dir2, &r, &t1, &t2}) b->get(nloc);
    cols_a.get(std::max<long>(L.n0 * nc, L.d * nloc));
    cols_b.get(std::max<long>(L.n0 * nc, L.N));
    wbuf.get(std::max<long>(nloc, L.n0 * nc));
    halo.get((nr + 2) * L.M);
    wmap.get(static_cast<size_t>(L.d) * nloc);
    packed.get(2 * nloc * (3 + L.d));
    chain_c.get(L.n0 * nc);
    chain_r.get(nloc);
    key.get(nloc);
    cmask.get(nloc);
    // block offsets (elements): rows->cols send blocks (nr x nc_q), cols->rows
    // receive blocks (nr x nc_q); (q, chain) byte blocks padded to 8 bytes
    boff_r2c.assign(L.P + 1, 0);
    boff_c2r.assign(L.P + 1, 0);
    qboff_send.assign(L.P + 1, 0);
    qboff_recv.assign(L.P + 1, 0);
    for (int q = 0; q < L.P; ++q) {
      boff_r2c[q + 1] = boff_r2c[q] + nr * L.ncols[q];
      boff_c2r[q + 1] = boff_c2r[q] + nr * L.ncols[q];
      qboff_send[q + 1] = qboff_send[q] + ((12 * L.nrows[q] * nc + 7) & ~7L);
      qboff_recv[q + 1] = qboff_recv[q] + ((12 * nr * L.ncols[q] + 7) & ~7L);
    }
    qsend.get(static_cast<size_t>(qboff_send[L.P]));
    qrecv.get(static_cast<size_t>(qboff_recv[L.P]));
    std::vector<long> m(8 * (L.P + 1), 0);
    for (int q = 0; q < L.P; ++q) {
      m[0 * (L.P + 1) + q] = L.col0[q];
      m[1 * (L.P + 1) + q] = L.ncols[q];
      m[2 * (L.P + 1) + q] = boff_r2c[q];
      m[3 * (L.P + 1) + q] = boff_c2r[q];
      m[4 * (L.P + 1) + q] = L.row0[q];
      m[5 * (L.P + 1) + q] = L.nrows[q];
      m[6 * (L.P + 1) + q] = qboff_send[q];
      m[7 * (L.P + 1) + q] = qboff_recv[q];
    }
    meta.get(m.size());
    BFM_CUDA(cudaMemcpyAsync(meta.p, m.data(), m.size() * sizeof(long), cudaMemcpyHostToDevice, stream));
    BFM_CUDA(cudaMemcpyAsync(mu.p, mu_rows, sizeof(double) * nloc, cudaMemcpyHostToDevice, stream));
    BFM_CUDA(cudaMemcpyAsync(nu.p, nu_rows, sizeof(double) * nloc, cudaMemcpyHostToDevice, stream));
    BFM_CUDA(cudaMemsetAsync(phi.p, 0, sizeof(double) * nloc, stream));
    BFM_CUDA(cudaMemsetAsync(psi.p, 0, sizeof(double) * nloc, stream));
    BFM_CUDA(cudaStreamSynchronize(stream));
    // sigma_0 = 8 / max(sup mu, sup nu) over all ranks (solver.hpp:160-163)
    double sups[2] = {0.0, 0.0};
    for (long i = 0; i < nloc; ++i) {
      sups[0] = std::max(sups[0], mu_rows[i]);
      sups[1] = std::max(sups[1], nu_rows[i]);
    }
    std::vector<double> all(2 * L.P);
    comm->allgather(sups, 2, all.data(), stream);
    const double sup = *std::max_element(all.begin(), all.end());
    sigma = cfg.sigma_init > 0.0 ? cfg.sigma_init : 8.0 / sup;
  }
};

namespace {
thread_local std::string g_dist_err;
template <class F>
int dguard(F&& f) {
  try {
    f();
    return BFM_OK;
  } catch (const bfm_dist_solver::BlowupError&) {
    g_dist_err = "solve: conjugation decreased the dual pair value";
    return BFM_ERR_NUMERICAL_BLOWUP;
  } catch (const CudaError& e) {
    g_dist_err = e.what();
    return BFM_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_dist_err = e.what();
    return BFM_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_dist_err = e.what();
    return BFM_ERR_ERROR;
  }
}
}  // namespace

extern "C" {

const char* bfm_dist_last_error(void) { return g_dist_err.c_str(); }

int bfm_nccl_unique_id(unsigned char* out128) {
  return dguard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int bfm_comm_create_nccl(const unsigned char* id128, int rank, int nranks, bfm_comm** out) {
  return dguard([&] {
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks)
      throw std::invalid_argument("bfm_comm_create_nccl: bad arguments");
    std::unique_ptr<bfm_comm> c(new bfm_comm);
    c->c.reset(new NcclComm(id128, rank, nranks));
    *out = c.release();
  });
}

int bfm_comm_create_local_group(int nranks, bfm_comm** out) {
  return dguard([&] {
    if (nranks < 1 || !out) throw std::invalid_argument("bfm_comm_create_local_group: bad arguments");
    auto g = std::make_shared<LocalGroup>(nranks);
    for (int r = 0; r < nranks; ++r) {
      out[r] = new bfm_comm;
      out[r]->c.reset(new LocalComm(g, r));
    }
  });
}

void bfm_comm_destroy(bfm_comm* c) { delete c; }

int bfm_dist_solver_create(bfm_comm* comm, int dim, const int* extents, const double* mu_rows,
                           const double* nu_rows, const bfm_config* cfg, bfm_dist_solver** out) {
  return dguard([&] {
    if (!comm || !extents || !mu_rows || !nu_rows || !out)
      throw std::invalid_argument("bfm_dist_solver_create: null argument");
    *out = nullptr;
    bfm_config c;
    bfm_config_default(&c);
    if (cfg) c = *cfg;
    std::unique_ptr<bfm_dist_solver> s(new bfm_dist_solver(comm->c.get(), dim, extents));
    s->setup(mu_rows, nu_rows, c);
    *out = s.release();
  });
}

void bfm_dist_solver_destroy(bfm_dist_solver* s) { delete s; }

int bfm_dist_solver_rows(const bfm_dist_solver* s, int* row0, int* nrows) {
  return dguard([&] {
    if (!s || !row0 || !nrows) throw std::invalid_argument("bfm_dist_solver_rows: null argument");
    *row0 = static_cast<int>(s->L.row0[s->rank]);
    *nrows = static_cast<int>(s->nr);
  });
}

int bfm_dist_solver_step(bfm_dist_solver* s, bfm_iteration_stats* out) {
  return dguard([&] {
    if (!s) throw std::invalid_argument("bfm_dist_solver_step: null handle");
    const bfm_iteration_stats st = s->step();
    if (out) *out = st;
  });
}

int bfm_dist_solver_probe(bfm_dist_solver* s, double* dual, double* residual) {
  return dguard([&] {
    if (!s) throw std::invalid_argument("bfm_dist_solver_probe: null handle");
    s->ensure_probe();
    if (dual) *dual = s->probe_dual;
    if (residual) *residual = std::sqrt(std::max(s->probe_gn, 0.0));
  });
}

int bfm_dist_solver_run(bfm_dist_solver* s, bfm_report* out) {
  return dguard([&] {
    if (!s) throw std::invalid_argument("bfm_dist_solver_run: null handle");
    bfm_report r;
    std::memset(&r, 0, sizeof(r));
    s->run(&r);
    if (out) *out = r;
  });
}

int bfm_dist_solver_field(bfm_dist_solver* s, int which, double* host_rows) {
  return dguard([&] {
    if (!s || !host_rows) throw std::invalid_argument("bfm_dist_solver_field: null argument");
    const double* src = which == BFM_FIELD_PHI ? s->phi.p : which == BFM_FIELD_PSI ? s->psi.p : nullptr;
    if (!src) throw std::invalid_argument("bfm_dist_solver_field: PHI or PSI only");
    BFM_CUDA(cudaMemcpyAsync(host_rows, src, sizeof(double) * s->nloc, cudaMemcpyDeviceToHost, s->stream));
    BFM_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int bfm_dist_solver_report_field(bfm_dist_solver* s, int which, double* host_full) {
  return dguard([&] {
    if (!s || !host_full) throw std::invalid_argument("bfm_dist_solver_report_field: null argument");
    if (!s->has_report) throw std::runtime_error("no report: call bfm_dist_solver_run first");
    const long N = s->L.N;
    if (which == BFM_FIELD_PHI) std::memcpy(host_full, s->rep_phi.data(), sizeof(double) * N);
    else if (which == BFM_FIELD_PSI) std::memcpy(host_full, s->rep_psi.data(), sizeof(double) * N);
    else if (which >= BFM_FIELD_MAP0 && which - BFM_FIELD_MAP0 < s->L.d)
      std::memcpy(host_full, s->rep_map.data() + (which - BFM_FIELD_MAP0) * N, sizeof(double) * N);
    else throw std::invalid_argument("bfm_dist_solver_report_field: bad field");
  });
}

int bfm_dist_solver_trace(const bfm_dist_solver* s, bfm_iteration_stats* out, int cap, int* count) {
  return dguard([&] {
    if (!s || !count || (cap > 0 && !out)) throw std::invalid_argument("bfm_dist_solver_trace: null argument");
    *count = static_cast<int>(s->trace.size());
    for (int i = 0; i < cap && i < *count; ++i) out[i] = s->trace[i];
  });
}

// k steps (each followed by the next iteration's probe, as run() pays it)
// between CUDA events on the solver's stream; device milliseconds
int bfm_dist_solver_time_steps(bfm_dist_solver* s, int k, double* ms) {
  return dguard([&] {
    if (!s || !ms || k < 0) throw std::invalid_argument("bfm_dist_solver_time_steps: bad argument");
    s->ensure_probe();
    cudaEvent_t e0, e1;
    BFM_CUDA(cudaEventCreate(&e0));
    BFM_CUDA(cudaEventCreate(&e1));
    BFM_CUDA(cudaEventRecord(e0, s->stream));
    for (int i = 0; i < k; ++i) {
      s->step();
      s->ensure_probe();
    }
    BFM_CUDA(cudaEventRecord(e1, s->stream));
    BFM_CUDA(cudaEventSynchronize(e1));
    float f = 0.0f;
    BFM_CUDA(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = f;
  });
}

int bfm_dist_solver_iteration(const bfm_dist_solver* s) { return s ? s->iteration : -1; }
double bfm_dist_solver_sigma(const bfm_dist_solver* s) {
  return s ? s->sigma : std::numeric_limits<double>::quiet_NaN();
}

}  // extern "C"
