// Host-side BFM iterate and the C ABI (include/bfm_b200.h).
//
// bfm_solver mirrors the reference's bfm::Solver (solver.hpp:146-368): same
// validation (checked on the host on the caller's arrays, exactly as
// solver.hpp:105-142), same probe/step split, stopping-rule order, step-size
// rule, dual-monotonicity checks and gauge fix. All field work runs on the
// device through CtPlan / PushforwardPlan / PoissonPlan / Reducer; only
// scalars cross to the host (one synchronising read per half step).
#include <cctype>
#include <cstdlib>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/bfm_b200.h"
#include "common.cuh"
#include "ctransform.cuh"
#include "ctransform_power.cuh"
#include "poisson.cuh"
#include "pushforward.cuh"
#include "reduce.cuh"
#include "pow_dd.h"
#include "solver_ctl.cuh"

namespace bfmgpu {
void debug_pow_device(const double* h_x, const double* h_y, int n, double* h_out);
int synthetic_densities(int config, int n, uint64_t seed, double* mu, double* nu, std::string& msg);
void debug_round_down(const double* h_terms, int m, int count, double* h_out);
void debug_fold(const double* h_w, const long* h_off, int nseq, int mode, double* h_out);
}

namespace {

using namespace bfmgpu;

thread_local std::string g_err;

struct BfmError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw BfmError{code, msg}; }

template <class F>
int guard(F&& f) {
  try {
    f();
    return BFM_OK;
  } catch (const BfmError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const CudaError& e) {
    g_err = e.what();
    return BFM_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return BFM_ERR_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& e) {
    g_err = "out of memory";
    return BFM_ERR_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BFM_ERR_ERROR;
  }
}

// grid.hpp:60-76 validation.
GridDesc checked_grid(int dim, const int* ext) {
  if (dim < 1 || dim > 3) fail(BFM_ERR_INVALID_ARGUMENT, "grid dimension must be 1, 2, or 3");
  for (int a = 0; a < dim; ++a)
    if (ext[a] < 2) fail(BFM_ERR_INVALID_ARGUMENT, "grid extent must be at least 2");
  return make_grid(dim, ext);
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(BFM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
}

// grid.hpp:124-133 Kahan accumulator (host-side validation only).
struct Kahan {
  double sum = 0.0, carry = 0.0;
  void add(double v) {
    const double y = v - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
};

// solver.hpp:105-116
void check_density(const char* name, const double* f, const GridDesc& g) {
  for (long i = 0; i < g.size; ++i) {
    const double v = f[i];
    if (!std::isfinite(v))
      fail(BFM_ERR_INFEASIBLE_INPUT, std::string(name) + ": density has a non-finite sample");
    if (v < 0.0) fail(BFM_ERR_NEGATIVE_INPUT, std::string(name) + ": density has a negative sample");
  }
  Kahan k;
  for (long i = 0; i < g.size; ++i) k.add(f[i]);
  const double mass = k.sum * g.vol;
  if (std::abs(mass - 1.0) > 1e-6)
    fail(BFM_ERR_INFEASIBLE_INPUT, std::string(name) + ": density mass " + std::to_string(mass) +
                                       " is not 1; normalize inputs first");
}

// solver.hpp:118-128
void check_config(const bfm_config& c) {
  if (c.max_iterations < 0) fail(BFM_ERR_INVALID_ARGUMENT, "solve: max_iterations is negative");
  if (c.threads < 0) fail(BFM_ERR_INVALID_ARGUMENT, "solve: threads is negative");
  if (c.sigma_init < 0.0) fail(BFM_ERR_INVALID_ARGUMENT, "solve: sigma_init is negative");
  if (c.sigma_min <= 0.0) fail(BFM_ERR_INVALID_ARGUMENT, "solve: sigma_min must be positive");
  if (!(c.beta_1 > 0.0) || !(c.beta_1 < c.beta_2) || !(c.beta_2 < 1.0))
    fail(BFM_ERR_INVALID_ARGUMENT, "solve: need 0 < beta_1 < beta_2 < 1");
  if (!(c.alpha_2 < 1.0) || !(c.alpha_2 > 0.0) || !(c.alpha_1 > 1.0))
    fail(BFM_ERR_INVALID_ARGUMENT, "solve: need 0 < alpha_2 < 1 < alpha_1");
  if (c.exact_tolerance < 0.0) fail(BFM_ERR_INVALID_ARGUMENT, "solve: exact_tolerance is negative");
}

void default_config(bfm_config* c) {
  c->mode = BFM_MODE_BACK_AND_FORTH;
  c->tolerance = 1e-4;
  c->max_iterations = 2000;
  c->threads = 0;
  c->sigma_init = 0.0;
  c->sigma_min = 0.01;
  c->beta_1 = 0.25;
  c->beta_2 = 0.75;
  c->alpha_1 = 1.25;
  c->alpha_2 = 0.8;
  c->has_exact_cost = 0;
  c->exact_cost = 0.0;
  c->exact_tolerance = 0.0;
}

double update_sigma(double sigma, double increase, double gn, const bfm_config& c) {
  const double predicted = sigma * gn;  // solver.hpp:68-76
  if (increase < c.beta_1 * predicted) sigma *= c.alpha_2;
  else if (increase > c.beta_2 * predicted) sigma *= c.alpha_1;
  return std::max(sigma, c.sigma_min);
}

struct DevBuf {
  double* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(long n) { BFM_CUDA(dmalloc(&p, n * sizeof(double))); }
  ~DevBuf() {
    if (p) dfree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void alloc(long n) {
    if (!p) BFM_CUDA(dmalloc(&p, n * sizeof(double)));
  }
};

enum { kSlotPair = 0, kSlotGn = 1, kSlotShift = 2, kSlotPrimal = 3, kSlotGn2 = 4 };

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host <-> device copies of a field: direct from/to pinned memory, otherwise
// through two pinned staging chunks so the DMA overlaps the host-side copy.
constexpr size_t kStage = size_t(8) << 20;  // bytes per staging chunk
struct Staging {
  double* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Staging() {
    for (int i = 0; i < 2; ++i) {
      BFM_CUDA(cudaMallocHost(&buf[i], kStage));
      BFM_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
};
// Per thread and device: the pinned chunks and events belong to the device
// that was current when they were made (bfm_set_device may switch later).
Staging& staging() {
  static thread_local std::unique_ptr<Staging> per_dev[64];
  int dev = 0;
  BFM_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) throw CudaError("staging: device index out of range");
  if (!per_dev[dev]) per_dev[dev].reset(new Staging);
  return *per_dev[dev];
}

// Host-side copy of a staging chunk split over a few threads: the first touch
// of freshly allocated (pageable) output pages dominates a single-threaded copy.
void par_memcpy(void* dst, const void* src, size_t len) {
  constexpr size_t kPart = size_t(1) << 20;
  const int parts = static_cast<int>(std::min<size_t>(8, (len + kPart - 1) / kPart));
  if (parts <= 1) {
    std::memcpy(dst, src, len);
    return;
  }
  const size_t step = (len + parts - 1) / parts;
  std::vector<std::thread> th;
  for (int i = 1; i < parts; ++i) {
    const size_t o = i * step;
    if (o >= len) break;
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(step, len - o));
    });
  }
  std::memcpy(dst, src, std::min(step, len));
  for (auto& t : th) t.join();
}

void copy_h2d(double* dst, const double* src, long n, cudaStream_t s) {
  const size_t bytes = n * sizeof(double);
  if (is_pinned(src) || bytes <= kStage) {
    BFM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    if (!is_pinned(src)) BFM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  Staging& st = staging();
  size_t off = 0;
  for (int b = 0; off < bytes; b ^= 1) {
    const size_t len = std::min(kStage, bytes - off);
    BFM_CUDA(cudaEventSynchronize(st.ev[b]));  // the chunk's previous DMA is done
    par_memcpy(st.buf[b], reinterpret_cast<const char*>(src) + off, len);
    BFM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, st.buf[b], len,
                             cudaMemcpyHostToDevice, s));
    BFM_CUDA(cudaEventRecord(st.ev[b], s));
    off += len;
  }
  BFM_CUDA(cudaStreamSynchronize(s));
}

void copy_d2h(double* dst, const double* src, long n, cudaStream_t s) {
  const size_t bytes = n * sizeof(double);
  if (is_pinned(dst) || bytes <= kStage) {
    BFM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    BFM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  Staging& st = staging();
  size_t off = 0, prev_off = 0, prev_len = 0;
  int b = 0;
  while (off < bytes || prev_len) {
    size_t len = 0;
    if (off < bytes) {
      len = std::min(kStage, bytes - off);
      BFM_CUDA(cudaMemcpyAsync(st.buf[b], reinterpret_cast<const char*>(src) + off, len,
                               cudaMemcpyDeviceToHost, s));
      BFM_CUDA(cudaEventRecord(st.ev[b], s));
    }
    if (prev_len) {  // previous chunk: wait for its DMA, then copy out while this one flies
      BFM_CUDA(cudaEventSynchronize(st.ev[b ^ 1]));
      par_memcpy(reinterpret_cast<char*>(dst) + prev_off, st.buf[b ^ 1], prev_len);
    }
    prev_off = off;
    prev_len = len;
    off += len;
    b ^= 1;
  }
}

}  // namespace

struct bfm_workspace {
  GridDesc g;
  // host-pointer operator calls (bfm_workspace_ctransform / _solve_neumann):
  // device copies of the operand and result, and a stream, made on first use
  DevBuf io_in, io_out;
  cudaStream_t io_stream = nullptr;
  ~bfm_workspace() {
    if (io_stream) cudaStreamDestroy(io_stream);
  }
  cudaStream_t io() {
    if (!io_stream) BFM_CUDA(cudaStreamCreateWithFlags(&io_stream, cudaStreamNonBlocking));
    io_in.alloc(g.size);
    io_out.alloc(g.size);
    return io_stream;
  }
  std::unique_ptr<CtPlan> ct;
  std::unique_ptr<PoissonPlan> pois;
  std::unique_ptr<PushforwardPlan> pf;
  std::unique_ptr<Reducer> red;
  LaunchCounter lc;
  int last_launches = 0;
  CtPlan& ctp() {
    if (!ct) {
      ct.reset(new CtPlan);
      ct->init(g);
    }
    return *ct;
  }
  PoissonPlan& poisp() {
    if (!pois) {
      pois.reset(new PoissonPlan);
      pois->init(g);
    }
    return *pois;
  }
  PushforwardPlan& pfp() {
    if (!pf) {
      pf.reset(new PushforwardPlan);
      pf->init(g);
    }
    return *pf;
  }
  Reducer& redp() {
    if (!red) {
      red.reset(new Reducer);
      red->init();
    }
    return *red;
  }
};

// Rank-local plans of the multi-GPU slab decomposition.
struct bfm_slab {
  GridDesc g;  // global grid
  int row0 = 0, nrows = 0;
  long col0 = 0;
  int ncols = 0;
  LaunchCounter lc;
  int last_launches = 0;
  CtPlan ct_cols, ct_rows;
  PoissonPlan pois_rows, pois_cols;
  PushforwardPlan pf;
  Reducer red;
};

struct bfm_solver {
  GridDesc g;
  bfm_config cfg;
  CtlConfig kcfg;
  cudaStream_t stream = nullptr;
  bfm_workspace ws;
  DevBuf mu, nu, phi, psi, dir, dir2, r;
  DevBuf rep_phi, rep_psi, rep_map;
  double sigma0 = 0.0;
  // Side stream: the pair-value reductions and every decision kernel run on
  // it, overlapping the bandwidth-bound reductions with the issue-bound
  // c-transform / pushforward kernels of the main stream (events order the
  // hazards; see enqueue_step). Its reductions use their own Reducer.
  cudaStream_t side = nullptr;
  Reducer side_red;
  cudaEvent_t xev[16] = {};
  int xev_i = 0;
  // separable power cost (cost.hpp:17-81): exponents per axis, the exact
  // c-transform on dense axis-cost tables and the pow inverse-gradient map
  bool power = false;
  double pexp[3] = {2.0, 2.0, 2.0};
  std::unique_ptr<CtPowerPlan> ctpow;
  // Scalar state lives on the device (solver_ctl.cuh); h is the pinned mirror
  // every unit copies back, ring the per-step stats of a batch.
  SolverCtl* d_ctl = nullptr;
  SolverCtl* h_ctl = nullptr;
  CtlStats* d_ring = nullptr;
  CtlStats* h_ring = nullptr;
  int iteration = 0;
  bool fresh = false;
  bool probe_blowup = false;  // certified blow-up in a prefetched probe (thrown when consumed)
  bool has_report = false;
  bool use_graphs = true;
  int force_near_iter = -1, force_near_probe = 0;  // test hook (bfm_solver_debug_force_exact)
  long exact_replays = 0;
  std::vector<bfm_iteration_stats> trace;
  std::chrono::steady_clock::time_point start;

  // Optional per-operator device timing (bench.py's live roofline): events
  // recorded on the solver stream around each operator (external event nodes
  // inside captured graphs), resolved after the unit's synchronisation.
  bool timing = false;
  struct Pending {
    cudaEvent_t a, b;
    int op;
  };
  std::vector<Pending> pending;         // eager launches
  std::vector<Pending>* capture_ev = nullptr;  // set while capturing a graph
  std::vector<const std::vector<Pending>*> graph_pending;
  std::vector<cudaEvent_t> free_events;
  double op_ms[BFM_OP_COUNT] = {};
  long op_n[BFM_OP_COUNT] = {};

  // One iteration unit as a CUDA graph: kind 0 probe, 1 step, 2 step + probe.
  struct UnitGraph {
    cudaGraphExec_t exec = nullptr;
    long launches = 0;
    int uses = 0;
    std::vector<Pending> ev;
  };
  UnitGraph graphs[3][2];

  cudaEvent_t take_event() {
    if (free_events.empty()) {
      cudaEvent_t e;
      BFM_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  // NVTX range per operator (visible in nsys / ncu --nvtx; free without a tool)
  static const char* op_name(int op) {
    static const char* names[BFM_OP_COUNT] = {"bfm.ctransform", "bfm.pushforward", "bfm.poisson",
                                              "bfm.reduce"};
    return op >= 0 && op < BFM_OP_COUNT ? names[op] : "bfm.op";
  }
  template <class F>
  void timed(int op, F&& f, cudaStream_t on = nullptr) {
    nvtxRangePushA(op_name(op));
    struct Pop {
      ~Pop() { nvtxRangePop(); }
    } pop;
    if (!timing) {
      f();
      return;
    }
    const cudaStream_t st = on ? on : stream;
    cudaEvent_t a = take_event(), b = take_event();
    if (capture_ev) {
      BFM_CUDA(cudaEventRecordWithFlags(a, st, cudaEventRecordExternal));
      f();
      BFM_CUDA(cudaEventRecordWithFlags(b, st, cudaEventRecordExternal));
      capture_ev->push_back({a, b, op});
      return;
    }
    BFM_CUDA(cudaEventRecord(a, st));
    f();
    BFM_CUDA(cudaEventRecord(b, st));
    pending.push_back({a, b, op});
  }
  // cross-stream ordering (dependency edges inside a captured graph)
  cudaEvent_t next_xev() {
    cudaEvent_t& e = xev[xev_i++ & 15];
    if (!e) BFM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }
  cudaEvent_t mark(cudaStream_t st) {
    const cudaEvent_t e = next_xev();
    BFM_CUDA(cudaEventRecord(e, st));
    return e;
  }
  // With per-operator timing on, the side work runs on the main stream
  // (serialised: each operator's events then time that operator alone).
  cudaStream_t sd() const { return timing ? stream : side; }
  void side_after_main() {
    if (!timing) BFM_CUDA(cudaStreamWaitEvent(side, mark(stream), 0));
  }
  void main_after_side() {
    if (!timing) BFM_CUDA(cudaStreamWaitEvent(stream, mark(side), 0));
  }
  void add_time(const Pending& q) {
    BFM_CUDA(cudaEventSynchronize(q.b));
    float ms = 0.0f;
    BFM_CUDA(cudaEventElapsedTime(&ms, q.a, q.b));
    op_ms[q.op] += ms;
    op_n[q.op] += 1;
  }
  void resolve_times() {
    for (const Pending& q : pending) {
      add_time(q);
      free_events.push_back(q.a);
      free_events.push_back(q.b);
    }
    pending.clear();
    for (const auto* v : graph_pending)
      for (const Pending& q : *v) add_time(q);
    graph_pending.clear();
  }

  ~bfm_solver() {
    for (cudaEvent_t e : xev)
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    for (const Pending& q : pending) {
      cudaEventDestroy(q.a);
      cudaEventDestroy(q.b);
    }
    for (auto& row : graphs)
      for (UnitGraph& G : row) {
        if (G.exec) cudaGraphExecDestroy(G.exec);
        for (const Pending& q : G.ev) {
          cudaEventDestroy(q.a);
          cudaEventDestroy(q.b);
        }
      }
    for (cudaEvent_t e : free_events) cudaEventDestroy(e);
    if (d_ctl) dfree(d_ctl);
    if (d_ring) dfree(d_ring);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (h_ring) cudaFreeHost(h_ring);
    if (stream) cudaStreamDestroy(stream);
  }

  // ---- scalar state -------------------------------------------------------
  void init_ctl() {  // solver.hpp:148-167,360-368
    std::memset(h_ctl, 0, sizeof(SolverCtl));
    h_ctl->sigma = sigma0;
    h_ctl->last_pair = 0.0;
    h_ctl->prev_dual = std::numeric_limits<double>::quiet_NaN();
    upload_ctl();
  }
  void upload_ctl() {
    BFM_CUDA(cudaMemcpyAsync(d_ctl, h_ctl, sizeof(SolverCtl), cudaMemcpyHostToDevice, stream));
    BFM_CUDA(cudaStreamSynchronize(stream));
  }
  // decisions run on the side stream in program order (they share ctl);
  // pair values come from the side Reducer, gn values from the main one
  void decide(int stage, int slot) {
    const double* res = (slot == kSlotGn || slot == kSlotGn2) ? ws.redp().device_results()
                                                              : side_red.device_results();
    timed(BFM_OP_REDUCE, [&] {
      ctl_decide(d_ctl, res, slot, slot >= 0 ? kBoundSlot + slot : 0, stage, kcfg, d_ring, sd(), &ws.lc);
    }, sd());
  }

  // ---- device units (no host synchronisation) ------------------------------
  // pair value on the side stream, after the main stream's pending work
  void pair_value_async() {  // solver.hpp:240
    side_after_main();
    timed(BFM_OP_REDUCE, [&] {
      side_red.dot(phi.p, nu.p, psi.p, mu.p, g.size, g.vol, kSlotPair, sd(), &ws.lc);
    }, sd());
  }
  // before_last: the output's readers on the side stream (the last pass waits)
  // concave: the input is itself a c-transform (a speed hint for the plan, see CtPlan::run)
  void ctransform(const double* in, double* out, cudaEvent_t before_last = nullptr, bool concave = false) {
    timed(BFM_OP_CTRANSFORM, [&] {
      if (power) {
        if (before_last) BFM_CUDA(cudaStreamWaitEvent(stream, before_last, 0));
        ctpow->run(in, out, stream, &ws.lc);
      } else {
        ws.ctp().run(in, out, stream, &ws.lc, before_last, concave);
      }
    });
  }
  void axpy_device(double* u, const double* d) {
    timed(BFM_OP_REDUCE, [&] { axpy_dev(u, &d_ctl->sigma, d, g.size, stream, &ws.lc); });
  }
  // solver.hpp:245-260 (result left in d_dir, gn in gn_slot of the main Reducer)
  void ascent_direction_async(const double* u, const double* source, const double* target,
                              double* d_dir, int gn_slot = kSlotGn) {
    timed(BFM_OP_PUSHFORWARD,
          [&] { ws.pfp().from_potential(u, source, target, r.p, nullptr, stream, &ws.lc); });
    timed(BFM_OP_POISSON, [&] { ws.poisp().solve(r.p, d_dir, stream, &ws.lc); });
    timed(BFM_OP_REDUCE, [&] {
      ws.redp().dot(r.p, d_dir, nullptr, nullptr, g.size, g.vol, gn_slot, stream, &ws.lc);
    });
  }
  // Stream layout of a unit. Main: axpys, c-transforms, ascents (gn). Side:
  // pair values and decisions. A pair value reads phi and psi while the next
  // c-transform's early passes run; that c-transform's LAST pass (which
  // overwrites one of them) waits for it (pending_read). An axpy waits for
  // the decision that produced its sigma.
  cudaEvent_t pending_read = nullptr;  // side-stream reads of phi/psi not yet fenced
  // which c-concave-input calls ask for the staged c-transform kernel (bit 0:
  // the probe's phi -> psi, bit 1: the step's psi -> phi); BFM_CT_HINTS overrides
  int ct_hints = getenv("BFM_CT_HINTS") ? atoi(getenv("BFM_CT_HINTS")) : 3;
  void enqueue_probe() {  // solver.hpp:264-280
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      ctransform(phi.p, psi.p, pending_read, (ct_hints & 1) != 0);  // phi = psi^c from the last step
      pending_read = nullptr;
      pair_value_async();
      pending_read = timing ? nullptr : mark(side);
      decide(kStageProbePair, kSlotPair);
    } else {
      decide(kStageProbeGA, -1);
    }
    ascent_direction_async(psi.p, mu.p, nu.p, dir.p, kSlotGn);
    side_after_main();
    decide(kStageProbeGn, kSlotGn);
  }
  void enqueue_step() {  // solver.hpp:286-328
    decide(kStageStepBegin, -1);
    main_after_side();  // sigma, and the side stream's reads of phi/psi
    pending_read = nullptr;
    axpy_device(phi.p, dir.p);
    ctransform(phi.p, psi.p);
    pair_value_async();
    pending_read = timing ? nullptr : mark(side);
    decide(kStageFirst, kSlotPair);
    ctransform(psi.p, phi.p, pending_read, (ct_hints & 2) != 0);  // psi = phi^c
    pending_read = nullptr;
    pair_value_async();
    pending_read = timing ? nullptr : mark(side);
    if (cfg.mode != BFM_MODE_BACK_AND_FORTH) {
      decide(kStageGAv3, kSlotPair);
      return;
    }
    decide(kStageV4, kSlotPair);
    ascent_direction_async(phi.p, nu.p, mu.p, dir2.p, kSlotGn2);
    side_after_main();
    decide(kStageGn2, kSlotGn2);
    main_after_side();  // sigma (kStageFirst) and the pair value's read of psi
    pending_read = nullptr;
    axpy_device(psi.p, dir2.p);
    ctransform(psi.p, phi.p);
    pair_value_async();
    pending_read = timing ? nullptr : mark(side);
    decide(kStageV5, kSlotPair);
  }
  void enqueue_unit(int kind) {
    pending_read = nullptr;
    side_after_main();  // forks the side stream into a capture; orders it after main's prior work
    if (kind != 1 && kind != 2) enqueue_probe();
    if (kind != 0) enqueue_step();
    if (kind == 2) enqueue_probe();
    main_after_side();  // every decision is in ctl before the copy back
    pending_read = nullptr;
    BFM_CUDA(cudaMemcpyAsync(h_ctl, d_ctl, sizeof(SolverCtl), cudaMemcpyDeviceToHost, stream));
  }
  // Launches one unit: eagerly the first time (plans allocate lazily), then as
  // a captured CUDA graph replayed with a single launch.
  void launch_unit(int kind) {
    static const char* unit_names[3] = {"bfm.probe", "bfm.step", "bfm.step+probe"};
    nvtxRangePushA(unit_names[kind]);
    struct Pop {
      ~Pop() { nvtxRangePop(); }
    } pop;
    if (!use_graphs) return enqueue_unit(kind);
    UnitGraph& G = graphs[kind][timing ? 1 : 0];
    if (G.uses++ == 0) return enqueue_unit(kind);
    if (!G.exec) {
      const long before = ws.lc.count;
      cudaGraph_t graph = nullptr;
      BFM_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      capture_ev = &G.ev;
      try {
        enqueue_unit(kind);
      } catch (...) {
        capture_ev = nullptr;
        cudaStreamEndCapture(stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      capture_ev = nullptr;
      BFM_CUDA(cudaStreamEndCapture(stream, &graph));
      const cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
      cudaGraphDestroy(graph);
      BFM_CUDA(e);
      G.launches = ws.lc.count - before;
      ws.lc.count = before;
    }
    BFM_CUDA(cudaGraphLaunch(G.exec, stream));
    ws.lc.add(G.launches);
    if (timing) graph_pending.push_back(&G.ev);
  }
  void sync() {
    BFM_CUDA(cudaStreamSynchronize(stream));
    if (timing) resolve_times();
  }
  void clear_flags() {
    BFM_CUDA(cudaMemsetAsync(&d_ctl->flags, 0, sizeof(int), stream));
  }

  [[noreturn]] void blowup() {
    fail(BFM_ERR_NUMERICAL_BLOWUP, "solve: conjugation decreased the dual pair value");
  }

  // ---- exact scalars (rare path) ------------------------------------------
  // The reference's sequential Kahan sums (grid.hpp:124-133,171-176) of the
  // device fields, on the host.
  std::vector<double> host_field(const double* d) {
    std::vector<double> h(g.size);
    copy_d2h(h.data(), d, g.size, stream);
    return h;
  }
  double kahan_dot(const double* da, const double* db) {
    const std::vector<double> a = host_field(da), b = host_field(db);
    Kahan k;
    for (long i = 0; i < g.size; ++i) k.add(a[i] * b[i]);
    return k.sum * g.vol;
  }
  double kahan_pair() { return kahan_dot(phi.p, nu.p) + kahan_dot(psi.p, mu.p); }  // solver.hpp:240

  void exact_probe() {  // solver.hpp:264-280 with reference-order scalars
    SolverCtl& c = *h_ctl;
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      ctransform(phi.p, psi.p);
      const double v = kahan_pair();
      if (v < c.last_pair - 1e-10) blowup();
      c.last_pair = v;
      c.last_pair_b = 0.0;
      c.probe_dual = v;
    } else {
      c.probe_dual = c.last_pair;
    }
    c.probe_dual_b = 0.0;
    ascent_direction_async(psi.p, mu.p, nu.p, dir.p);
    c.probe_gn = kahan_dot(r.p, dir.p);
    c.probe_gn_b = 0.0;
  }
  bfm_iteration_stats exact_step() {  // solver.hpp:189-207,286-328
    SolverCtl& c = *h_ctl;
    bfm_iteration_stats st;
    std::memset(&st, 0, sizeof(st));
    st.iteration = iteration + 1;
    st.residual = std::sqrt(std::max(c.probe_gn, 0.0));
    st.sigma_first = c.sigma;
    st.grad_norm_sq_first = c.probe_gn;
    timed(BFM_OP_REDUCE, [&] { axpy(phi.p, c.sigma, dir.p, g.size, stream, &ws.lc); });
    ctransform(phi.p, psi.p);
    const double v2 = c.probe_dual, v3 = kahan_pair();
    st.increase_first = v3 - v2;
    c.sigma = update_sigma(c.sigma, st.increase_first, c.probe_gn, cfg);
    ctransform(psi.p, phi.p);
    const double v4 = kahan_pair();
    if (v4 < v3 - 1e-10) blowup();
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      ascent_direction_async(phi.p, nu.p, mu.p, dir2.p);
      const double gn2 = kahan_dot(r.p, dir2.p);
      st.sigma_second = c.sigma;
      st.grad_norm_sq_second = gn2;
      timed(BFM_OP_REDUCE, [&] { axpy(psi.p, c.sigma, dir2.p, g.size, stream, &ws.lc); });
      ctransform(psi.p, phi.p);
      const double v5 = kahan_pair();
      st.increase_second = v5 - v4;
      c.sigma = update_sigma(c.sigma, st.increase_second, gn2, cfg);
      st.dual_value = v5;
    } else {
      st.dual_value = v4;
    }
    c.last_pair = st.dual_value;
    c.last_pair_b = 0.0;
    if (std::abs(st.dual_value - c.prev_dual) < 1e-12) ++c.stall;
    else c.stall = 0;
    c.prev_dual = st.dual_value;
    c.prev_dual_b = 0.0;
    return st;
  }

  // Iteration k's probe (and its step when with_step) could not be certified
  // to follow the reference's branches: recompute from the initial state —
  // iterations 1..k-1 on the device (their decisions were certified, so they
  // reproduce bit for bit), then iteration k with every scalar in the
  // reference's Kahan order. Leaves iteration = k (or k-1 with a fresh probe).
  void replay_exact(int k, bool with_step) {
    ++exact_replays;
    for (DevBuf* b : {&phi, &psi})
      BFM_CUDA(cudaMemsetAsync(b->p, 0, g.size * sizeof(double), stream));
    init_ctl();
    for (int j = 1; j < k; ++j) {
      clear_flags();
      enqueue_unit(0);
      enqueue_unit(1);
    }
    sync();
    if (k > 1 && (h_ctl->flags & (kCtlNear | kCtlBlowup)))
      fail(BFM_ERR_ERROR, "internal error: device replay diverged from the certified run");
    if (h_ctl->done != k - 1) fail(BFM_ERR_ERROR, "internal error: replay iteration count");
    if (k > 1) {  // the end-of-iteration pair value in the reference's order
      const double v = kahan_pair();
      h_ctl->last_pair = h_ctl->prev_dual = v;
      h_ctl->last_pair_b = h_ctl->prev_dual_b = 0.0;
    }
    iteration = k - 1;
    trace.resize(k - 1);
    exact_probe();
    fresh = true;
    probe_blowup = false;
    if (with_step) {
      const bfm_iteration_stats st = exact_step();
      trace.push_back(st);
      iteration = k;
      h_ctl->done = k;
      fresh = false;
    }
    h_ctl->flags = 0;
    upload_ctl();
  }

  // ---- host API -----------------------------------------------------------
  void ensure_probe() {  // solver.hpp:264-280
    if (fresh) {
      if (probe_blowup) blowup();
      return;
    }
    clear_flags();
    launch_unit(0);
    sync();
    const int done = h_ctl->done;
    if ((h_ctl->flags & kCtlNear) || (force_near_iter == done + 1 && force_near_probe)) {
      force_near_iter = -1;
      replay_exact(done + 1, false);
      return;
    }
    if (h_ctl->flags & kCtlBlowup) blowup();
    fresh = true;
  }

  // n consecutive steps with one synchronisation (prefetch: also the probe
  // that follows the last step). Stats come back through the device ring.
  void steps(int n, bool prefetch, cudaEvent_t end_event = nullptr) {
    ensure_probe();
    if (n > kCtlRing) n = kCtlRing;
    const int done0 = h_ctl->done;
    clear_flags();
    for (int i = 0; i < n; ++i) launch_unit(i + 1 < n || prefetch ? 2 : 1);
    if (end_event) BFM_CUDA(cudaEventRecord(end_event, stream));
    if (n > 1)
      BFM_CUDA(cudaMemcpyAsync(h_ring, d_ring, kCtlRing * sizeof(CtlStats), cudaMemcpyDeviceToHost,
                               stream));
    sync();
    const SolverCtl c = *h_ctl;
    // Events of step j+1 (0-based j) and of the probe it consumed carry
    // near_iter / blowup_iter == j; probe stages order before step stages.
    auto key = [](int it, int stage) { return static_cast<long>(it) * 16 + stage; };
    const long near_at = (c.flags & kCtlNear) ? key(c.near_iter, c.near_stage) : LONG_MAX;
    const long blow_at = (c.flags & kCtlBlowup) ? key(c.blowup_iter, c.blowup_stage) : LONG_MAX;
    for (int j = done0; j < done0 + n; ++j) {
      const long end_j = key(j + 1, 0);
      const bool forced = force_near_iter == j + 1 && !force_near_probe;
      if (forced || (near_at < end_j && near_at < blow_at)) {
        // the first uncertified decision belongs to iteration j+1: replay it
        // with reference-order scalars (the later steps of the batch are redone)
        force_near_iter = -1;
        replay_exact(j + 1, true);
        if (prefetch) ensure_probe();
        return;
      }
      if (blow_at < end_j) {  // certified blow-up inside iteration j+1
        iteration = j;
        fresh = false;
        blowup();
      }
      const CtlStats& x = n > 1 ? h_ring[j % kCtlRing] : c.last;
      bfm_iteration_stats st;
      st.iteration = j + 1;
      st.residual = x.residual;
      st.dual_value = x.dual_value;
      st.sigma_first = x.sigma_first;
      st.sigma_second = x.sigma_second;
      st.grad_norm_sq_first = x.gn_first;
      st.grad_norm_sq_second = x.gn_second;
      st.increase_first = x.inc_first;
      st.increase_second = x.inc_second;
      trace.push_back(st);
      iteration = j + 1;
    }
    fresh = prefetch;
    probe_blowup = false;
    if (!prefetch) return;
    // the trailing probe belongs to iteration done0 + n + 1
    const int k = done0 + n + 1;
    if ((force_near_iter == k && force_near_probe) || (near_at != LONG_MAX && near_at < blow_at)) {
      force_near_iter = -1;
      replay_exact(k, false);
      return;
    }
    if (blow_at != LONG_MAX) probe_blowup = true;
  }

  bfm_iteration_stats step() {  // solver.hpp:189-207
    steps(1, false);
    return trace.back();
  }

  void finish(int term, double residual, bfm_report* rep) {  // solver.hpp:330-349
    rep->termination = term;
    rep->iterations = iteration;
    rep->dual_value = h_ctl->probe_dual;
    rep->residual = residual;
    rep_phi.alloc(g.size);
    rep_psi.alloc(g.size);
    rep_map.alloc(g.d * g.size);
    BFM_CUDA(cudaMemcpyAsync(rep_phi.p, phi.p, g.size * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    BFM_CUDA(cudaMemcpyAsync(rep_psi.p, psi.p, g.size * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    // The gauge shift feeds every reported field, so it must be the reference's
    // exact sequential Kahan sum (grid.hpp:179-183): computed on the host.
    std::vector<double> hphi(g.size);
    BFM_CUDA(cudaMemcpyAsync(hphi.data(), rep_phi.p, g.size * sizeof(double), cudaMemcpyDeviceToHost,
                             stream));
    BFM_CUDA(cudaStreamSynchronize(stream));
    Kahan k;
    for (long i = 0; i < g.size; ++i) k.add(hphi[i]);
    const double shift = k.sum * g.vol;
    add_scalar(rep_phi.p, -shift, g.size, stream, &ws.lc);
    add_scalar(rep_psi.p, shift, g.size, stream, &ws.lc);
    ws.pfp().map_only(rep_psi.p, rep_map.p, stream, &ws.lc);
    ws.redp().primal(rep_map.p, mu.p, g.d, g.size, g.vol, kSlotPrimal, stream, &ws.lc,
                     power ? pexp : nullptr);
    double v[kSlotPrimal + 1];
    ws.redp().fetch(v, kSlotPrimal + 1, stream);
    rep->primal_cost = v[kSlotPrimal];
    rep->wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    has_report = true;
  }

  void run(bfm_report* rep) {  // solver.hpp:211-226
    while (true) {
      ensure_probe();
      const SolverCtl& c = *h_ctl;
      const double residual = std::sqrt(std::max(c.probe_gn, 0.0));
      // the rules compare certified probe scalars: |sqrt(a) - sqrt(b)| <=
      // sqrt(|a - b|); a near tie replays the probe with exact scalars
      const double u4 = 4.0 * 0x1.0p-53;
      if (cfg.tolerance >= 0.0 &&
          near_tie(residual, std::sqrt(c.probe_gn_b) + u4 * residual, cfg.tolerance))
        continue;
      if (cfg.tolerance >= 0.0 && residual <= cfg.tolerance)
        return finish(BFM_TERM_TOLERANCE_MET, residual, rep);
      if (cfg.has_exact_cost && cfg.exact_tolerance > 0.0) {
        const double dev = std::abs(c.probe_dual - cfg.exact_cost);
        if (near_tie(dev, c.probe_dual_b + u4 * dev, cfg.exact_tolerance)) continue;
        if (dev <= cfg.exact_tolerance) return finish(BFM_TERM_COST_TARGET_MET, residual, rep);
      }
      if (iteration >= cfg.max_iterations) return finish(BFM_TERM_MAX_ITERATIONS, residual, rep);
      if (c.stall >= 10) return finish(BFM_TERM_DUAL_STALLED, residual, rep);
      // steps no rule can interrupt run back to back with one synchronisation:
      // only the iteration cap and the stall counter (+1 per step at most) apply
      int batch = 1;
      if (cfg.tolerance < 0.0 && !(cfg.has_exact_cost && cfg.exact_tolerance > 0.0) && !timing)
        batch = std::max(1, std::min(cfg.max_iterations - iteration, 10 - c.stall));
      steps(batch, true);
    }
  }

  // A stopping comparison x <= thr whose x is within its bound of thr: replay
  // the probe with reference-order scalars (then the loop re-evaluates).
  bool near_tie(double x, double bound, double thr) {
    if (!(bound > 0.0) || std::abs(x - thr) > 2.0 * bound) return false;
    replay_exact(iteration + 1, false);
    return true;
  }
};

namespace {

struct HostOp {
  GridDesc g;
  bfm_workspace ws;
  cudaStream_t s = nullptr;
  HostOp(int dim, const int* ext) {
    g = checked_grid(dim, ext);
    require_device();
    ws.g = g;
  }
  ~HostOp() { release(); }
  double* up(const double* h, long n) {
    double* d = nullptr;
    BFM_CUDA(dmalloc(&d, n * sizeof(double)));
    keep.push_back(d);
    if (h) BFM_CUDA(cudaMemcpy(d, h, n * sizeof(double), cudaMemcpyHostToDevice));
    return d;
  }
  void down(double* h, const double* d, long n) {
    BFM_CUDA(cudaDeviceSynchronize());
    BFM_CUDA(cudaMemcpy(h, d, n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  std::vector<double*> keep;
  void release() {
    for (double* p : keep) dfree(p);
    keep.clear();
  }
};

}  // namespace

namespace {
template <class F>
int slab_op(bfm_slab* s, F&& f) {
  return guard([&] {
    if (!s) fail(BFM_ERR_INVALID_ARGUMENT, "slab: null handle");
    const long before = s->lc.count;
    f();
    s->last_launches = static_cast<int>(s->lc.count - before);
  });
}
}  // namespace

extern "C" {

const char* bfm_last_error(void) { return g_err.c_str(); }

int bfm_debug_round_down(const double* terms, int m, int count, double* out) {
  return guard([&] {
    require_device();
    bfmgpu::debug_round_down(terms, m, count, out);
  });
}

int bfm_debug_pow(const double* x, const double* y, int n, int on_device, double* out) {
  return guard([&] {
    if (n < 0 || (n > 0 && (!x || !y || !out))) throw std::invalid_argument("debug_pow: bad arguments");
    if (!on_device) {
      for (int i = 0; i < n; ++i) out[i] = bfmpow::pow_cr(x[i], y[i]);
      return;
    }
    require_device();
    bfmgpu::debug_pow_device(x, y, n, out);
  });
}

int bfm_debug_fold(const double* w, const long* offsets, int nseq, int mode, double* out) {
  return guard([&] {
    require_device();
    if (nseq < 0 || (mode != 0 && mode != 1) || (nseq > 0 && (!w || !offsets || !out)))
      throw std::invalid_argument("debug_fold: bad arguments");
    bfmgpu::debug_fold(w, offsets, nseq, mode, out);
  });
}

int bfm_set_device(int device) {
  return guard([&] { BFM_CUDA(cudaSetDevice(device)); });
}

int bfm_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n > 0 ? 1 : 0;
}

void bfm_config_default(bfm_config* cfg) { default_config(cfg); }

double bfm_update_sigma(double sigma, double increase, double gn, const bfm_config* cfg) {
  bfm_config d;
  default_config(&d);
  return update_sigma(sigma, increase, gn, cfg ? *cfg : d);
}

int bfm_solver_create(int dim, const int* extents, const double* mu, const double* nu,
                      const bfm_config* cfg, bfm_solver** out) {
  return bfm_solver_create_cost(dim, extents, nullptr, mu, nu, cfg, out);
}

int bfm_solver_create_cost(int dim, const int* extents, const double* exponents, const double* mu,
                           const double* nu, const bfm_config* cfg, bfm_solver** out) {
  return guard([&] {
    *out = nullptr;
    bfm_config c;
    default_config(&c);
    if (cfg) c = *cfg;
    const GridDesc g = checked_grid(dim, extents);
    check_config(c);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      check_density("mu", mu, g);  // input errors take precedence, as before a device is needed
      check_density("nu", nu, g);
    }
    require_device();
    std::unique_ptr<bfm_solver> s(new bfm_solver);
    s->start = std::chrono::steady_clock::now();
    s->g = g;
    s->cfg = c;
    s->ws.g = g;
    BFM_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    BFM_CUDA(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
    s->side_red.init();
    const long N = g.size;
    for (DevBuf* b : {&s->mu, &s->nu, &s->phi, &s->psi, &s->dir, &s->dir2, &s->r}) b->alloc(N);
    copy_h2d(s->mu.p, mu, N, s->stream);
    copy_h2d(s->nu.p, nu, N, s->stream);
    BFM_CUDA(cudaMemsetAsync(s->phi.p, 0, N * sizeof(double), s->stream));
    BFM_CUDA(cudaMemsetAsync(s->psi.p, 0, N * sizeof(double), s->stream));
    // solver.hpp:105-116 on the device: sup, non-finite / negative flags and
    // the mass (double-double). Any flag, or a mass within 1e-9 of the
    // tolerance, re-runs the reference's exact host check (first offending
    // sample, sequential Kahan mass) so errors and messages are identical.
    Reducer& red = s->ws.redp();
    red.scan_density(s->mu.p, N, 4, s->stream, nullptr);
    red.scan_density(s->nu.p, N, 7, s->stream, nullptr);
    red.sum(s->mu.p, N, g.vol, 10, s->stream, nullptr);
    red.sum(s->nu.p, N, g.vol, 11, s->stream, nullptr);
    double v[12];
    red.fetch(v, 12, s->stream);
    auto needs_host = [](double bad, double neg, double mass) {
      return bad != 0.0 || neg != 0.0 || !(std::abs(std::abs(mass - 1.0) - 1e-6) > 1e-9);
    };
    if (needs_host(v[5], v[6], v[10]) || std::abs(v[10] - 1.0) > 1e-6) check_density("mu", mu, g);
    if (needs_host(v[8], v[9], v[11]) || std::abs(v[11] - 1.0) > 1e-6) check_density("nu", nu, g);
    const double sup = std::max(v[4], v[7]);  // solver.hpp:160-163
    s->sigma0 = c.sigma_init > 0.0 ? c.sigma_init : 8.0 / sup;
    if (exponents) {
      for (int a = 0; a < dim; ++a) {
        if (!(exponents[a] > 1.0)) fail(BFM_ERR_INVALID_ARGUMENT, "cost exponents must satisfy p > 1");
        s->pexp[a] = exponents[a];
        s->power = s->power || exponents[a] != 2.0;
      }
      if (s->power) {
        s->ctpow.reset(new CtPowerPlan);
        s->ctpow->init(g, exponents);
        s->ws.pfp().set_cost(exponents);
      }
    }
    s->kcfg = CtlConfig{c.beta_1, c.beta_2, c.alpha_1, c.alpha_2, c.sigma_min};
    BFM_CUDA(dmalloc(&s->d_ctl, sizeof(SolverCtl)));
    BFM_CUDA(dmalloc(&s->d_ring, kCtlRing * sizeof(CtlStats)));
    BFM_CUDA(cudaMallocHost(&s->h_ctl, sizeof(SolverCtl)));
    BFM_CUDA(cudaMallocHost(&s->h_ring, kCtlRing * sizeof(CtlStats)));
    s->init_ctl();
    if (const char* e = std::getenv("BFM_NO_GRAPHS")) s->use_graphs = e[0] == '0';
    s->ws.ctp();
    s->ws.poisp();
    s->ws.pfp();
    s->ws.redp();
    BFM_CUDA(cudaStreamSynchronize(s->stream));
    *out = s.release();
  });
}

void bfm_solver_destroy(bfm_solver* s) { delete s; }
int bfm_solver_iteration(const bfm_solver* s) { return s ? s->iteration : -1; }
double bfm_solver_sigma(const bfm_solver* s) {
  return s ? s->h_ctl->sigma : std::numeric_limits<double>::quiet_NaN();
}

int bfm_solver_dual_value(bfm_solver* s, double* out) {
  return guard([&] {
    if (!s || !out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_dual_value: null argument");
    s->ensure_probe();
    *out = s->h_ctl->probe_dual;
  });
}

int bfm_solver_residual(bfm_solver* s, double* out) {
  return guard([&] {
    if (!s || !out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_residual: null argument");
    s->ensure_probe();
    *out = std::sqrt(std::max(s->h_ctl->probe_gn, 0.0));
  });
}

int bfm_solver_step(bfm_solver* s, bfm_iteration_stats* out) {
  return guard([&] {
    if (!s) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_step: null handle");
    const bfm_iteration_stats st = s->step();
    if (out) *out = st;
  });
}

int bfm_solver_run(bfm_solver* s, bfm_report* out) {
  return guard([&] {
    if (!s) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_run: null handle");
    bfm_report r;
    std::memset(&r, 0, sizeof(r));
    s->run(&r);
    if (out) *out = r;
  });
}

int bfm_solver_trace(const bfm_solver* s, bfm_iteration_stats* out, int cap, int* count) {
  return guard([&] {
    if (!s || !count || (cap > 0 && !out))
      fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_trace: null argument");
    *count = static_cast<int>(s->trace.size());
    for (int i = 0; i < cap && i < *count; ++i) out[i] = s->trace[i];
  });
}

int bfm_solver_field(bfm_solver* s, int which, double* host_out) {
  return guard([&] {
    if (!s || !host_out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_field: null argument");
    const double* src = which == BFM_FIELD_PHI ? s->phi.p : which == BFM_FIELD_PSI ? s->psi.p : nullptr;
    if (!src) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_field: PHI or PSI only");
    copy_d2h(host_out, src, s->g.size, s->stream);
  });
}

int bfm_solver_report_field(bfm_solver* s, int which, double* host_out) {
  return guard([&] {
    if (!s || !host_out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_report_field: null argument");
    if (!s->has_report) fail(BFM_ERR_ERROR, "no report: call bfm_solver_run first");
    const double* src = nullptr;
    if (which == BFM_FIELD_PHI) src = s->rep_phi.p;
    else if (which == BFM_FIELD_PSI) src = s->rep_psi.p;
    else if (which >= BFM_FIELD_MAP0 && which - BFM_FIELD_MAP0 < s->g.d)
      src = s->rep_map.p + (which - BFM_FIELD_MAP0) * s->g.size;
    else fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_report_field: bad field");
    copy_d2h(host_out, src, s->g.size, s->stream);
  });
}

int bfm_ctransform(int dim, const int* extents, const double* phi, double* out) {
  return guard([&] {
    HostOp op(dim, extents);
    double* a = op.up(phi, op.g.size);
    double* b = op.up(nullptr, op.g.size);
    op.ws.ctp().run(a, b, nullptr, &op.ws.lc);
    op.down(out, b, op.g.size);
    op.release();
  });
}

int bfm_ctransform_cost(int dim, const int* extents, const double* exponents, const double* phi,
                        double* out) {
  return guard([&] {
    HostOp op(dim, extents);
    bool quadratic = true;
    for (int a = 0; a < dim; ++a) {
      if (!exponents || !(exponents[a] > 1.0))
        fail(BFM_ERR_INVALID_ARGUMENT, "cost exponents must satisfy p > 1");
      quadratic = quadratic && exponents[a] == 2.0;
    }
    double* a = op.up(phi, op.g.size);
    double* b = op.up(nullptr, op.g.size);
    if (quadratic) {
      op.ws.ctp().run(a, b, nullptr, &op.ws.lc);
    } else {
      CtPowerPlan plan;
      plan.init(op.g, exponents);
      plan.run(a, b, nullptr, &op.ws.lc);
    }
    op.down(out, b, op.g.size);
    op.release();
  });
}

int bfm_map_from_conjugate(int dim, const int* extents, const double* u, int /*side*/,
                           double* disp) {
  return guard([&] {
    HostOp op(dim, extents);
    double* a = op.up(u, op.g.size);
    double* m = op.up(nullptr, op.g.d * op.g.size);
    op.ws.pfp().map_only(a, m, nullptr, &op.ws.lc);
    op.down(disp, m, op.g.d * op.g.size);
    op.release();
  });
}

int bfm_pushforward_density(int dim, const int* extents, const double* disp, const double* mu,
                            double* rho) {
  return guard([&] {
    HostOp op(dim, extents);
    double* m = op.up(disp, op.g.d * op.g.size);
    double* a = op.up(mu, op.g.size);
    double* b = op.up(nullptr, op.g.size);
    op.ws.pfp().from_displacement(m, 1.0, a, b, nullptr, &op.ws.lc);
    op.down(rho, b, op.g.size);
    op.release();
  });
}

int bfm_displacement_interpolant(int dim, const int* extents, const double* disp,
                                 const double* mu, double t, double* rho) {
  return guard([&] {
    if (!(t >= 0.0 && t <= 1.0))  // interpolation.hpp:20-21
      fail(BFM_ERR_T_OUT_OF_RANGE, "displacement_interpolant: t must lie in [0, 1]");
    HostOp op(dim, extents);
    double* m = op.up(disp, op.g.d * op.g.size);
    double* a = op.up(mu, op.g.size);
    double* b = op.up(nullptr, op.g.size);
    op.ws.pfp().from_displacement(m, t, a, b, nullptr, &op.ws.lc);
    op.down(rho, b, op.g.size);
    op.release();
  });
}

int bfm_solve_neumann(int dim, const int* extents, const double* rhs, double* out) {
  return guard([&] {
    HostOp op(dim, extents);
    double* a = op.up(rhs, op.g.size);
    double* b = op.up(nullptr, op.g.size);
    op.ws.poisp().solve(a, b, nullptr, &op.ws.lc);
    op.down(out, b, op.g.size);
    op.release();
  });
}

int bfm_integrate(int dim, const int* extents, const double* f, const double* w, double* out) {
  return guard([&] {
    HostOp op(dim, extents);
    double* a = op.up(f, op.g.size);
    if (w) {
      double* b = op.up(w, op.g.size);
      op.ws.redp().dot(a, b, nullptr, nullptr, op.g.size, op.g.vol, 0, nullptr, &op.ws.lc);
    } else {
      op.ws.redp().sum(a, op.g.size, op.g.vol, 0, nullptr, &op.ws.lc);
    }
    double v[1];
    op.ws.redp().fetch(v, 1, nullptr);
    *out = v[0];
    op.release();
  });
}

int bfm_primal_cost(int dim, const int* extents, const double* disp, const double* mu,
                    double* out) {
  return bfm_primal_cost_cost(dim, extents, nullptr, disp, mu, out);
}

int bfm_map_from_conjugate_cost(int dim, const int* extents, const double* exponents,
                                const double* u, int /*side*/, double* disp) {
  return guard([&] {
    HostOp op(dim, extents);
    double* a = op.up(u, op.g.size);
    double* m = op.up(nullptr, op.g.d * op.g.size);
    op.ws.pfp().set_cost(exponents);
    op.ws.pfp().map_only(a, m, nullptr, &op.ws.lc);
    op.down(disp, m, op.g.d * op.g.size);
    op.release();
  });
}

int bfm_primal_cost_cost(int dim, const int* extents, const double* exponents, const double* disp,
                         const double* mu, double* out) {
  return guard([&] {
    HostOp op(dim, extents);
    if (exponents)
      for (int a = 0; a < dim; ++a)
        if (!(exponents[a] > 1.0)) fail(BFM_ERR_INVALID_ARGUMENT, "cost exponents must satisfy p > 1");
    double* m = op.up(disp, op.g.d * op.g.size);
    double* a = op.up(mu, op.g.size);
    op.ws.redp().primal(m, a, op.g.d, op.g.size, op.g.vol, 0, nullptr, &op.ws.lc, exponents);
    double v[1];
    op.ws.redp().fetch(v, 1, nullptr);
    *out = v[0];
    op.release();
  });
}

int bfm_workspace_create(int dim, const int* extents, bfm_workspace** out) {
  return guard([&] {
    *out = nullptr;
    const GridDesc g = checked_grid(dim, extents);
    require_device();
    std::unique_ptr<bfm_workspace> w(new bfm_workspace);
    w->g = g;
    *out = w.release();
  });
}

void bfm_workspace_destroy(bfm_workspace* ws) { delete ws; }

int bfm_ctransform_device(bfm_workspace* ws, const double* d_phi, double* d_out, void* stream) {
  return guard([&] {
    const long before = ws->lc.count;
    ws->ctp().run(d_phi, d_out, static_cast<cudaStream_t>(stream), &ws->lc);
    ws->last_launches = static_cast<int>(ws->lc.count - before);
  });
}

int bfm_workspace_ctransform(bfm_workspace* ws, const double* phi, double* out) {
  return guard([&] {
    if (!ws || !phi || !out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_workspace_ctransform: null argument");
    const cudaStream_t st = ws->io();
    copy_h2d(ws->io_in.p, phi, ws->g.size, st);
    const long before = ws->lc.count;
    ws->ctp().run(ws->io_in.p, ws->io_out.p, st, &ws->lc);
    ws->last_launches = static_cast<int>(ws->lc.count - before);
    copy_d2h(out, ws->io_out.p, ws->g.size, st);
  });
}

int bfm_workspace_solve_neumann(bfm_workspace* ws, const double* rhs, double* out) {
  return guard([&] {
    if (!ws || !rhs || !out) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_workspace_solve_neumann: null argument");
    const cudaStream_t st = ws->io();
    copy_h2d(ws->io_in.p, rhs, ws->g.size, st);
    const long before = ws->lc.count;
    ws->poisp().solve(ws->io_in.p, ws->io_out.p, st, &ws->lc);
    ws->last_launches = static_cast<int>(ws->lc.count - before);
    copy_d2h(out, ws->io_out.p, ws->g.size, st);
  });
}

int bfm_pushforward_residual_device(bfm_workspace* ws, const double* d_u, const double* d_source,
                                    const double* d_target, double* d_r, void* stream) {
  return guard([&] {
    const long before = ws->lc.count;
    ws->pfp().from_potential(d_u, d_source, d_target, d_r, nullptr,
                             static_cast<cudaStream_t>(stream), &ws->lc);
    ws->last_launches = static_cast<int>(ws->lc.count - before);
  });
}

int bfm_solve_neumann_device(bfm_workspace* ws, const double* d_rhs, double* d_out, void* stream) {
  return guard([&] {
    const long before = ws->lc.count;
    ws->poisp().solve(d_rhs, d_out, static_cast<cudaStream_t>(stream), &ws->lc);
    ws->last_launches = static_cast<int>(ws->lc.count - before);
  });
}

int bfm_workspace_last_launches(const bfm_workspace* ws) { return ws->last_launches; }

// ---- multi-GPU slabs -------------------------------------------------------
// ---- fixtures of the paper-case harness (host only) --------------------------
namespace {
struct Shape {  // io.hpp builtin shapes: disc / ball (Euclidean), square / cube
  bool euclid = true;
  int dim = 2;
  double c[3] = {0.0, 0.0, 0.0};
  double r = 0.0;
};

double spec_number(const std::string& tok, const std::string& shape) {
  try {
    size_t pos = 0;
    const double v = std::stod(tok, &pos);
    if (pos != tok.size()) throw std::invalid_argument("");
    return v;
  } catch (const std::exception&) {
    fail(BFM_ERR_INVALID_ARGUMENT, "builtin: malformed number '" + tok + "' in '" + shape + "'");
  }
}

Shape parse_shape(const std::string& tok) {
  const size_t colon = tok.find(':');
  const std::string name = tok.substr(0, colon);
  Shape s;
  if (name == "disc") { s.euclid = true; s.dim = 2; }
  else if (name == "ball") { s.euclid = true; s.dim = 3; }
  else if (name == "square") { s.euclid = false; s.dim = 2; }
  else if (name == "cube") { s.euclid = false; s.dim = 3; }
  else fail(BFM_ERR_INVALID_ARGUMENT, "builtin: unknown shape '" + name + "'");
  std::vector<double> prm;
  if (colon != std::string::npos) {
    std::string rest = tok.substr(colon + 1);
    size_t b = 0;
    while (true) {
      const size_t e = rest.find(',', b);
      prm.push_back(spec_number(rest.substr(b, e == std::string::npos ? std::string::npos : e - b), tok));
      if (e == std::string::npos) break;
      b = e + 1;
    }
  }
  if (static_cast<int>(prm.size()) != s.dim + 1)
    fail(BFM_ERR_INVALID_ARGUMENT, "builtin: '" + name + "' takes " + std::to_string(s.dim + 1) +
                                       " parameters");
  for (int a = 0; a < s.dim; ++a) s.c[a] = prm[a];
  const double extent = prm.back();
  if (!(extent > 0.0)) fail(BFM_ERR_INVALID_ARGUMENT, "builtin: '" + name + "' needs a positive size");
  s.r = s.euclid ? extent : 0.5 * extent;
  return s;
}

bool shape_contains(const Shape& s, const double* x) {
  if (s.euclid) {
    double d2 = 0.0;
    for (int a = 0; a < s.dim; ++a) {
      const double d = x[a] - s.c[a];
      d2 += d * d;
    }
    return d2 <= s.r * s.r;
  }
  for (int a = 0; a < s.dim; ++a)
    if (std::abs(x[a] - s.c[a]) > s.r) return false;
  return true;
}
}  // namespace

int bfm_builtin_density(int dim, const int* extents, const char* spec, double* out) {
  return guard([&] {
    const GridDesc g = checked_grid(dim, extents);
    const std::string sp = spec ? spec : "";
    if (sp.empty()) fail(BFM_ERR_INVALID_ARGUMENT, "builtin: empty spec");
    // '+' separates shapes only when a shape name follows (keeps 1e+2 intact)
    std::vector<Shape> shapes;
    size_t start = 0;
    for (size_t i = 0; i <= sp.size(); ++i) {
      const bool cut = i == sp.size() ||
                       (sp[i] == '+' && i + 1 < sp.size() && std::isalpha(static_cast<unsigned char>(sp[i + 1])));
      if (!cut) continue;
      const std::string tok = sp.substr(start, i - start);
      if (tok.empty()) fail(BFM_ERR_INVALID_ARGUMENT, "builtin: empty union member");
      shapes.push_back(parse_shape(tok));
      if (shapes.back().dim != dim)
        fail(BFM_ERR_INVALID_ARGUMENT, "builtin: shape dimension does not match the grid");
      start = i + 1;
    }
    const int n0 = g.n[0], n1 = dim > 1 ? g.n[1] : 1, n2 = dim > 2 ? g.n[2] : 1;
    long lin = 0;
    for (int i0 = 0; i0 < n0; ++i0)
      for (int i1 = 0; i1 < n1; ++i1)
        for (int i2 = 0; i2 < n2; ++i2, ++lin) {
          const double x[3] = {coord(g.h[0], i0), dim > 1 ? coord(g.h[1], i1) : 0.0,
                               dim > 2 ? coord(g.h[2], i2) : 0.0};
          double v = 0.0;
          for (const Shape& sh : shapes)
            if (shape_contains(sh, x)) {
              v = 1.0;
              break;
            }
          out[lin] = v;
        }
  });
}

int bfm_normalize(int dim, const int* extents, const double* raw, double* out) {
  return guard([&] {
    const GridDesc g = checked_grid(dim, extents);
    Kahan k;  // grid.hpp:151-164
    for (long i = 0; i < g.size; ++i) {
      if (raw[i] < 0.0) fail(BFM_ERR_NEGATIVE_INPUT, "normalize: negative density sample");
      k.add(raw[i]);
    }
    const double mass = k.sum * g.vol;
    if (mass <= 0.0) fail(BFM_ERR_ALL_ZERO_INPUT, "normalize: density has zero total mass");
    for (long i = 0; i < g.size; ++i) out[i] = raw[i] / mass;
  });
}

int bfm_synthetic_densities(int config, int n, unsigned long long seed, double* mu, double* nu) {
  return guard([&] {
    std::string msg;
    const int rc = synthetic_densities(config, n, seed, mu, nu, msg);
    if (rc != BFM_OK) fail(rc, msg);
  });
}

int bfm_validate_inputs(int dim, const int* extents, const double* mu, const double* nu,
                        const bfm_config* cfg) {
  return guard([&] {
    bfm_config c;
    default_config(&c);
    if (cfg) c = *cfg;
    const GridDesc g = checked_grid(dim, extents);
    check_config(c);
    check_density("mu", mu, g);
    check_density("nu", nu, g);
  });
}

int bfm_slab_create(int dim, const int* extents, int row0, int nrows, long col0, int ncols,
                    bfm_slab** out) {
  return guard([&] {
    *out = nullptr;
    const GridDesc g = checked_grid(dim, extents);
    if (dim < 2) fail(BFM_ERR_INVALID_ARGUMENT, "slab: the decomposition needs d >= 2");
    const long M = g.size / g.n[0];
    if (row0 < 0 || nrows < 1 || row0 + nrows > g.n[0])
      fail(BFM_ERR_INVALID_ARGUMENT, "slab: row range outside the grid");
    if (col0 < 0 || ncols < 1 || col0 + ncols > M)
      fail(BFM_ERR_INVALID_ARGUMENT, "slab: column range outside the grid");
    require_device();
    std::unique_ptr<bfm_slab> s(new bfm_slab);
    s->g = g;
    s->row0 = row0;
    s->nrows = nrows;
    s->col0 = col0;
    s->ncols = ncols;
    s->ct_cols.init_slab_cols(g, ncols);
    s->ct_rows.init_slab_rows(g, row0, nrows);
    s->pois_rows.init_slab_rows(g, nrows);
    s->pois_cols.init_slab_cols(g, col0, ncols);
    s->pf.init_slab(g, row0, nrows);
    s->red.init();
    *out = s.release();
  });
}

void bfm_slab_destroy(bfm_slab* s) { delete s; }

int bfm_slab_ct_cols(bfm_slab* s, const double* d_phi_cols, uint32_t* d_chain, double* d_q,
                     void* stream) {
  return slab_op(s, [&] {
    s->ct_cols.run_cols(d_phi_cols, d_chain, d_q, static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_ct_rows(bfm_slab* s, const uint32_t* d_chain, const double* d_q, double* d_out,
                     void* stream) {
  return slab_op(s, [&] {
    s->ct_rows.run_rows(d_chain, d_q, d_out, static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_poisson_rows_forward(bfm_slab* s, const double* d_in, double* d_out, void* stream) {
  return slab_op(s, [&] {
    s->pois_rows.rows_forward(d_in, d_out, static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_poisson_cols(bfm_slab* s, const double* d_in, double* d_out, void* stream) {
  return slab_op(s, [&] {
    s->pois_cols.cols_fused(d_in, d_out, static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_poisson_rows_inverse(bfm_slab* s, double* d_inout, void* stream) {
  return slab_op(s, [&] {
    s->pois_rows.rows_inverse(d_inout, static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_pf_map(bfm_slab* s, const double* d_u_halo, const double* d_source, uint32_t* d_key,
                    double* d_w, uint8_t* d_cmask, double* d_disp, void* stream) {
  return slab_op(s, [&] {
    s->pf.map_records(d_u_halo, d_source, d_key, d_w, d_cmask, d_disp,
                      static_cast<cudaStream_t>(stream), &s->lc);
  });
}

long bfm_slab_pf_num_cells(const bfm_slab* s) { return s ? s->pf.num_cells() : -1; }

int bfm_slab_set_partition(bfm_slab* s, int nranks, const int* row_starts) {
  return slab_op(s, [&] {
    if (nranks < 1 || !row_starts || row_starts[0] != 0 || row_starts[nranks] != s->g.n[0])
      fail(BFM_ERR_INVALID_ARGUMENT, "slab: bad partition");
    for (int q = 0; q < nranks; ++q)
      if (row_starts[q + 1] <= row_starts[q]) fail(BFM_ERR_INVALID_ARGUMENT, "slab: empty rank");
    s->pf.set_partition(nranks, row_starts);
  });
}

int bfm_slab_pf_route(bfm_slab* s, const uint32_t* d_key, const double* d_w, const uint8_t* d_cmask,
                      const double* d_mass, double* d_packed, long* counts, void* stream) {
  return slab_op(s, [&] {
    s->pf.route(d_key, d_w, d_cmask, d_mass, d_packed, counts, static_cast<cudaStream_t>(stream),
                &s->lc);
  });
}

int bfm_slab_pf_unpack(bfm_slab* s, long nrec, const double* d_packed, uint32_t* d_keys,
                       double* d_mass, double* d_w, uint8_t* d_cmask, void* stream) {
  return slab_op(s, [&] {
    s->pf.unpack(d_packed, nrec, d_keys, d_mass, d_w, d_cmask, static_cast<cudaStream_t>(stream),
                 &s->lc);
  });
}

int bfm_slab_pf_gather(bfm_slab* s, long nrec, const uint32_t* d_keys, const double* d_mass,
                       const double* d_w, const uint8_t* d_cmask, const double* d_target,
                       double* d_out, void* stream) {
  return slab_op(s, [&] {
    if (nrec < 0) fail(BFM_ERR_INVALID_ARGUMENT, "slab: negative record count");
    s->pf.gather(nrec, d_keys, d_mass, d_w, d_cmask, d_target, d_out,
                 static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_dot(bfm_slab* s, const double* d_a1, const double* d_b1, const double* d_a2,
                 const double* d_b2, double* out4, void* stream) {
  return slab_op(s, [&] {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    s->red.dot_raw(d_a1, d_b1, d_a2, d_b2, static_cast<long>(s->nrows) * (s->g.size / s->g.n[0]),
                   0, st, &s->lc);
    s->red.fetch(out4, 4, st);
  });
}

int bfm_slab_primal(bfm_slab* s, const double* d_disp, const double* d_mu, double* out2,
                    void* stream) {
  return slab_op(s, [&] {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    s->red.primal_raw(d_disp, d_mu, s->g.d, static_cast<long>(s->nrows) * (s->g.size / s->g.n[0]),
                      0, st, &s->lc);
    s->red.fetch(out2, 2, st);
  });
}

int bfm_slab_axpy(bfm_slab* s, double* d_u, double sigma, const double* d_dir, void* stream) {
  return slab_op(s, [&] {
    axpy(d_u, sigma, d_dir, static_cast<long>(s->nrows) * (s->g.size / s->g.n[0]),
         static_cast<cudaStream_t>(stream), &s->lc);
  });
}

int bfm_slab_last_launches(const bfm_slab* s) { return s ? s->last_launches : 0; }

long bfm_solver_launches(const bfm_solver* s) { return s ? s->ws.lc.count : -1; }

int bfm_debug_pf_tiers(bfm_solver* s, int* out3) {
  return guard([&] { s->ws.pfp().tier_counts(out3); });
}

int bfm_debug_ct_stats(bfm_solver* s, unsigned long long* out8) {
  return guard([&] { s->ws.ctp().stats(out8); });
}

int bfm_debug_ws_ct_stats(bfm_workspace* ws, unsigned long long* out32) {
  return guard([&] { ws->ctp().stats(out32); });
}

int bfm_solver_set_timing(bfm_solver* s, int on) {
  return guard([&] {
    s->resolve_times();
    s->timing = on != 0;
    for (int i = 0; i < BFM_OP_COUNT; ++i) {
      s->op_ms[i] = 0.0;
      s->op_n[i] = 0;
    }
  });
}

int bfm_solver_op_times(bfm_solver* s, double* ms, long* calls) {
  return guard([&] {
    s->resolve_times();
    for (int i = 0; i < BFM_OP_COUNT; ++i) {
      ms[i] = s->op_ms[i];
      calls[i] = s->op_n[i];
    }
  });
}

int bfm_solver_time_steps(bfm_solver* s, int k, double* ms) {
  return guard([&] {
    if (!s || !ms || k < 0) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_time_steps: bad argument");
    s->ensure_probe();
    cudaEvent_t e0, e1;
    BFM_CUDA(cudaEventCreate(&e0));
    BFM_CUDA(cudaEventCreate(&e1));
    BFM_CUDA(cudaEventRecord(e0, s->stream));
    // run()'s loop body: k steps, each followed by the next iteration's probe,
    // in batches with one synchronisation (one per step while timing ops)
    for (int left = k; left > 0;) {
      const int b = s->timing ? 1 : std::min(left, kCtlRing);
      s->steps(b, true, left == b ? e1 : nullptr);
      left -= b;
    }
    if (k == 0) BFM_CUDA(cudaEventRecord(e1, s->stream));
    BFM_CUDA(cudaEventSynchronize(e1));
    float f = 0.0f;
    BFM_CUDA(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = f;
  });
}

int bfm_solver_set_graphs(bfm_solver* s, int on) {
  return guard([&] {
    if (!s) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_set_graphs: null handle");
    s->use_graphs = on != 0;
  });
}

int bfm_solver_debug_force_exact(bfm_solver* s, int iteration, int probe_only) {
  return guard([&] {
    if (!s) fail(BFM_ERR_INVALID_ARGUMENT, "bfm_solver_debug_force_exact: null handle");
    s->force_near_iter = iteration;
    s->force_near_probe = probe_only ? 1 : 0;
  });
}

long bfm_solver_exact_replays(const bfm_solver* s) { return s ? s->exact_replays : -1; }

}  // extern "C"
