// Exact quadratic c-transform on sm_100a (reference transforms.hpp:396-432).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace bfmgpu {

struct CtAxis {
  int n;
  long stride;
  double h;
  int dyadic;          // 1: g(k,j) = 0.5 (x_k - y_j)^2 is an exact double
  const double4* G;    // else: [n*n] exact limbs (hi, mid, lo, 0) of hs(x_k)+hs(y_j)-x_k*y_j
  // non-dyadic axes with n <= 512: the same values as exact fixed-point
  // integers g * 2^124 (every coordinate is then a multiple of 2^-62)
  const __int128* GF;
};

struct CtPass {
  int d;
  int a;      // axis of this pass
  int last;   // 1 on the final pass (writes psi)
  long nlines;
  int tpl, C, lpc;
  int strided;
  CtAxis ax[3];
  const double* phi;
  const uint32_t* state_in;  // argmin chain of previous passes (a > 0)
  uint32_t* state_out;       // non-last passes
  double* out;               // last pass
  // global row of local row 0 (multi-GPU row slab), else 0
  int k0_off;
  // phi holds phi(chain*, y) at every node y (the previous pass's q_out):
  // candidates read their own node instead of gathering along the chain
  int pregathered;
  double* q_out;  // non-last passes: phi at the winner's chain, per node
  // shared-memory carve-up (bytes, per line)
  int off_fv, off_chain, off_hidx, off_H, off_flag, off_list, off_lohi, off_scal, line_bytes;
  int fixed;  // non-dyadic kernel: every non-dyadic axis has a fixed-point table
  // pass 0 on the transposed potential (2-D dyadic grids): its lines are the
  // rows of phi^T, contiguous like the last pass's
  int t0;
  // small line state (contiguous dyadic passes of long lines): q and the chain
  // are read from global memory where needed instead of being staged, so four
  // lines fit one SM's shared memory
  int qglobal;
  // statistics (device counters, may be null): lines that needed exact resolution
  unsigned long long* slow_queries;
  unsigned long long* stats;  // optional diagnostics (env BFM_CT_STATS=1)
};

class CtPlan {
 public:
  CtPlan() = default;
  ~CtPlan();
  CtPlan(const CtPlan&) = delete;
  CtPlan& operator=(const CtPlan&) = delete;

  void init(const GridDesc& g);
  // out = phi^c (exactly rounded toward -inf). phi and out are device pointers
  // (may not alias). Enqueues g.d kernels on stream.
  // before_last (optional): an event the last pass waits for — the pass that
  // writes d_out — so readers of d_out on another stream can overlap the
  // earlier passes.
  // concave_input: a hint that phi is itself a c-transform (exactly collinear
  // runs); picks the staged form of the long contiguous passes over the
  // small-state one (see setup). The result does not depend on it.
  void run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc,
           cudaEvent_t before_last = nullptr, bool concave_input = false);

  // Multi-GPU slab decomposition along axis 0. Column slab:
  // the (n0 x ncols) block of the flattened non-axis-0 columns; pass 0 writes
  // the argmin j0* and Q = phi(j0*, column) per node. Row slab: rows
  // [row0, row0 + nrows) of the global grid; passes 1..d-1 read the chain and
  // Q of their own rows (after the transpose) and write phi^c.
  void init_slab_cols(const GridDesc& global, int ncols);
  void init_slab_rows(const GridDesc& global, int row0, int nrows);
  void run_cols(const double* d_phi_cols, uint32_t* d_chain, double* d_q, cudaStream_t stream,
                LaunchCounter* lc);
  void run_rows(const uint32_t* d_chain0, const double* d_q, double* d_out, cudaStream_t stream,
                LaunchCounter* lc);
  unsigned long long slow_query_count();  // diagnostic (synchronous)
  void stats(unsigned long long* out8);     // diagnostic counters (synchronous)
  const GridDesc& grid() const { return g_; }

 private:
  void setup(const GridDesc& loc, const GridDesc& global, int pb, int pe, int k0_off,
             bool pregathered, bool virtual_cols);
  void launch(const CtPass& P, cudaStream_t stream, LaunchCounter* lc);
  int pb_ = 0, pe_ = 0, k0_off_ = 0;
  GridDesc g_;
  CtAxis ax_[3] = {};
  double4* tables_[3] = {nullptr, nullptr, nullptr};
  __int128* ftables_[3] = {nullptr, nullptr, nullptr};
  uint32_t* state_[2] = {nullptr, nullptr};
  double* qbuf_[2] = {nullptr, nullptr};  // phi at the argmin chain, per node (pass outputs)
  unsigned long long* slow_ = nullptr;
  unsigned long long* stats_ = nullptr;
  CtPass pass_[3] = {};
  // transposed pass 0 (2-D dyadic single-GPU plans): phi^T, and pass 0's
  // chain and q in transposed layout before they are transposed back
  CtPass pass0t_ = {};
  bool t0_ = false;
  // small-state forms of the last pass and of the transposed pass 0
  CtPass passq_ = {};
  CtPass pass0tq_ = {};
  bool have_q_ = false, have_qt_ = false;
  bool pass0_needs_t0_ = false;  // pass 0's lines are too long for the staged form: transposed small-state pass only
  bool q_only_ = false;  // the last pass's line is too long for the staged form (pass_[d-1] is the small-state one)
  int qg_mode_ = 2;
  int qg_mix_ = 0;  // hinted calls: passes that still take the small-state form (bit 0: pass 0, bit 1: last)
  double* phit_ = nullptr;
  uint32_t* statet_ = nullptr;
  double* qt_ = nullptr;
  bool ready_ = false;
  bool dyadic_ = false;
};

}  // namespace bfmgpu
