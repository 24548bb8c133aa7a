// Device-resident scalar state of the BFM solver and its decision kernels.
//
// The reference keeps sigma, the last pair value, the probe and the stall
// counter on the host and decides after every reduction
// (solver.hpp:68-76,189-207,264-310). Here those decisions run in one-thread
// kernels between the field kernels, so a whole iteration is enqueued (and
// captured as a CUDA graph) with a single host synchronisation at its end.
//
// Every decision is CERTIFIED: our reductions are double-double tree sums
// while the reference sums sequentially with Kahan compensation
// (grid.hpp:124-133), so each scalar carries a rigorous bound on its distance
// from the reference's value (reduce.cu red_final_kernel). A comparison whose
// two sides are closer than their combined bounds sets NEAR; the host then
// replays that iteration with every scalar recomputed in the reference's
// exact Kahan order (capi.cu, bfm_solver::replay_exact), so sigma, the
// blow-up checks and the stall counter always follow the reference's branch.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace bfmgpu {

enum CtlFlag { kCtlNear = 1, kCtlBlowup = 2 };

// Decision stages (one launch each).
enum CtlStage {
  kStageProbePair = 0,  // BAF probe: v = pair(phi, phi^c); monotone check vs last pair
  kStageProbeGA = 1,    // GA probe: probe dual = last pair
  kStageProbeGn = 2,    // probe gn (mu side)
  kStageStepBegin = 3,  // stats: sigma_first, gn_first, residual
  kStageFirst = 4,      // BAF v3 / GA v2: increase_first, sigma update
  kStageV4 = 5,         // BAF v4: monotone check vs v3
  kStageGn2 = 6,        // BAF gn2: sigma_second, gn_second
  kStageV5 = 7,         // BAF v5: increase_second, sigma update, dual, stall
  kStageGAv3 = 8        // GA v3: monotone check vs v2, dual, stall
};

// Stats of one step (bfm_iteration_stats without the iteration number).
struct CtlStats {
  double residual, dual_value, sigma_first, sigma_second, gn_first, gn_second, inc_first,
      inc_second;
};

// Steps per batch: the device writes each step's stats to ring[done % kCtlRing].
constexpr int kCtlRing = 1024;

struct SolverCtl {
  // solver state (solver.hpp:349-368); *_b = bound on |ours - reference|
  double sigma;
  double last_pair, last_pair_b;
  double prev_dual, prev_dual_b;
  double probe_dual, probe_dual_b;
  double probe_gn, probe_gn_b;
  double v_ref, v_ref_b;  // the value the next increase / monotone check is measured from
  double gn2, gn2_b;
  int stall;
  int done;  // completed steps
  int flags;
  int near_stage, near_iter;      // first near tie: stage and `done` at the time
  int blowup_stage, blowup_iter;  // first certified blow-up
  int pad;
  CtlStats last;  // the step in flight / last completed
};

struct CtlConfig {
  double beta_1, beta_2, alpha_1, alpha_2, sigma_min;
};

// One decision: reads results[slot] and its bound results[bound_slot].
void ctl_decide(SolverCtl* d_ctl, const double* d_results, int slot, int bound_slot, int stage,
                const CtlConfig& cfg, CtlStats* d_ring, cudaStream_t s, LaunchCounter* lc);

}  // namespace bfmgpu
