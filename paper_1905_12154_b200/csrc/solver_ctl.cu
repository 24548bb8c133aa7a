// Certified scalar decisions of the BFM iteration on the device (see
// solver_ctl.cuh). Reference: solver.hpp:68-76 (update_sigma), :189-207 (stall
// counter), :264-280 (probe), :286-328 (the two step modes).
#include <cmath>

#include "solver_ctl.cuh"

namespace bfmgpu {
namespace {

constexpr double kU4 = 4.0 * 0x1.0p-53;  // 4 units in the last place (relative)

__device__ void mark_near(SolverCtl* c, int stage) {
  if (!(c->flags & kCtlNear)) {
    c->near_stage = stage;
    c->near_iter = c->done;
  }
  c->flags |= kCtlNear;
}

// (x < y) as the reference would evaluate it on its own values x', y' with
// |x - x'| <= bx and |y - y'| <= by. When the outcome cannot be certified the
// NEAR flag is raised (the host replays the iteration with exact scalars).
// Zero bounds mean both sides hold the reference's exact values.
__device__ bool cert_less(double x, double bx, double y, double by, SolverCtl* c, int stage) {
  const double m = 2.0 * (bx + by);
  if (m > 0.0 && !(fabs(x - y) > m)) mark_near(c, stage);
  return x < y;
}

// update_sigma (solver.hpp:68-76) with certified comparisons.
__device__ void update_sigma(SolverCtl* c, double inc, double inc_b, double gn, double gn_b,
                             const CtlConfig& k, int stage) {
  double sigma = c->sigma;
  const double pred = sigma * gn;
  const double pred_b = sigma * gn_b + kU4 * fabs(pred);
  const double t1 = k.beta_1 * pred;
  const double t2 = k.beta_2 * pred;
  if (cert_less(inc, inc_b, t1, k.beta_1 * pred_b + kU4 * fabs(t1), c, stage))
    sigma *= k.alpha_2;
  else if (cert_less(t2, k.beta_2 * pred_b + kU4 * fabs(t2), inc, inc_b, c, stage))
    sigma *= k.alpha_1;
  c->sigma = fmax(sigma, k.sigma_min);
}

// v < ref - 1e-10 (solver.hpp:269-270,298-299,323-324)
__device__ void monotone_check(SolverCtl* c, double v, double v_b, double ref, double ref_b,
                               int stage) {
  const double y = ref - 1e-10;
  if (cert_less(v, v_b, y, ref_b + kU4 * fabs(y), c, stage) && !(c->flags & kCtlBlowup)) {
    c->flags |= kCtlBlowup;
    c->blowup_stage = stage;
    c->blowup_iter = c->done;
  }
}

// step(): stall counter on |dual - prev_dual| < 1e-12 (solver.hpp:199-203)
__device__ void stall_update(SolverCtl* c, double dual, double dual_b, int stage) {
  const double diff = fabs(dual - c->prev_dual);
  const double diff_b = dual_b + c->prev_dual_b + kU4 * diff;
  if (cert_less(diff, diff_b, 1e-12, 0.0, c, stage)) c->stall += 1;
  else c->stall = 0;
  c->prev_dual = dual;
  c->prev_dual_b = dual_b;
}

__device__ void end_step(SolverCtl* c, CtlStats* ring) {
  ring[c->done % kCtlRing] = c->last;
  c->done += 1;
}

__global__ void ctl_decide_kernel(SolverCtl* c, const double* res, int slot, int bslot, int stage,
                                  CtlConfig k, CtlStats* ring) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double v = slot >= 0 ? res[slot] : 0.0;
  const double vb = slot >= 0 ? res[bslot] : 0.0;
  switch (stage) {
    case kStageProbePair:
      monotone_check(c, v, vb, c->last_pair, c->last_pair_b, stage);
      c->last_pair = v;
      c->last_pair_b = vb;
      c->probe_dual = v;
      c->probe_dual_b = vb;
      break;
    case kStageProbeGA:
      c->probe_dual = c->last_pair;
      c->probe_dual_b = c->last_pair_b;
      break;
    case kStageProbeGn:
      c->probe_gn = v;
      c->probe_gn_b = vb;
      break;
    case kStageStepBegin:
      c->last.sigma_first = c->sigma;
      c->last.gn_first = c->probe_gn;
      c->last.residual = sqrt(fmax(c->probe_gn, 0.0));
      c->v_ref = c->probe_dual;
      c->v_ref_b = c->probe_dual_b;
      c->last.sigma_second = 0.0;
      c->last.gn_second = 0.0;
      c->last.inc_second = 0.0;
      break;
    case kStageFirst: {
      const double inc = v - c->v_ref;
      c->last.inc_first = inc;
      update_sigma(c, inc, vb + c->v_ref_b + kU4 * fabs(inc), c->probe_gn, c->probe_gn_b, k, stage);
      c->v_ref = v;
      c->v_ref_b = vb;
      break;
    }
    case kStageV4:
      monotone_check(c, v, vb, c->v_ref, c->v_ref_b, stage);
      c->v_ref = v;
      c->v_ref_b = vb;
      break;
    case kStageGn2:
      c->gn2 = v;
      c->gn2_b = vb;
      c->last.sigma_second = c->sigma;
      c->last.gn_second = v;
      break;
    case kStageV5: {
      const double inc = v - c->v_ref;
      c->last.inc_second = inc;
      update_sigma(c, inc, vb + c->v_ref_b + kU4 * fabs(inc), c->gn2, c->gn2_b, k, stage);
      c->last.dual_value = v;
      c->last_pair = v;
      c->last_pair_b = vb;
      stall_update(c, v, vb, stage);
      end_step(c, ring);
      break;
    }
    case kStageGAv3:
      monotone_check(c, v, vb, c->v_ref, c->v_ref_b, stage);
      c->last.dual_value = v;
      c->last_pair = v;
      c->last_pair_b = vb;
      stall_update(c, v, vb, stage);
      end_step(c, ring);
      break;
    default:
      break;
  }
}

}  // namespace

void ctl_decide(SolverCtl* d_ctl, const double* d_results, int slot, int bound_slot, int stage,
                const CtlConfig& cfg, CtlStats* d_ring, cudaStream_t s, LaunchCounter* lc) {
  ctl_decide_kernel<<<1, 32, 0, s>>>(d_ctl, d_results, slot, bound_slot, stage, cfg, d_ring);
  BFM_LAUNCH_CHECK("ctl_decide_kernel");
  if (lc) lc->add();
}

}  // namespace bfmgpu
