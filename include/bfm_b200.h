/*
 * bfm_b200.h — C ABI of the B200-native back-and-forth (BFM) optimal-transport
 * solver (quadratic cost, float64, cell-centred grids on [0,1]^d, d = 1..3).
 *
 * This is the drop-in boundary for the reference's header-only C++ solver API
 * (/root/reference/proj/include/bfm/<name>.hpp). Every entry point below names the
 * reference interface it replaces. Plain pointers and sizes only; fields are
 * row-major float64 with the last axis fastest (grid.hpp:73-75). Host-pointer
 * entry points copy in/out; *_device entry points take device pointers and a
 * cudaStream_t passed as void*.
 *
 * Errors: every int-returning call returns BFM_OK (0) or a status that maps 1:1
 * onto the reference exception types (errors.hpp:8-42); bfm_last_error() gives
 * the message (thread-local). There is no CPU fallback: without a usable CUDA
 * device every compute call fails with BFM_ERR_CUDA.
 */
#ifndef BFM_B200_H
#define BFM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (errors.hpp:8-42). */
enum {
  BFM_OK = 0,
  BFM_ERR_ERROR = 1,            /* bfm::Error */
  BFM_ERR_INVALID_ARGUMENT = 2, /* bfm::InvalidArgument */
  BFM_ERR_GRID_MISMATCH = 3,    /* bfm::GridMismatch */
  BFM_ERR_NEGATIVE_INPUT = 4,   /* bfm::NegativeInput */
  BFM_ERR_ALL_ZERO_INPUT = 5,   /* bfm::AllZeroInput */
  BFM_ERR_INFEASIBLE_INPUT = 6, /* bfm::InfeasibleInput */
  BFM_ERR_NUMERICAL_BLOWUP = 7, /* bfm::NumericalBlowup */
  BFM_ERR_T_OUT_OF_RANGE = 8,   /* bfm::TOutOfRange */
  BFM_ERR_IO = 9,               /* bfm::IoError */
  BFM_ERR_CUDA = 10             /* device failure (surfaces as bfm::Error) */
};

/* solver.hpp:32 SolverMode */
enum { BFM_MODE_BACK_AND_FORTH = 0, BFM_MODE_GRADIENT_ASCENT = 1 };
/* solver.hpp:34 Termination */
enum {
  BFM_TERM_TOLERANCE_MET = 0,
  BFM_TERM_MAX_ITERATIONS = 1,
  BFM_TERM_DUAL_STALLED = 2,
  BFM_TERM_COST_TARGET_MET = 3
};
/* pushforward.hpp:22 MapSource */
enum { BFM_MAP_MU_SIDE = 0, BFM_MAP_NU_SIDE = 1 };
/* Field selectors for bfm_solver_field / bfm_solver_report_field. */
enum {
  BFM_FIELD_PHI = 0,
  BFM_FIELD_PSI = 1,
  BFM_FIELD_MAP0 = 2, /* displacement along axis 0 (report only) */
  BFM_FIELD_MAP1 = 3,
  BFM_FIELD_MAP2 = 4
};

/* solver.hpp:46-63 SolverConfig. has_exact_cost stands in for std::optional. */
typedef struct bfm_config {
  int mode;
  double tolerance;
  int max_iterations;
  int threads; /* accepted for API parity; the device ignores it */
  double sigma_init;
  double sigma_min;
  double beta_1;
  double beta_2;
  double alpha_1;
  double alpha_2;
  int has_exact_cost;
  double exact_cost;
  double exact_tolerance;
} bfm_config;

/* solver.hpp:78-88 IterationStats */
typedef struct bfm_iteration_stats {
  int iteration;
  double residual;
  double dual_value;
  double sigma_first;
  double sigma_second;
  double grad_norm_sq_first;
  double grad_norm_sq_second;
  double increase_first;
  double increase_second;
} bfm_iteration_stats;

/* solver.hpp:90-101 SolveReport (scalars; fields via bfm_solver_report_field,
 * trace via bfm_solver_trace). */
typedef struct bfm_report {
  int termination;
  int iterations;
  double dual_value;
  double primal_cost;
  double residual;
  double wall_seconds;
} bfm_report;

typedef struct bfm_solver bfm_solver;

/* Fills the reference defaults (solver.hpp:46-63). */
void bfm_config_default(bfm_config* cfg);

/* solver.hpp:68-76 update_sigma. cfg may be NULL (defaults). */
double bfm_update_sigma(double sigma, double increase, double grad_norm_sq,
                        const bfm_config* cfg);

/* solver.hpp:148-167 Solver::Solver — validates exactly as
 * checked_solver_inputs (:132-142) and copies mu, nu (host pointers, N each). */
int bfm_solver_create(int dim, const int* extents, const double* mu, const double* nu,
                      const bfm_config* cfg, bfm_solver** out);
/* Solver(CostModel::power(exponents), mu, nu, cfg) (cost.hpp:24-30; exponents
 * p_a > 1 per axis, NULL = quadratic): the exact c-transform on dense axis-cost
 * tables (extents up to 2048; bitwise the reference's generic path,
 * transforms.hpp:378-386), the map's inverse gradient |v|^(1/(p-1)) correctly
 * rounded (glibc's pow, which the reference calls, is not: about 0.1 % of its
 * results are one ulp off), primal cost with |d|^p / p. */
int bfm_solver_create_cost(int dim, const int* extents, const double* exponents, const double* mu,
                           const double* nu, const bfm_config* cfg, bfm_solver** out);
void bfm_solver_destroy(bfm_solver* s);

int bfm_solver_iteration(const bfm_solver* s);                 /* :169 */
double bfm_solver_sigma(const bfm_solver* s);                  /* :170 */
int bfm_solver_dual_value(bfm_solver* s, double* out);         /* :178-181 */
int bfm_solver_residual(bfm_solver* s, double* out);           /* :183-186 */
int bfm_solver_step(bfm_solver* s, bfm_iteration_stats* out);  /* :189-207 */
int bfm_solver_run(bfm_solver* s, bfm_report* out);            /* :211-226, finish :330-349 */
/* Copies up to cap trace entries (:173); *count receives the trace length. */
int bfm_solver_trace(const bfm_solver* s, bfm_iteration_stats* out, int cap, int* count);
/* Current iterate phi()/psi() (:171-172) into host memory (N doubles). */
int bfm_solver_field(bfm_solver* s, int which, double* host_out);
/* Gauge-fixed report fields of the last run() (:337-344): PHI, PSI, MAP0..2. */
int bfm_solver_report_field(bfm_solver* s, int which, double* host_out);

/* ---- Operators (host pointers) ------------------------------------------ */
/* transforms.hpp:396-432 ctransform (quadratic cost, exactly rounded). */
int bfm_ctransform(int dim, const int* extents, const double* phi, double* out);
/* pushforward.hpp:70-91 map_from_conjugate: disp is d*N (SoA, axis-major). */
/* ctransform for a CostModel::power(exponents) (cost.hpp:24-48; p_a > 1 per
 * axis): the generic path of transforms.hpp:335-427 (all p_a == 2 is the
 * quadratic model and takes the same shortcut as bfm_ctransform). Axis
 * extents up to 2048 for p != 2. */
int bfm_ctransform_cost(int dim, const int* extents, const double* exponents, const double* phi,
                        double* out);
int bfm_map_from_conjugate(int dim, const int* extents, const double* u, int side,
                           double* disp);
/* pushforward.hpp:176-178 pushforward_density (disp d*N, mu N -> rho N). */
int bfm_pushforward_density(int dim, const int* extents, const double* disp,
                            const double* mu, double* rho);
/* interpolation.hpp:18-22 displacement_interpolant: splat at x + t*disp. */
int bfm_displacement_interpolant(int dim, const int* extents, const double* disp,
                                 const double* mu, double t, double* rho);
/* poisson.hpp:87-106 SpectralPlan::solve_neumann. */
int bfm_solve_neumann(int dim, const int* extents, const double* rhs, double* out);
/* grid.hpp:171-183 integrate(f, w) (w == NULL: Lebesgue). */
int bfm_integrate(int dim, const int* extents, const double* f, const double* w,
                  double* out);
/* pushforward.hpp:181-196 primal_cost. */
/* map_from_conjugate / primal_cost with a power cost (exponents per axis). */
int bfm_map_from_conjugate_cost(int dim, const int* extents, const double* exponents,
                                const double* u, int side, double* disp);
int bfm_primal_cost_cost(int dim, const int* extents, const double* exponents, const double* disp,
                         const double* mu, double* out);
int bfm_primal_cost(int dim, const int* extents, const double* disp, const double* mu,
                    double* out);

/* ---- Operators on device memory (C5 sweep, benches) ---------------------- */
typedef struct bfm_workspace bfm_workspace;
int bfm_workspace_create(int dim, const int* extents, bfm_workspace** out);
void bfm_workspace_destroy(bfm_workspace* ws);
int bfm_ctransform_device(bfm_workspace* ws, const double* d_phi, double* d_out,
                          void* stream);
/* Fused map_from_conjugate + pushforward_density + residual (solver.hpp:249-253):
 * d_r = d_target - T#d_source with T from d_u (side selects mu/nu semantics). */
int bfm_pushforward_residual_device(bfm_workspace* ws, const double* d_u,
                                    const double* d_source, const double* d_target,
                                    double* d_r, void* stream);
int bfm_solve_neumann_device(bfm_workspace* ws, const double* d_rhs, double* d_out,
                             void* stream);
/* Number of device kernels the last *_device call on ws enqueued. */
int bfm_workspace_last_launches(const bfm_workspace* ws);
/* Host-pointer operator calls on a workspace: the plans (and their device
 * tables) are built once and reused across calls — the reference's
 * TransformWorkspace / SpectralPlan reuse (transforms.hpp:231-283,
 * poisson.hpp:42-73). N doubles in, N doubles out. */
int bfm_workspace_ctransform(bfm_workspace* ws, const double* phi, double* out); /* transforms.hpp:396 */
int bfm_workspace_solve_neumann(bfm_workspace* ws, const double* rhs, double* out); /* poisson.hpp:87 */

/* ---- Multi-GPU building blocks (one process per GPU) ---------
 * The reference has no distributed mode; these are the rank-local halves of
 * its operators under an axis-0 slab decomposition, driven by
 * paper_1905_12154_b200/dist.py over torch.distributed (NCCL). A rank owns
 * rows [row0, row0+nrows) of the grid and, for axis-0 work, the flattened
 * columns [col0, col0+ncols) of the n1*n2 non-axis-0 index. All pointers are
 * device pointers; `stream` is a cudaStream_t. Results equal the single-GPU
 * operators bit for bit once the exchanges in dist.py are applied. */
/* Host-only fixtures of the paper-case harness (benchmark.hpp:27-43):
 * indicator of a '+'-union of builtin shapes "disc:x,y,r", "ball:x,y,z,r",
 * "square:x,y,side", "cube:x,y,z,side" (io.hpp:360-476, not normalised), and
 * normalisation to unit mass with the Kahan mass of grid.hpp:151-164. */
int bfm_builtin_density(int dim, const int* extents, const char* spec, double* out);
int bfm_normalize(int dim, const int* extents, const double* raw, double* out);
/* Host-only: the seeded synthetic densities of BASELINE.json configs C1-C4
 * (SURVEY 8(d) shared generator: std::mt19937_64(seed), u = (rng()>>11)*2^-53,
 * unit-peak Gaussians, closed indicators, Kahan normalisation). config 1..3
 * fill n*n samples per density, config 4 n*n*n. Default seeds: C1 1, C2 2,
 * C3 3, C4 4. The reference has no generator (its fixtures are builtin
 * shapes, io.hpp:352-476); this is the input side of the benchmark harness. */
int bfm_synthetic_densities(int config, int n, unsigned long long seed, double* mu, double* nu);

typedef struct bfm_slab bfm_slab;
/* Host-only: the validation of bfm_solver_create (solver.hpp:105-142,148-167)
 * without creating a solver (every rank of the multi-GPU driver runs it). */
int bfm_validate_inputs(int dim, const int* extents, const double* mu, const double* nu,
                        const bfm_config* cfg);
int bfm_slab_create(int dim, const int* extents, int row0, int nrows, long col0, int ncols,
                    bfm_slab** out);
void bfm_slab_destroy(bfm_slab* s);
/* c-transform (transforms.hpp:396-432): pass 0 on the (n0 x ncols) column
 * slab -> argmin chain j0* (uint32) and Q = phi(j0*, column); passes 1..d-1
 * on the row slab from (chain, Q) of its rows -> phi^c. */
int bfm_slab_ct_cols(bfm_slab* s, const double* d_phi_cols, uint32_t* d_chain, double* d_q,
                     void* stream);
int bfm_slab_ct_rows(bfm_slab* s, const uint32_t* d_chain, const double* d_q, double* d_out,
                     void* stream);
/* solve_neumann (poisson.hpp:87-106): DCT-II along axes d-1..1 (rows), the
 * fused axis-0 [DCT-II, divide, DCT-III] (columns), DCT-III along 1..d-1. */
int bfm_slab_poisson_rows_forward(bfm_slab* s, const double* d_in, double* d_out, void* stream);
int bfm_slab_poisson_cols(bfm_slab* s, const double* d_in, double* d_out, void* stream);
int bfm_slab_poisson_rows_inverse(bfm_slab* s, double* d_inout, void* stream);
/* pushforward (pushforward.hpp:70-91,141-172): deposit records of the rank's
 * sources from u with one halo row above and below ((nrows+2) rows): global
 * lo-corner cell (massless: global N), upper weights (d x nrows*M SoA), clamp
 * mask, optional displacement (d x nrows*M). Gather: records from all ranks
 * in global source order, keys relative to the rank's cells (global cell -
 * (row0-1)*M; sentinel bfm_slab_pf_num_cells) -> target - rho (or rho). */
int bfm_slab_pf_map(bfm_slab* s, const double* d_u_halo, const double* d_source, uint32_t* d_key,
                    double* d_w, uint8_t* d_cmask, double* d_disp, void* stream);
long bfm_slab_pf_num_cells(const bfm_slab* s);
/* Routing of the map's records to the owners of the target rows they reach
 * (row_starts[0..nranks] partitions axis 0): packed (3 + d doubles per
 * record: key relative to the destination's cells as raw bits, mass, d
 * weights, clamp mask; capacity 2 * nrows*M records) grouped by destination
 * rank, each group in source order; counts[q] records for rank q. Unpack
 * turns the received concatenation into bfm_slab_pf_gather's inputs. */
int bfm_slab_set_partition(bfm_slab* s, int nranks, const int* row_starts);
int bfm_slab_pf_route(bfm_slab* s, const uint32_t* d_key, const double* d_w, const uint8_t* d_cmask,
                      const double* d_mass, double* d_packed, long* counts, void* stream);
int bfm_slab_pf_unpack(bfm_slab* s, long nrec, const double* d_packed, uint32_t* d_keys,
                       double* d_mass, double* d_w, uint8_t* d_cmask, void* stream);
int bfm_slab_pf_gather(bfm_slab* s, long nrec, const uint32_t* d_keys, const double* d_mass,
                       const double* d_w, const uint8_t* d_cmask, const double* d_target,
                       double* d_out, void* stream);
/* Scalars: unscaled double-double partial sums of the rank's rows
 * (out4 = hi1, lo1, hi2, lo2 of sum a1*b1, sum a2*b2; a2/b2 may be null),
 * combined in rank order by the driver; primal (pushforward.hpp:181-196). */
int bfm_slab_dot(bfm_slab* s, const double* d_a1, const double* d_b1, const double* d_a2,
                 const double* d_b2, double* out4, void* stream);
int bfm_slab_primal(bfm_slab* s, const double* d_disp, const double* d_mu, double* out2,
                    void* stream);
int bfm_slab_axpy(bfm_slab* s, double* d_u, double sigma, const double* d_dir, void* stream);
int bfm_slab_last_launches(const bfm_slab* s);

/* ---- Multi-GPU solver with a C++ host (one process per GPU) -----------------
 * bfm::Solver's loop (solver.hpp:146-368) over an axis-0 slab decomposition:
 * the rank-local kernels above plus NCCL grouped send/recv exchanges issued
 * by the library (libnccl.so.2, loaded at first use) on the solver's stream.
 * Results equal the single-GPU solver bit for bit. The caller distributes the
 * 128-byte NCCL unique id (from rank 0's bfm_nccl_unique_id) however it
 * likes (MPI, torch.distributed, a file). bfm_comm_create_local_group makes
 * nranks handles whose ranks run as threads of this process on one device
 * (host-synchronised exchanges; tests on a single GPU). Errors: the status
 * codes above, message from bfm_dist_last_error(). */
typedef struct bfm_comm bfm_comm;
typedef struct bfm_dist_solver bfm_dist_solver;
int bfm_nccl_unique_id(unsigned char* out128);
int bfm_comm_create_nccl(const unsigned char* id128, int rank, int nranks, bfm_comm** out);
int bfm_comm_create_local_group(int nranks, bfm_comm** out /* nranks handles */);
void bfm_comm_destroy(bfm_comm* c);
/* mu_rows, nu_rows: this rank's rows [row0, row0 + nrows) of the densities
 * (rows split as evenly as possible, lower ranks first; host pointers). The
 * caller validates the full densities (bfm_validate_inputs) as every rank of
 * the reference-order check must agree. */
int bfm_dist_solver_create(bfm_comm* comm, int dim, const int* extents, const double* mu_rows,
                           const double* nu_rows, const bfm_config* cfg, bfm_dist_solver** out);
void bfm_dist_solver_destroy(bfm_dist_solver* s);
int bfm_dist_solver_rows(const bfm_dist_solver* s, int* row0, int* nrows);
int bfm_dist_solver_step(bfm_dist_solver* s, bfm_iteration_stats* out);        /* :189-207 */
int bfm_dist_solver_probe(bfm_dist_solver* s, double* dual, double* residual); /* :178-186 */
int bfm_dist_solver_run(bfm_dist_solver* s, bfm_report* out);                  /* :211-226 */
int bfm_dist_solver_field(bfm_dist_solver* s, int which, double* host_rows);   /* this rank's rows */
/* gauge-fixed report fields of the whole grid (every rank holds them) */
int bfm_dist_solver_report_field(bfm_dist_solver* s, int which, double* host_full);
int bfm_dist_solver_trace(const bfm_dist_solver* s, bfm_iteration_stats* out, int cap, int* count);
int bfm_dist_solver_iteration(const bfm_dist_solver* s);
/* bench helper: k steps + trailing probes between CUDA events on the
 * solver's stream (device milliseconds) */
int bfm_dist_solver_time_steps(bfm_dist_solver* s, int k, double* ms);
double bfm_dist_solver_sigma(const bfm_dist_solver* s);
const char* bfm_dist_last_error(void);

/* Total device kernels the solver has enqueued so far (launch evidence). */
long bfm_solver_launches(const bfm_solver* s);

/* Bench helper: runs k step()s (plus the trailing probe each step() of the
 * reference also pays, solver.hpp:213) between two CUDA events recorded on the
 * solver's stream; *ms receives the device-timed duration. */
int bfm_solver_time_steps(bfm_solver* s, int k, double* ms);

/* Iterations run as captured CUDA graphs (one launch per step + probe, a
 * single host synchronisation per batch of steps); on by default, env
 * BFM_NO_GRAPHS=1 or this call switches to eager launches (same kernels,
 * same bits). */
int bfm_solver_set_graphs(bfm_solver* s, int on);
/* Test hook: treat iteration `iteration` (1-based) as a near tie — in its
 * step, or only in its probe when probe_only — so the solver replays it with
 * every scalar in the reference's sequential Kahan order (the rare path taken
 * when a sigma / blow-up / stall / stopping decision cannot be certified). */
int bfm_solver_debug_force_exact(bfm_solver* s, int iteration, int probe_only);
/* Number of exact replays so far (near ties met, or forced by the hook). */
long bfm_solver_exact_replays(const bfm_solver* s);

/* Bench helper: per-operator device time (CUDA events on the solver stream
 * around each operator call) accumulated while timing is on; switching it
 * (on or off) resets the totals. ms[op] / calls[op] for op in
 * BFM_OP_CTRANSFORM .. BFM_OP_REDUCE (reduce = pair values, gn, axpy). */
enum { BFM_OP_CTRANSFORM = 0, BFM_OP_PUSHFORWARD = 1, BFM_OP_POISSON = 2, BFM_OP_REDUCE = 3,
       BFM_OP_COUNT = 4 };
int bfm_solver_set_timing(bfm_solver* s, int on);
int bfm_solver_op_times(bfm_solver* s, double* ms, long* calls);

/* Diagnostics: targets in the warp / CTA / huge gather tiers of the solver's
 * last pushforward. */
int bfm_debug_pf_tiers(bfm_solver* s, int* out3);
/* Test hook: c-transform diagnostic counters (needs env BFM_CT_STATS=1). */
int bfm_debug_ct_stats(bfm_solver* s, unsigned long long* out8);
int bfm_debug_ws_ct_stats(bfm_workspace* ws, unsigned long long* out32);
/* Test hook: device evaluation of the exact round-down of `count` sums of m
 * doubles each (terms row-major). Used by the parity tests only. */
int bfm_debug_round_down(const double* terms, int m, int count, double* out);
/* Test hook: the pushforward's parallel evaluation of the sequential fold
 * rho = ((0 + w_0) + w_1) + ... of each sequence w[offsets[i] .. offsets[i+1])
 * (exact_fold.cuh), by a 512-thread CTA (mode 0) or one warp (mode 1). */
int bfm_debug_fold(const double* w, const long* offsets, int nseq, int mode, double* out);

/* Test hook: correctly rounded x^y (pow_dd.h) on the host or the device. */
int bfm_debug_pow(const double* x, const double* y, int n, int on_device, double* out);

const char* bfm_last_error(void);
/* Selects the CUDA device for subsequent calls on this thread (one process
 * per GPU: pass LOCAL_RANK). */
int bfm_set_device(int device);
/* 1 if a CUDA device is usable, else 0 (never throws). */
int bfm_device_available(void);

#ifdef __cplusplus
}
#endif
#endif /* BFM_B200_H */
