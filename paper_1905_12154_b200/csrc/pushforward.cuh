// Transport map + density pushforward on sm_100a (reference pushforward.hpp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "radix_sort.cuh"

namespace bfmgpu {

class PushforwardPlan {
 public:
  PushforwardPlan() = default;
  ~PushforwardPlan();
  PushforwardPlan(const PushforwardPlan&) = delete;
  PushforwardPlan& operator=(const PushforwardPlan&) = delete;

  void init(const GridDesc& g);
  // Multi-GPU row slab: sources and targets are rows
  // [row0, row0 + nrows) of `global`; u arrays carry one halo row above and
  // below; deposit records arrive from every rank (see map_records/gather).
  void init_slab(const GridDesc& global, int row0, int nrows);

  // out = target - T#source with T = x - grad(u) (map_from_conjugate,
  // pushforward.hpp:70-91) — or, if target == nullptr, out = T#source.
  // disp_out (d*N, may be null) receives the displacement field.
  void from_potential(const double* d_u, const double* d_source, const double* d_target,
                      double* d_out, double* d_disp_out, cudaStream_t stream, LaunchCounter* lc);
  // rho = splat of source at x + scale*disp (pushforward.hpp:141-172).
  void from_displacement(const double* d_disp, double scale, const double* d_source,
                         double* d_rho, cudaStream_t stream, LaunchCounter* lc);
  // Map only (displacements), no splat.
  void map_only(const double* d_u, double* d_disp, cudaStream_t stream, LaunchCounter* lc);
  // Deposit records of this plan's sources: global lo-corner cell (sentinel:
  // global N for massless sources), upper weights w (d x N SoA), clamp mask.
  void map_records(const double* d_u, const double* d_source, uint32_t* d_key, double* d_w,
                   uint8_t* d_cmask, double* d_disp_out, cudaStream_t stream, LaunchCounter* lc);
  // out = target - rho (or rho) for this plan's targets from nrec records in
  // global source order: keys are cells of this plan (slab: global cell minus
  // (row0 - 1) * row stride; sentinel num_cells()), mass, w (d x nrec), mask.
  void gather(long nrec, const uint32_t* d_keys, const double* d_mass, const double* d_w,
              const uint8_t* d_cmask, const double* d_target, double* d_out, cudaStream_t stream,
              LaunchCounter* lc);
  long num_cells() const { return ncells_; }
  // Separable power cost (cost.hpp:58-68): per axis p_a > 1; the map's inverse
  // gradient is then sign(v) |v|^(1/(p_a - 1)) (capped at sqrt d); p_a == 2
  // keeps the quadratic |v|. nullptr restores the quadratic cost.
  void set_cost(const double* exponents);
  // diagnostics: targets in the warp / CTA / huge tiers of the last gather
  void tier_counts(int* out3) const {
    int v[6] = {};
    BFM_CUDA(cudaMemcpy(v, nheavy_, sizeof(v), cudaMemcpyDeviceToHost));
    out3[0] = v[0];
    out3[1] = v[4];
    out3[2] = v[1];
  }
  // Multi-GPU routing of this slab's deposit records (map_records output) to
  // the owners of the target rows they reach: row_starts[0..P] partition
  // axis 0. packed receives, per destination in rank order and within it in
  // source order, (3 + d) doubles per record: key relative to the
  // destination's cells (raw bits), mass, d weights, clamp mask; counts[q]
  // the number of records for rank q. Capacity: 2 * nodes records.
  void set_partition(int P, const int* row_starts);
  void route(const uint32_t* d_key, const double* d_w, const uint8_t* d_cmask,
             const double* d_mass, double* d_packed, long* counts, cudaStream_t stream,
             LaunchCounter* lc);
  // received packed records -> gather inputs (keys, mass, w SoA, mask)
  void unpack(const double* d_packed, long nrec, uint32_t* d_keys, double* d_mass, double* d_w,
              uint8_t* d_cmask, cudaStream_t stream, LaunchCounter* lc);

 private:
  void setup(const GridDesc& loc, const GridDesc& global, int row0, bool slab);
  void ensure_records(long nrec);
  double iexp_[3] = {0.0, 0.0, 0.0};  // 1/(p_a - 1) per axis, 0 = quadratic axis
  GridDesc g_;    // this plan's nodes
  GridDesc gg_;   // problem grid
  int row_off_ = 0;
  long cell_shift_ = 0;
  long ncells_ = 0;
  long rec_cap_ = 0;
  int nranks_ = 0;
  int* row0_ = nullptr;      // [P + 1] partition (routing)
  int* bcount_ = nullptr;    // [P * blocks + 1] routing counts / offsets
  int* hcounts_ = nullptr;   // pinned
  uint32_t* key_ = nullptr;  // [N] lo-corner cell of each source (N = no mass)
  uint8_t* cmask_ = nullptr; // [N] axes on which the source is clamped (lo == hi)
  double* w_ = nullptr;      // [d*N] upper-node weight per axis
  int* off_ = nullptr;       // [N+1] first sorted position of each cell
  int* end_ = nullptr;       // [N+1] one past the last
  int* heavy_ = nullptr;     // [N] medium targets (bottom) and huge targets (top)
  unsigned long long* nheavy_ = nullptr;  // [0] heavy count, [1] buffer fill
  double* hbuf_ = nullptr;   // [2^d * N] merged heavy deposits
  double* wts_ = nullptr;    // [2^d][N] deposit weights per corner, in sorted order (corner-major)
  RadixSorter sorter_;
  int key_bits_ = 0;
  int med_blocks_ = 1;       // medium-gather CTAs (each warp owns a kMedium slice of hbuf_)
  int large_blocks_ = 1;     // large-gather CTAs (each owns a kLarge slice of hbuf_)
  int* large_ = nullptr;     // [N] targets of the CTA-per-target tier
  long long* lmeta_ = nullptr;  // per large target: hbuf offset << 13 | K
  long lmeta_cap_ = 0;
};

}  // namespace bfmgpu
