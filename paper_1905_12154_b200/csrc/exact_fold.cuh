// Parallel evaluation of a SEQUENTIAL floating-point fold, bit for bit.
//
// The reference accumulates a target's deposits one at a time in source
// order (pushforward.hpp:141-172: out[node] += w), so the result is
//   rho_0 = +0,  rho_j = RN(rho_{j-1} + w_j),
// with every partial sum rounded. All weights are >= 0 (density times
// barycentric weights), so rho is non-decreasing. While rho stays in one
// binade [2^e, 2^(e+1)) its ulp u = 2^(e-52) is fixed and, writing
// rho = M u (M an integer in [2^52, 2^53)) and w_j / u = a_j + f_j
// (a_j integer, 0 <= f_j < 1, exact: a power-of-two scaling),
//   M_j = M_{j-1} + a_j + [f_j > 1/2] + [f_j == 1/2] * ((M_{j-1} + a_j) & 1)
// (round to nearest, ties to the even multiple of u). Each step is therefore
// a function of the PARITY of M_{j-1} only: a two-state transducer
// p -> (inc(p), (p + inc(p)) & 1). Transducers compose associatively, so a
// parallel prefix scan yields every M_j exactly. The scan is valid up to the
// first element whose exact sum may leave the binade (M_{j-1} + a_j + 1 >=
// 2^53); that element is added with one ordinary IEEE addition (the
// reference's own operation) and the scan restarts in the new binade. The
// number of restarts is bounded by the number of binades rho crosses.
#pragma once

#include <cuda_runtime.h>

namespace bfmgpu {

struct FoldTr {
  long long i0, i1;  // increment of M for start parity 0 / 1
};

__device__ __forceinline__ long long fold_sat(long long v) {
  constexpr long long kSat = 1LL << 60;  // beyond any valid prefix (< 2^53)
  return v > kSat ? kSat : v;
}

// a then b. Element increments are clamped to 2^54, so up to 256 composed
// elements stay below 2^62 without saturation (per-thread and warp scans);
// the cross-warp combination saturates.
__device__ __forceinline__ FoldTr fold_compose(FoldTr a, FoldTr b) {
  FoldTr r;
  r.i0 = a.i0 + ((a.i0 & 1) ? b.i1 : b.i0);
  r.i1 = a.i1 + (((1 + a.i1) & 1) ? b.i1 : b.i0);
  return r;
}
__device__ __forceinline__ FoldTr fold_compose_sat(FoldTr a, FoldTr b) {
  FoldTr r = fold_compose(a, b);
  r.i0 = fold_sat(r.i0);
  r.i1 = fold_sat(r.i1);
  return r;
}

__device__ __forceinline__ long long fold_apply(FoldTr t, long long M) {
  return (M & 1) ? t.i1 : t.i0;
}

// Transducer of one weight w >= 0 at binade exponent e (rho in [2^e, 2^(e+1))).
// a is returned separately (clamped to 2^54) for the crossing test.
__device__ __forceinline__ FoldTr fold_elem(double w, int e, long long& a_out) {
  // w * 2^(52 - e), exact: the power of two is built from its bits (the fold
  // keeps e in [-960, 1020], so 52 - e is a normal exponent); products that
  // underflow only occur for w < 2^-1000 relative, far below 1/2 an ulp
  const double x = w * __longlong_as_double(static_cast<long long>(52 - e + 1023) << 52);
  long long a;
  int cls;  // 0: f < 1/2, 1: f == 1/2, 2: f > 1/2
  if (!(x >= 0.0 && x < 18014398509481984.0)) {  // >= 2^54, negative or NaN: a crossing
    a = 1LL << 54;
    cls = 0;
  } else {
    const double fl = floor(x);
    a = static_cast<long long>(fl);
    const double f = x - fl;  // exact
    cls = f > 0.5 ? 2 : (f == 0.5 ? 1 : 0);
  }
  a_out = a;
  FoldTr t;
  const long long up = cls == 2 ? 1 : 0;
  t.i0 = a + up + (cls == 1 ? (a & 1) : 0);        // parity 0: tie -> even (M + a even iff a even)
  t.i1 = a + up + (cls == 1 ? ((a + 1) & 1) : 0);  // parity 1
  return t;
}

// Group-wide (NT threads, all calling) fold of w[0..K) from rho = +0.
// w may live in global or shared memory. scratch: >= 2 * (NT/32) FoldTr +
// 4 words of shared memory, private to the group. Result valid in all threads.
// NT must be a multiple of 32; `bar` synchronises the group.
template <int NT, int ITEMS, class Sync>
__device__ double exact_fold(const double* w, int K, FoldTr* scratch, int* iscr, Sync bar) {
  static_assert(32 * ITEMS <= 256, "unsaturated per-warp composition range");
  constexpr int kWarps = NT / 32;
  constexpr int kChunk = NT * ITEMS;
  constexpr long long kTop = 1LL << 53;
  const int tid = threadIdx.x % NT;
  const int lane = tid & 31, warp = tid >> 5;
  double rho = 0.0;
  int i0 = 0;
  while (i0 < K) {
    if (!(rho >= 0x1p-960 && rho <= 0x1p1020)) {
      // rho == +0 (leading zeros), tiny, huge, negative or not finite: plain
      // sequential steps, uniform in the group
      if (rho == 0.0) {
        // skip to the first nonzero weight: RN(0 + w) = w
        int first = K;
        for (int j = i0 + tid; j < min(K, i0 + kChunk); j += NT)
          if (w[j] != 0.0) {
            first = j;
            break;
          }
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        if (lane == 0) iscr[warp] = first;
        bar();
        int f = K;
        for (int q = 0; q < kWarps; ++q) f = min(f, iscr[q]);
        bar();
        if (f >= min(K, i0 + kChunk)) {
          i0 = min(K, i0 + kChunk);
        } else {
          rho = w[f];
          i0 = f + 1;
        }
      } else {
        rho = rho + w[i0];
        ++i0;
      }
      continue;
    }
    int e;
    frexp(rho, &e);
    e -= 1;  // rho in [2^e, 2^(e+1))
    const long long M = static_cast<long long>(ldexp(rho, 52 - e));
    // elements [i0, lim): a binade crossing is likely about when the sum has
    // doubled, i.e. after ~i0 more elements of similar size, so the span
    // grows with i0 (restarts then redo little work)
    const int lim = min(K, i0 + min(kChunk, max(NT, i0)));
    // per-thread transducers of ITEMS consecutive elements
    const int base = i0 + tid * ITEMS;
    FoldTr tr[ITEMS];
    long long av[ITEMS];
    FoldTr loc{0, 0};
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int j = base + u;
      if (j < lim) {
        tr[u] = fold_elem(w[j], e, av[u]);
      } else {
        tr[u] = FoldTr{0, 0};
        av[u] = 0;
      }
      loc = fold_compose(loc, tr[u]);
    }
    // exclusive scan of loc across the group (warp shuffles + shared memory)
    FoldTr inc = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      FoldTr o;
      o.i0 = __shfl_up_sync(0xffffffffu, inc.i0, d);
      o.i1 = __shfl_up_sync(0xffffffffu, inc.i1, d);
      if (lane >= d) inc = fold_compose(o, inc);
    }
    if (lane == 31) scratch[warp] = inc;
    FoldTr excl;
    excl.i0 = __shfl_up_sync(0xffffffffu, inc.i0, 1);
    excl.i1 = __shfl_up_sync(0xffffffffu, inc.i1, 1);
    if (lane == 0) excl = FoldTr{0, 0};
    bar();
    FoldTr wpre{0, 0};
    for (int q = 0; q < warp; ++q) wpre = fold_compose_sat(wpre, scratch[q]);
    FoldTr total{0, 0};
    for (int q = 0; q < kWarps; ++q) total = fold_compose_sat(total, scratch[q]);
    excl = fold_compose_sat(wpre, excl);
    // M before each element, and the first element that may leave the binade
    long long Mp = M + fold_apply(excl, M);
    int cross = K;
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int j = base + u;
      if (j < lim && cross == K && Mp + av[u] + 1 >= kTop) cross = j;
      if (cross == K) Mp += fold_apply(tr[u], Mp);
    }
    for (int o = 16; o > 0; o >>= 1) cross = min(cross, __shfl_xor_sync(0xffffffffu, cross, o));
    bar();
    if (lane == 0) iscr[warp] = cross;
    bar();
    int jc = K;
    for (int q = 0; q < kWarps; ++q) jc = min(jc, iscr[q]);
    if (jc == K) {
      rho = ldexp(static_cast<double>(M + fold_apply(total, M)), e - 52);  // exact (< 2^53 u)
      i0 = lim;
    } else {
      // M just before jc: the owner thread publishes it
      const int owner = (jc - i0) / ITEMS;
      if (tid == owner) {
        long long m2 = M + fold_apply(excl, M);
        for (int u = 0; u < ITEMS && base + u < jc; ++u) m2 += fold_apply(tr[u], m2);
        reinterpret_cast<long long*>(scratch)[2 * kWarps] = m2;
      }
      bar();
      const long long Mjc = reinterpret_cast<long long*>(scratch)[2 * kWarps];
      rho = ldexp(static_cast<double>(Mjc), e - 52) + w[jc];  // the reference's own addition
      i0 = jc + 1;
    }
    bar();
  }
  return rho;
}

}  // namespace bfmgpu
