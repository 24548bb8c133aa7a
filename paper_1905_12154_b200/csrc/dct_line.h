// Per-line DCT-II / DCT-III arithmetic shared by the sm_100a Poisson kernels
// and by the oracle's FFTW-subset shim (oracle/fftw3.h).
//
// The reference solves the Neumann Poisson problem with FFTW's REDFT10
// (DCT-II, Y_k = 2 sum_j x_j cos(pi k (2j+1) / 2n)) and REDFT01 (DCT-III,
// Y_k = x_0 + 2 sum_{j>=1} x_j cos(pi j (2k+1) / 2n)), see
// /root/reference/proj/include/bfm/poisson.hpp:45-71,91,104. FFTW is not
// available in this image, so both the GPU and the CPU oracle use THIS
// algorithm. Every output element is produced by the same sequence of IEEE
// operations on both sides (GPU built with -fmad=false, CPU with
// -ffp-contract=off), so the Poisson step is bitwise identical between the
// device kernels and the CPU reference build. The GPU only changes which
// thread evaluates which butterfly.
//
// Algorithm (n even, n/2 = 2^a 3^b): Makhoul's reordering into a real
// sequence v, packed into n/2 complex points, an in-place decimation-in-
// frequency FFT of length m = n/2 with radix 4/2/3 stages (output in
// mixed-radix digit-reversed order), then the real-FFT unpack fused with
// the DCT post-twiddle. DCT-III runs the same steps in reverse. Other n use
// a direct O(n^2) sum against a host-computed cosine table.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define BFM_HD __host__ __device__ __forceinline__
#else
#define BFM_HD inline
#endif

namespace bfmdct {

struct cplx {
  double re, im;
};

enum LineKind : int { kFft = 0, kNaive = 1 };
constexpr int kMaxStages = 40;

// Plan for one axis. Table pointers are host or device pointers depending on
// who executes the line; the values are identical (built by build_tables).
struct LinePlan {
  int n = 0;
  int kind = kNaive;
  int m = 0;            // n/2 (FFT kind)
  int nstages = 0;
  int radix[kMaxStages] = {};
  int span[kMaxStages] = {};  // sub-transform length entering stage s
  const cplx* wm = nullptr;     // [m]   e^{-2 pi i j / m}
  const int* rev = nullptr;     // [m]   frequency k -> storage slot after DIF
  const cplx* cs = nullptr;     // [m+1] (cos(pi k / 2n), sin(pi k / 2n))
  const cplx* wn = nullptr;     // [m+1] (cos(2 pi k / n), sin(2 pi k / n))
  const double* cosmat = nullptr;  // [n*n] cos(pi k (2j+1) / 2n) at k*n+j
};

// Table reads (twiddles, digit reversal): read-only for a whole launch, so
// the device reads them through the non-coherent path (same values).
BFM_HD cplx tab_c(const cplx* t, int i) {
#if defined(__CUDA_ARCH__)
  const double2 v = __ldg(reinterpret_cast<const double2*>(t) + i);
  return cplx{v.x, v.y};
#else
  return t[i];
#endif
}
BFM_HD int tab_i(const int* t, int i) {
#if defined(__CUDA_ARCH__)
  return __ldg(t + i);
#else
  return t[i];
#endif
}

BFM_HD cplx cmul(cplx a, cplx b) {
  cplx r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}
BFM_HD cplx cmulc(cplx a, cplx b) {  // a * conj(b)
  cplx r;
  r.re = a.re * b.re + a.im * b.im;
  r.im = a.im * b.re - a.re * b.im;
  return r;
}
BFM_HD cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
BFM_HD cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }

// Number of butterflies in stage s.
BFM_HD int stage_butterflies(const LinePlan& p, int s) { return p.m / p.radix[s]; }

// Arithmetic of one DIF butterfly of radix r on x[0..r) (in place), twiddle
// exponent tw for output digit 1. Shared verbatim by the CPU shim (through
// butterfly_core) and the GPU's register-resident fused stages, so both
// evaluate the same IEEE operations.
BFM_HD void butterfly_regs(const LinePlan& p, int r, cplx* x, int tw, bool inverse) {
  const int m = p.m;
  if (r == 2) {
    const cplx a = x[0];
    const cplx c = x[1];
    x[0] = cadd(a, c);
    const cplx d = csub(a, c);
    const cplx w = tab_c(p.wm, tw);
    x[1] = inverse ? cmulc(d, w) : cmul(d, w);
  } else if (r == 4) {
    const cplx x0 = x[0], x1 = x[1], x2 = x[2], x3 = x[3];
    const cplx a0 = cadd(x0, x2), a1 = csub(x0, x2);
    const cplx b0 = cadd(x1, x3), b1 = csub(x1, x3);
    // forward: y1 = a1 - i b1, y3 = a1 + i b1; inverse swaps the rotation.
    const cplx ib1{-b1.im, b1.re};
    const cplx y0 = cadd(a0, b0);
    const cplx y2 = csub(a0, b0);
    const cplx y1 = inverse ? cadd(a1, ib1) : csub(a1, ib1);
    const cplx y3 = inverse ? csub(a1, ib1) : cadd(a1, ib1);
    x[0] = y0;
    int t2 = 2 * tw;
    if (t2 >= m) t2 -= m;
    int t3 = t2 + tw;
    if (t3 >= m) t3 -= m;
    const cplx w1 = tab_c(p.wm, tw);
    const cplx w2 = tab_c(p.wm, t2);
    const cplx w3 = tab_c(p.wm, t3);
    if (inverse) {
      x[1] = cmulc(y1, w1);
      x[2] = cmulc(y2, w2);
      x[3] = cmulc(y3, w3);
    } else {
      x[1] = cmul(y1, w1);
      x[2] = cmul(y2, w2);
      x[3] = cmul(y3, w3);
    }
  } else {  // r == 3
    const cplx x0 = x[0], x1 = x[1], x2 = x[2];
    const cplx t1 = cadd(x1, x2);
    const cplx y0 = cadd(x0, t1);
    const cplx t2c{x0.re - 0.5 * t1.re, x0.im - 0.5 * t1.im};
    const cplx d = csub(x1, x2);
    const double h3 = 0.86602540378443864676;  // sqrt(3)/2
    const cplx u{h3 * d.re, h3 * d.im};
    const cplx iu{-u.im, u.re};
    // forward: y1 = t2 - i u, y2 = t2 + i u.
    const cplx y1 = inverse ? cadd(t2c, iu) : csub(t2c, iu);
    const cplx y2 = inverse ? csub(t2c, iu) : cadd(t2c, iu);
    x[0] = y0;
    int t2 = 2 * tw;
    if (t2 >= m) t2 -= m;
    const cplx w1 = tab_c(p.wm, tw);
    const cplx w2 = tab_c(p.wm, t2);
    if (inverse) {
      x[1] = cmulc(y1, w1);
      x[2] = cmulc(y2, w2);
    } else {
      x[1] = cmul(y1, w1);
      x[2] = cmul(y2, w2);
    }
  }
}

// One DIF butterfly on z[base + t*q], t < r (in place).
BFM_HD void butterfly_core(const LinePlan& p, int r, int base, int q, int tw, cplx* z,
                           bool inverse) {
  cplx x[4];
  for (int t = 0; t < r; ++t) x[t] = z[base + t * q];
  butterfly_regs(p, r, x, tw, inverse);
  for (int t = 0; t < r; ++t) z[base + t * q] = x[t];
}

// One DIF butterfly of stage s on the complex buffer z (in place).
// inverse = true uses e^{+2 pi i / m}.
BFM_HD void fft_butterfly(const LinePlan& p, int s, int b, cplx* z, bool inverse) {
  const int r = p.radix[s];
  const int L = p.span[s];
  const int q = L / r;
  const int blk = b / q;
  const int j = b - blk * q;
  butterfly_core(p, r, blk * L + j, q, (p.m / L) * j, z, inverse);
}

// ---- DCT-II (REDFT10) ----------------------------------------------------
// Pack: z_q = v_{2q} + i v_{2q+1}, v_p = x_{2p} (p < m), v_p = x_{2(n-1-p)+1}.
BFM_HD double dct2_v(const LinePlan& p, const double* x, long stride, int idx) {
  const int src = idx < p.m ? 2 * idx : 2 * (p.n - 1 - idx) + 1;
  return x[static_cast<long>(src) * stride];
}
BFM_HD void dct2_pack(const LinePlan& p, const double* x, long stride, cplx* z, int q) {
  z[q] = cplx{dct2_v(p, x, stride, 2 * q), dct2_v(p, x, stride, 2 * q + 1)};
}
// Unpack for k in [0, m] from zk = Z_k (Z_m = Z_0) and zm = Z_{m-k}: gives
// Y_k and, for 0 < k < m, Y_{n-k}.
BFM_HD void dct2_unpack_vals(const LinePlan& p, cplx zk, cplx zm, int k, double& yk,
                             double& ynk) {
  const cplx E = zk;
  const cplx F{zm.re, -zm.im};
  const cplx S{0.5 * (E.re + F.re), 0.5 * (E.im + F.im)};
  const cplx D{0.5 * (E.re - F.re), 0.5 * (E.im - F.im)};
  const cplx wk = tab_c(p.wn, k);
  const cplx w{wk.re, -wk.im};  // e^{-2 pi i k / n}
  // V = S - i w D
  const double vr = S.re + (w.re * D.im + w.im * D.re);
  const double vi = S.im - (w.re * D.re - w.im * D.im);
  const cplx csk = tab_c(p.cs, k);
  const double c = csk.re, s = csk.im;
  yk = 2.0 * (c * vr + s * vi);
  ynk = 2.0 * (s * vr - c * vi);
}
BFM_HD void dct2_unpack(const LinePlan& p, const cplx* z, double* y, long stride, int k) {
  const int m = p.m;
  const cplx zk = z[tab_i(p.rev, k == m ? 0 : k)];
  const cplx zm = z[tab_i(p.rev, k == 0 ? 0 : m - k)];
  double yk, ynk;
  dct2_unpack_vals(p, zk, zm, k, yk, ynk);
  y[static_cast<long>(k) * stride] = yk;
  if (k > 0 && k < m) y[static_cast<long>(p.n - k) * stride] = ynk;
}

// ---- DCT-III (REDFT01) ---------------------------------------------------
// V_j = (x_j - i x_{n-j}) e^{i pi j / 2n}, x_n = 0;
// Z_k = (V_k + conj V_{m-k}) + i e^{2 pi i k / n} (V_k - conj V_{m-k}), k < m.
// V_j from a = x_j and b = x_{n-j} (b = 0 for j = 0).
BFM_HD cplx dct3_V_vals(const LinePlan& p, double a, double b, int j) {
  const cplx csj = tab_c(p.cs, j);
  const double c = csj.re, s = csj.im;
  // (a - i b)(c + i s) = (a c + b s) + i (a s - b c)
  return cplx{a * c + b * s, a * s - b * c};
}
BFM_HD cplx dct3_V(const LinePlan& p, const double* x, long stride, int j) {
  const double a = x[static_cast<long>(j) * stride];
  const double b = j == 0 ? 0.0 : x[static_cast<long>(p.n - j) * stride];
  return dct3_V_vals(p, a, b, j);
}
// Z_k from A = V_k and Bv = V_{m-k}.
BFM_HD cplx dct3_pre_vals(const LinePlan& p, cplx A, cplx Bv, int k) {
  const cplx B{Bv.re, -Bv.im};
  const cplx sum = cadd(A, B);
  const cplx dif = csub(A, B);
  const cplx w = tab_c(p.wn, k);  // e^{+2 pi i k / n}
  const cplx wd = cmul(w, dif);
  // + i * wd
  return cplx{sum.re - wd.im, sum.im + wd.re};
}
BFM_HD void dct3_pre(const LinePlan& p, const double* x, long stride, cplx* z, int k) {
  const int m = p.m;
  z[k] = dct3_pre_vals(p, dct3_V(p, x, stride, k), dct3_V(p, x, stride, m - k), k);
}
// Output position of v_p in y: y_{2p} = v_p (p < m), y_{2(n-1-p)+1} = v_p.
BFM_HD int dct3_ypos(const LinePlan& p, int vp) {
  return vp < p.m ? 2 * vp : 2 * (p.n - 1 - vp) + 1;
}
// Input position of x_j in the packed DCT-II sequence v (inverse of dct2_v).
BFM_HD int dct2_vpos(const LinePlan& p, int j) {
  return (j & 1) == 0 ? j / 2 : p.n - 1 - (j - 1) / 2;
}
// After the inverse FFT: z_q at slot rev[q] holds (v_{2q}, v_{2q+1});
// y_{2p} = v_p, y_{2p+1} = v_{n-1-p}.
BFM_HD void dct3_post(const LinePlan& p, const cplx* z, double* y, long stride, int q) {
  const cplx v = z[tab_i(p.rev, q)];
  const int n = p.n;
  const int m = p.m;
  const int p0 = 2 * q, p1 = 2 * q + 1;
  const int y0 = p0 < m ? 2 * p0 : 2 * (n - 1 - p0) + 1;
  const int y1 = p1 < m ? 2 * p1 : 2 * (n - 1 - p1) + 1;
  y[static_cast<long>(y0) * stride] = v.re;
  y[static_cast<long>(y1) * stride] = v.im;
}

// ---- direct O(n^2) forms -------------------------------------------------
BFM_HD double dct2_naive(const LinePlan& p, const double* x, long stride, int k) {
  const int n = p.n;
  double acc = 0.0;
  const double* row = p.cosmat + static_cast<long>(k) * n;
  for (int j = 0; j < n; ++j) acc = acc + x[static_cast<long>(j) * stride] * row[j];
  return 2.0 * acc;
}
BFM_HD double dct3_naive(const LinePlan& p, const double* x, long stride, int k) {
  const int n = p.n;
  double acc = 0.0;
  for (int j = 1; j < n; ++j)
    acc = acc + x[static_cast<long>(j) * stride] * p.cosmat[static_cast<long>(j) * n + k];
  return x[0] + 2.0 * acc;
}

}  // namespace bfmdct
