// Branch-free FP64 sincos for the Helmholtz kernel, |x| <= 2^20.
//
// kappa * r stays small in every configuration (kappa = 10, r <= sqrt(3) in
// the unit cube), so the general library sincos -- which keeps a Payne-Hanek
// slow path behind a branch -- does more work than needed.  Here: Cody-Waite
// reduction by pi/2 in three FMA steps (fdlibm's pio2_1/pio2_2/pio2_2t split,
// exact for |j| < 2^20), then the fdlibm __kernel_sin / __kernel_cos minimax
// polynomials on |t| <= pi/4 (< 1 ulp), then the quadrant swap.  About 22
// FP64 instructions.  Checked against the CUDA math library in
// tests/test_kernels_gpu.py.
#pragma once

#include <cmath>

namespace sfmm_gpu {

// ---- table-driven variant (the translation kernels) ----------------------
// x = n pi/128 + t with |t| <= pi/256 (Cody-Waite, the fdlibm pi/2 split
// scaled by 1/64, exact for |n| < 2^20); sin t and cos t from their Taylor
// series to degree 7 / 6 (truncation < 1e-20); then one complex product with
// (cos, sin)(k pi/128), k = n mod 256, from a 256-entry table the caller keeps
// in shared memory.  The scale w (1/r in the kernels) is folded into the table
// entry.  About 16 FP64 instructions; checked in tests/test_kernels_gpu.py.
constexpr int kSinCosTab = 256;
constexpr double kSinCosTabMaxArg = 2.0e4;  // |n| < 2^20 with margin (2^20 pi/128 = 25736)

// (cos, sin)(k pi/128), correctly rounded from long double.
inline void fill_sincos_table(double2* out) {
  const long double step = 3.141592653589793238462643383279502884L / 128.0L;
  for (int k = 0; k < kSinCosTab; ++k) {
    out[k].x = static_cast<double>(cosl(step * k));
    out[k].y = static_cast<double>(sinl(step * k));
  }
}

// ---- table-driven log (the Laplace-2D kernels) ----------------------------
// x = 2^e m, m in [1, 2); k = top 7 mantissa bits; c = 1 + k/128 (left end,
// m < sqrt 2) or 1 + (k+1)/128 with e + 1 (right end, so x just below 1 gives
// no cancellation); t = m (1/c)_rounded - 1, |t| < 1/128; log x = e ln2 +
// log(1/(1/c)_rounded) + log1p(t) with a degree-8 Taylor log1p (truncation
// < 2e-20 relative).  Zero, subnormal, inf and NaN take the library log (so
// coincident points still give -inf).  About 14 FP64 instructions instead of
// the library's 29; checked in tests/test_kernels_gpu.py.
constexpr int kLogTab = 128;

// per entry: {1/c rounded, -log(that) - (k >= 53 ? ln2 : 0) as hi + lo}
inline void fill_log_table(double* out) {
  const long double ln2 = 0.693147180559945309417232121458176568L;
  for (int k = 0; k < kLogTab; ++k) {
    const bool upper = k >= 53;  // m >= 1 + 53/128 > sqrt 2
    const long double c = 1.0L + (upper ? k + 1 : k) / 128.0L;
    const double inv = static_cast<double>(1.0L / c);
    const long double lc = -logl(static_cast<long double>(inv)) - (upper ? ln2 : 0.0L);
    const double hi = static_cast<double>(lc);
    out[3 * k] = inv;
    out[3 * k + 1] = hi;
    out[3 * k + 2] = static_cast<double>(lc - hi);
  }
}

__device__ __forceinline__ double log_tab(const double* __restrict__ tab, double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  if (hi < 0x00100000 || hi >= 0x7ff00000) return log(x);  // 0, subnormal, inf, NaN, < 0
  const int k = (hi >> 13) & (kLogTab - 1);
  const int e = (hi >> 20) - 1023 + (k >= 53 ? 1 : 0);
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double t = fma(m, tab[3 * k], -1.0);
  double p = fma(t, 1.0 / 8, -1.0 / 7);
  p = fma(t, p, 1.0 / 6);
  p = fma(t, p, -1.0 / 5);
  p = fma(t, p, 1.0 / 4);
  p = fma(t, p, -1.0 / 3);
  p = fma(t, p, 0.5);
  p = fma(t, -p, 1.0);
  p = p * t;  // log1p(t)
  // e as a double through the 2^52 magic (integer ops and one DADD)
  const double ed = __hiloint2double(0x43300000, e ^ 0x80000000) - 4503601774854144.0;
  const double a = fma(ed, 6.93147180369123816490e-01, tab[3 * k + 1]);  // ln2 hi: e ln2_hi exact
  const double b = fma(ed, 1.90821492927058770002e-10, tab[3 * k + 2] + p);
  return a + b;
}

// 2-part Cody-Waite reduction in sincos_tab_scaled (A/B, complex K2 at N=2e6:
// 65.7 -> 63.3 ms; 16-RHS K2m at 4e6: 613.8 -> 606.9 ms)
#ifndef SFMM_SC_2PART
#define SFMM_SC_2PART 1
#endif
// kappa * r from r^2 and y = 1/r: (kappa r^2) y starts before the rsqrt ends
#ifndef SFMM_KR_EARLY
#define SFMM_KR_EARLY 1
#endif
#if SFMM_KR_EARLY
#define KR_ARG(kappa, r2, y) (((kappa) * (r2)) * (y))
#else
#define KR_ARG(kappa, r2, y) ((kappa) * ((r2) * (y)))
#endif
__device__ __forceinline__ void sincos_tab_scaled(const double2* __restrict__ tab, double x,
                                                  double w, double* re, double* im) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: n lands in the low word
  const double nd = fma(x, 40.74366543152520595683, magic);  // 128/pi
  const int k = __double2loint(nd) & (kSinCosTab - 1);
  const double n = nd - magic;
#if SFMM_SC_2PART
  // |n| < 2^20 (|x| <= kSinCosTabMaxArg): the 33-bit head of pi/2 times n is
  // exact and its 53-bit tail leaves an argument error below 1e-22
  double t = fma(-n, 1.57079632673412561417e+00 / 64, x);
  t = fma(-n, 6.07710050650619224932e-11 / 64, t);
#else
  double t = fma(-n, 1.57079632673412561417e+00 / 64, x);
  t = fma(-n, 6.07710050630396597660e-11 / 64, t);
  t = fma(-n, 2.02226624879595063154e-21 / 64, t);
#endif
  const double z = t * t;
  double ps = fma(z, -1.0 / 5040, 1.0 / 120);
  ps = fma(z, ps, -1.0 / 6);
  const double s = fma(t * z, ps, t);
  double pc = fma(z, -1.0 / 720, 1.0 / 24);
  pc = fma(z, pc, -0.5);
  const double c = fma(z, pc, 1.0);
  const double2 T = tab[k];
  const double tc = T.x * w, ts = T.y * w;
  *re = fma(tc, c, -ts * s);
  *im = fma(ts, c, tc * s);
}

__device__ __forceinline__ void sincos_fast(double x, double* sp, double* cp) {
  const double j = rint(x * 0.63661977236758134308);  // 2/pi
  double t = fma(-j, 1.57079632673412561417e+00, x);
  t = fma(-j, 6.07710050630396597660e-11, t);
  t = fma(-j, 2.02226624879595063154e-21, t);
  const double z = t * t;
  // sin(t) = t + t^3 (S1 + z S2 + ... + z^5 S6)
  double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  ps = fma(z, ps, 2.75573137070700676789e-06);
  ps = fma(z, ps, -1.98412698298579493134e-04);
  ps = fma(z, ps, 8.33333333332248946124e-03);
  ps = fma(z, ps, -1.66666666666666324348e-01);
  const double s = fma(t * z, ps, t);
  // cos(t) = 1 - z/2 + z^2 (C1 + z C2 + ... + z^5 C6), fdlibm's error-compensated form
  double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  pc = fma(z, pc, -2.75573143513906633035e-07);
  pc = fma(z, pc, 2.48015872894767294178e-05);
  pc = fma(z, pc, -1.38888888888741095749e-03);
  pc = fma(z, pc, 4.16666666666666019037e-02);
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double c = w + (((1.0 - w) - hz) + z * z * pc);
  const int q = static_cast<int>(static_cast<long long>(j) & 3);
  const double sv = (q & 1) ? c : s;
  const double cv = (q & 1) ? s : c;
  *sp = (q & 2) ? -sv : sv;
  *cp = ((q + 1) & 2) ? -cv : cv;
}

}  // namespace sfmm_gpu
