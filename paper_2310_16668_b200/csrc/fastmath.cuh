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

__device__ __forceinline__ void sincos_tab_scaled(const double2* __restrict__ tab, double x,
                                                  double w, double* re, double* im) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: n lands in the low word
  const double nd = fma(x, 40.74366543152520595683, magic);  // 128/pi
  const int k = __double2loint(nd) & (kSinCosTab - 1);
  const double n = nd - magic;
  double t = fma(-n, 1.57079632673412561417e+00 / 64, x);
  t = fma(-n, 6.07710050630396597660e-11 / 64, t);
  t = fma(-n, 2.02226624879595063154e-21 / 64, t);
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
